// Parallel host copy (host_copy.hpp). A job is cut into fixed pieces; the
// caller and the helpers claim pieces from a generation-tagged counter, so a
// helper that wakes after the job ended claims nothing, and a job's fields
// stay valid while any of its pieces is unfinished. Helpers spin briefly
// after a job (lookups come in bursts), then sleep on a futex.
#include "host_copy.hpp"

#include <emmintrin.h>
#include <pthread.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace tkv {
namespace {

constexpr size_t kParallelMin = 128 << 10;  // below this one thread is as fast
constexpr size_t kPiece = 64 << 10;

void copy_stream(void* dst, const void* src, size_t n) {
    auto* d = static_cast<char*>(dst);
    auto* s = static_cast<const char*>(src);
    // align the destination to 16 bytes, then streaming stores
    const size_t head = std::min(n, size_t((16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15));
    std::memcpy(d, s, head);
    d += head;
    s += head;
    n -= head;
    auto* dv = reinterpret_cast<__m128i*>(d);
    auto* sv = reinterpret_cast<const __m128i*>(s);
    const size_t v = n / 16;
    size_t i = 0;
    for (; i + 4 <= v; i += 4) {
        const __m128i a = _mm_loadu_si128(sv + i), b = _mm_loadu_si128(sv + i + 1);
        const __m128i c = _mm_loadu_si128(sv + i + 2), e = _mm_loadu_si128(sv + i + 3);
        _mm_stream_si128(dv + i, a);
        _mm_stream_si128(dv + i + 1, b);
        _mm_stream_si128(dv + i + 2, c);
        _mm_stream_si128(dv + i + 3, e);
    }
    for (; i < v; ++i) _mm_stream_si128(dv + i, _mm_loadu_si128(sv + i));
    std::memcpy(d + 16 * v, s + 16 * v, n - 16 * v);
}

// A forked child has the crew's state but none of its threads: it copies
// alone (its copies never wait for helpers that do not exist).
std::atomic<bool> g_forked{false};

class CopyCrew {
public:
    CopyCrew() {
        pthread_atfork(nullptr, nullptr, [] { g_forked.store(true); });
        const char* e = std::getenv("TKV_COPY_THREADS");  // helpers besides the caller
        unsigned k = e ? unsigned(std::atoi(e)) : std::min(3u, std::max(1u, std::thread::hardware_concurrency() / 4));
        for (unsigned t = 0; t < k; ++t) helpers_.emplace_back([this] { loop(); });
    }
    ~CopyCrew() {
        stop_.store(true);
        wake_.fetch_add(1);
        wake_.notify_all();
        for (auto& t : helpers_) t.join();
    }
    bool enabled() const { return !helpers_.empty() && !g_forked.load(std::memory_order_relaxed); }
    void prime() {
        wake_.fetch_add(1, std::memory_order_release);
        wake_.notify_all();
    }

    void run(void* dst, const void* src, size_t n) {
        std::unique_lock<std::mutex> lock(job_mu_, std::try_to_lock);
        if (!lock.owns_lock()) {  // another caller's job is running
            std::memcpy(dst, src, n);
            return;
        }
        dst_ = static_cast<char*>(dst);
        src_ = static_cast<const char*>(src);
        n_ = n;
        const uint32_t pieces = uint32_t((n + kPiece - 1) / kPiece);
        pieces_.store(pieces, std::memory_order_relaxed);
        done_.store(0, std::memory_order_relaxed);
        gen_ += 1;
        next_.store(uint64_t(gen_) << 32, std::memory_order_release);  // publishes the fields above
        wake_.fetch_add(1, std::memory_order_release);
        wake_.notify_all();
        work(gen_);
        while (done_.load(std::memory_order_acquire) != pieces) _mm_pause();
        _mm_sfence();
    }

private:
    // claims and copies pieces of job `gen` until none is left
    void work(uint32_t gen) {
        uint64_t cur = next_.load(std::memory_order_acquire);
        for (;;) {
            if (uint32_t(cur >> 32) != gen) return;
            const uint32_t k = uint32_t(cur);
            if (k >= pieces_.load(std::memory_order_relaxed)) return;
            if (!next_.compare_exchange_weak(cur, cur + 1, std::memory_order_acq_rel)) continue;
            const size_t b = size_t(k) * kPiece, len = std::min(kPiece, n_ - b);
            copy_stream(dst_ + b, src_ + b, len);
            _mm_sfence();
            done_.fetch_add(1, std::memory_order_release);
            cur = next_.load(std::memory_order_acquire);
        }
    }

    void loop() {
        uint32_t seen = wake_.load();
        while (!stop_.load(std::memory_order_relaxed)) {
            // spin ~100 us for the next job (or prime), then sleep until woken
            const auto t0 = std::chrono::steady_clock::now();
            uint32_t w;
            while ((w = wake_.load(std::memory_order_acquire)) == seen &&
                   std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(100))
                _mm_pause();
            if (w == seen) {
                wake_.wait(seen, std::memory_order_acquire);
                w = wake_.load(std::memory_order_acquire);
            }
            seen = w;
            if (stop_.load()) return;
            const uint64_t cur = next_.load(std::memory_order_acquire);
            work(uint32_t(cur >> 32));
        }
    }

    std::mutex job_mu_;
    std::vector<std::thread> helpers_;
    std::atomic<uint32_t> wake_{0};
    std::atomic<uint64_t> next_{0};  // (generation << 32) | next piece
    std::atomic<uint32_t> done_{0};
    std::atomic<bool> stop_{false};
    uint32_t gen_ = 0;  // guarded by job_mu_
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t n_ = 0;
    std::atomic<uint32_t> pieces_{0};
};

// Never destroyed: helpers may be asleep in a futex at process exit, and a
// joined-at-exit crew would hang a forked child that inherited it.
CopyCrew& crew() {
    static CopyCrew* c = new CopyCrew;
    return *c;
}

}  // namespace

void host_copy_prime() {
    CopyCrew& c = crew();
    if (c.enabled()) c.prime();
}

void host_copy(void* dst, const void* src, size_t n) {
    if (n < kParallelMin) {
        std::memcpy(dst, src, n);
        return;
    }
    CopyCrew& c = crew();
    if (!c.enabled()) {
        std::memcpy(dst, src, n);
        return;
    }
    c.run(dst, src, n);
}

}  // namespace tkv
