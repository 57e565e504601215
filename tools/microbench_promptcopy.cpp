// Host copy of one 128K-token prompt (512 KiB) into pooled pinned mapped
// buffers — the lookup's query-state copy and token packing — by plain
// memcpy, SSE2 streaming (non-temporal) stores, and split across persistent
// spinning helper threads. Build: g++ -O3 -std=c++20 -pthread
// tools/microbench_promptcopy.cpp -I/usr/local/cuda/include
// -L/usr/local/cuda/lib64 -lcudart -o /tmp/promptcopy
#include <cuda_runtime.h>
#include <emmintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void copy_nt(void* dst, const void* src, size_t n) {
    auto* d = static_cast<__m128i*>(dst);
    auto* s = static_cast<const __m128i*>(src);
    const size_t v = n / 16;
    size_t i = 0;
    for (; i + 4 <= v; i += 4) {
        const __m128i a = _mm_loadu_si128(s + i), b = _mm_loadu_si128(s + i + 1);
        const __m128i c = _mm_loadu_si128(s + i + 2), e = _mm_loadu_si128(s + i + 3);
        _mm_stream_si128(d + i, a);
        _mm_stream_si128(d + i + 1, b);
        _mm_stream_si128(d + i + 2, c);
        _mm_stream_si128(d + i + 3, e);
    }
    for (; i < v; ++i) _mm_stream_si128(d + i, _mm_loadu_si128(s + i));
    std::memcpy(static_cast<char*>(dst) + 16 * v, static_cast<const char*>(src) + 16 * v, n - 16 * v);
    _mm_sfence();
}

struct Helpers {
    std::vector<std::thread> th;
    std::atomic<uint64_t> gen{0};
    std::atomic<int> done{0};
    std::atomic<bool> stop{false};
    char* dst = nullptr;
    const char* src = nullptr;
    size_t n = 0;
    int parts = 1;
    bool nt = false;
    explicit Helpers(int k) : parts(k + 1) {
        for (int t = 0; t < k; ++t)
            th.emplace_back([this, t] {
                uint64_t seen = 0;
                while (!stop.load(std::memory_order_relaxed)) {
                    const uint64_t g = gen.load(std::memory_order_acquire);
                    if (g == seen) {
                        _mm_pause();
                        continue;
                    }
                    seen = g;
                    part(t + 1);
                    done.fetch_add(1, std::memory_order_release);
                }
            });
    }
    ~Helpers() {
        stop = true;
        for (auto& t : th) t.join();
    }
    void part(int p) {
        const size_t chunk = (n / parts + 63) / 64 * 64;
        const size_t b = std::min(n, chunk * size_t(p)), e = std::min(n, b + chunk);
        if (e > b) (nt ? copy_nt(dst + b, src + b, e - b) : (void)std::memcpy(dst + b, src + b, e - b));
    }
    void run(char* d, const char* s, size_t bytes, bool use_nt) {
        dst = d;
        src = s;
        n = bytes;
        nt = use_nt;
        done.store(0, std::memory_order_relaxed);
        gen.fetch_add(1, std::memory_order_release);
        part(0);
        while (done.load(std::memory_order_acquire) != parts - 1) _mm_pause();
    }
};

int main() {
    const size_t n = 512 * 1024;
    const int kBufs = 16;
    std::vector<char*> dst(kBufs);
    for (auto& d : dst) cudaHostAlloc(reinterpret_cast<void**>(&d), n, cudaHostAllocMapped | cudaHostAllocPortable);
    std::vector<char> src(n);
    for (size_t i = 0; i < n; ++i) src[i] = char(i * 7);
    std::vector<char> big(64 << 20, 1);  // evicts the caches for the cold-source rows
    auto bench = [&](const char* name, auto fn, bool cold_src) {
        std::vector<double> t;
        for (int r = 0; r < 64; ++r) {
            if (cold_src)
                for (size_t i = 0; i < big.size(); i += 64) big[i]++;
            else
                std::memcpy(big.data(), src.data(), 4096);
            char* d = dst[r % kBufs];
            const double t0 = now_us();
            fn(d);
            t.push_back(now_us() - t0);
        }
        std::sort(t.begin(), t.end());
        std::printf("{\"copy\": \"%s\", \"src\": \"%s\", \"median_us\": %.1f, \"p10_us\": %.1f, \"GBps\": %.1f}\n", name,
                    cold_src ? "cold" : "warm", t[t.size() / 2], t[t.size() / 10], n / t[t.size() / 2] / 1e3);
    };
    for (bool cold : {false, true}) {
        bench("memcpy", [&](char* d) { std::memcpy(d, src.data(), n); }, cold);
        bench("sse2-stream", [&](char* d) { copy_nt(d, src.data(), n); }, cold);
        for (int k : {1, 3, 7}) {
            Helpers h(k);
            char name[64];
            std::snprintf(name, sizeof name, "memcpy x%d threads", k + 1);
            bench(name, [&](char* d) { h.run(d, src.data(), n, false); }, cold);
            std::snprintf(name, sizeof name, "stream x%d threads", k + 1);
            bench(name, [&](char* d) { h.run(d, src.data(), n, true); }, cold);
        }
    }
    return 0;
}
