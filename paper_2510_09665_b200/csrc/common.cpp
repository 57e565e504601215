#include "common.hpp"

#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <utility>

#include "kernels.hpp"

namespace tkv {

namespace {
std::atomic<uint64_t> g_launches{0};
}
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

const char* errc_name(Errc e) {
    switch (e) {
        case Errc::ok: return "ok";
        case Errc::not_found: return "not_found";
        case Errc::tier_full: return "tier_full";
        case Errc::out_of_pages: return "out_of_pages";
        case Errc::duplicate_key: return "duplicate_key";
        case Errc::corrupt_chunk: return "corrupt_chunk";
        case Errc::size_mismatch: return "size_mismatch";
        case Errc::unpopulated_page: return "unpopulated_page";
        case Errc::unknown_codec: return "unknown_codec";
        case Errc::unknown_instance: return "unknown_instance";
        case Errc::unknown_query: return "unknown_query";
        case Errc::inconsistent_alloc: return "inconsistent_alloc";
        case Errc::chunk_missing: return "chunk_missing";
        case Errc::pinned: return "pinned";
        case Errc::protocol_error: return "protocol_error";
        case Errc::io_error: return "io_error";
        case Errc::invalid_argument: return "invalid_argument";
        case Errc::cuda_error: return "cuda_error";
    }
    return "unknown";
}

std::string Status::to_string() const {
    std::string s = errc_name(code);
    if (!detail.empty()) s += ": " + detail;
    return s;
}

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    throw CudaError(std::string(cudaGetErrorString(e)) + " in " + what + " at " + file + ":" +
                    std::to_string(line));
}

PinnedBuffer::PinnedBuffer(size_t n) { reserve(n); }

PinnedBuffer::~PinnedBuffer() { release(); }

void PinnedBuffer::release() {
    if (host) {
        if (map_base) {
            cudaHostUnregister(host);
            munmap(map_base, map_bytes);
        } else {
            cudaFreeHost(host);
        }
    }
    host = dev = nullptr;
    map_base = nullptr;
    bytes = map_bytes = 0;
}

void PinnedBuffer::reserve(size_t n) {
    if (n <= bytes) return;
    if (bytes) n = std::max(n, bytes + bytes / 2);  // regrow rarely: pinning is slow and synchronizes
    release();
    void* p = nullptr;
    constexpr size_t kHuge = size_t(2) << 20;
    if (huge && n >= 32 * kHuge) {
        const size_t len = (n + kHuge - 1) / kHuge * kHuge;
        void* m = mmap(nullptr, len + kHuge, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (m != MAP_FAILED) {
            auto* a = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(m) + kHuge - 1) & ~(kHuge - 1));
            madvise(a, len, MADV_HUGEPAGE);  // advisory: ignored where THP is off
            if (cudaHostRegister(a, len, cudaHostRegisterMapped | cudaHostRegisterPortable) == cudaSuccess) {
                p = a;
                map_base = m;
                map_bytes = len + kHuge;
            } else {
                cudaGetLastError();
                munmap(m, len + kHuge);
            }
        }
    }
    if (!p) TKV_CUDA(cudaHostAlloc(&p, n, cudaHostAllocMapped | cudaHostAllocPortable));
    host = static_cast<uint8_t*>(p);
    void* d = nullptr;
    TKV_CUDA(cudaHostGetDevicePointer(&d, p, 0));
    dev = static_cast<uint8_t*>(d);
    bytes = n;
}

DeviceBuffer::DeviceBuffer(size_t n) { reserve(n); }

DeviceBuffer::~DeviceBuffer() {
    if (ptr) cudaFree(ptr);
}

void DeviceBuffer::reserve(size_t n) {
    if (n <= bytes) return;
    if (bytes) n = std::max(n, bytes + bytes / 2);  // regrow rarely: cudaFree/cudaMalloc synchronize
    if (ptr) TKV_CUDA(cudaFree(ptr));
    ptr = nullptr;
    bytes = 0;
    void* p = nullptr;
    TKV_CUDA(cudaMalloc(&p, n));
    ptr = static_cast<uint8_t*>(p);
    bytes = n;
}

std::unique_ptr<DualBuffer> DualPool::acquire(size_t bytes) {
    {
        std::lock_guard lock(mu_);
        size_t best = free_.size();
        for (size_t i = 0; i < free_.size(); ++i)
            if (free_[i]->host.bytes >= bytes &&
                (best == free_.size() || free_[i]->host.bytes < free_[best]->host.bytes))
                best = i;
        if (best != free_.size()) {
            auto b = std::move(free_[best]);
            free_.erase(free_.begin() + long(best));
            return b;
        }
        ++created_;
    }
    size_t cap = 4096;
    while (cap < bytes) cap <<= 1;
    auto b = std::make_unique<DualBuffer>();
    b->host.reserve(cap);
    b->dev.reserve(cap);
    return b;
}

void DualPool::release(std::unique_ptr<DualBuffer> b) {
    if (!b) return;
    std::lock_guard lock(mu_);
    free_.push_back(std::move(b));
}

size_t DualPool::blocks() const {
    std::lock_guard lock(mu_);
    return created_;
}

Stream Stream::create(int priority) {
    cudaStream_t s = nullptr;
    TKV_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority));
    return Stream{s, true};
}

Stream::~Stream() {
    if (owned && s) cudaStreamDestroy(s);
}

Event::Event() { TKV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
Event::Event(bool timing) {
    TKV_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
}
Event::~Event() {
    if (e) cudaEventDestroy(e);
}
void Event::record(cudaStream_t s) const { TKV_CUDA(cudaEventRecord(e, s)); }
void Event::wait_on(cudaStream_t s) const { TKV_CUDA(cudaStreamWaitEvent(s, e, 0)); }
void Event::sync() const { TKV_CUDA(cudaEventSynchronize(e)); }

}  // namespace tkv
