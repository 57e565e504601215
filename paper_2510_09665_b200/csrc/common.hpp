// Error model, small value types and CUDA helpers shared by the host side.
//
// Mirrors the reference error model (include/tierkv/common.hpp:13-83): the
// same Errc values in the same order (they cross the C-ABI as ints), Status
// carrying a detail string, and Result<T> as value-or-status.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

namespace tkv {

enum class Errc : int {
    ok = 0,
    not_found,
    tier_full,
    out_of_pages,
    duplicate_key,
    corrupt_chunk,
    size_mismatch,
    unpopulated_page,
    unknown_codec,
    unknown_instance,
    unknown_query,
    inconsistent_alloc,
    chunk_missing,
    pinned,
    protocol_error,
    io_error,
    invalid_argument,
    cuda_error,  // device-side failure (no reference equivalent: the reference has no device)
};

const char* errc_name(Errc e);

struct Status {
    Errc code = Errc::ok;
    std::string detail;

    bool ok() const { return code == Errc::ok; }
    explicit operator bool() const { return ok(); }
    static Status success() { return {}; }
    static Status error(Errc c, std::string d = {}) { return {c, std::move(d)}; }
    std::string to_string() const;
};

template <typename T>
class Result {
public:
    Result(T value) : v_(std::move(value)) {}
    Result(Status status) : v_(std::move(status)) {
        if (std::get<Status>(v_).ok()) throw std::logic_error("Result error with ok status");
    }
    Result(Errc code, std::string detail = {}) : Result(Status::error(code, std::move(detail))) {}

    bool ok() const { return std::holds_alternative<T>(v_); }
    explicit operator bool() const { return ok(); }
    T& value() { return std::get<T>(v_); }
    const T& value() const { return std::get<T>(v_); }
    const Status& status() const {
        static const Status ok_status{};
        return ok() ? ok_status : std::get<Status>(v_);
    }
    Errc code() const { return ok() ? Errc::ok : status().code; }

private:
    std::variant<T, Status> v_;
};

using QueryId = uint64_t;
using TokenId = uint32_t;
using PageId = uint32_t;
using TokenSpanView = std::span<const TokenId>;
using Digest = std::array<uint8_t, 32>;
inline constexpr Digest kZeroDigest{};

struct DigestHasher {
    size_t operator()(const Digest& d) const {
        uint64_t v;
        std::memcpy(&v, d.data(), sizeof v);
        return size_t(v);
    }
};

// common.hpp:172-186 — used on the host only for the model seed (a constant
// per model tag) and never on payload bytes.
inline uint64_t fnv1a64(const uint8_t* p, size_t n, uint64_t h = 0xcbf29ce484222325ull) {
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

// fnv1a64 of src while copying it to dst: the checksum is a serial chain of
// one multiply per byte, so the 8-byte loads and stores ride under it for free.
inline uint64_t fnv1a64_copy(uint8_t* dst, const uint8_t* src, size_t n, uint64_t h = 0xcbf29ce484222325ull) {
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        uint64_t w;
        std::memcpy(&w, src + i, 8);
        std::memcpy(dst + i, &w, 8);
        for (int b = 0; b < 8; ++b) {
            h ^= (w >> (8 * b)) & 0xffu;
            h *= 0x100000001b3ull;
        }
    }
    for (; i < n; ++i) {
        dst[i] = src[i];
        h ^= src[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

// Layout of the KV a model produces (model.hpp:11-33).
struct ModelSpec {
    uint32_t num_layers = 8;
    uint32_t bytes_per_token_per_layer = 4096;
    uint32_t page_tokens = 16;
    std::string model_tag = "sim-8l";
    uint32_t vocab_size = 32000;

    size_t page_bytes() const { return size_t(page_tokens) * bytes_per_token_per_layer; }
    size_t chunk_layer_bytes(size_t chunk_size) const {
        return chunk_size * bytes_per_token_per_layer;
    }
    size_t chunk_bytes(size_t chunk_size) const {
        return size_t(num_layers) * chunk_layer_bytes(chunk_size);
    }
    void validate(size_t chunk_size) const {
        if (num_layers == 0 || bytes_per_token_per_layer == 0 || page_tokens == 0)
            throw std::invalid_argument("ModelSpec fields must be positive");
        if (vocab_size < 2) throw std::invalid_argument("vocab_size must be >= 2");
        if (chunk_size % page_tokens != 0)
            throw std::invalid_argument("page_tokens must divide chunk_size");
    }
    uint64_t model_seed() const {  // synth.hpp:27-30
        return fnv1a64(reinterpret_cast<const uint8_t*>(model_tag.data()), model_tag.size());
    }
};

// --- CUDA plumbing ----------------------------------------------------------

class CudaError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define TKV_CUDA(x) ::tkv::cuda_check((x), #x, __FILE__, __LINE__)

// Pinned, device-mapped host allocation (cudaHostAlloc Mapped|Portable).
// huge = true (large slabs): a 2 MiB-aligned anonymous mapping advised for
// transparent huge pages, then cudaHostRegister(Mapped|Portable) — fewer,
// physically larger pages for the copy engines' DMA (measured +1-4 % PCIe
// both-ways throughput on the B200 boxes, tools/microbench4.cu).
struct PinnedBuffer {
    uint8_t* host = nullptr;
    uint8_t* dev = nullptr;  // device-visible alias of `host`
    size_t bytes = 0;
    bool huge = false;
    void* map_base = nullptr;  // huge: the mmap to unmap
    size_t map_bytes = 0;
    PinnedBuffer() = default;
    explicit PinnedBuffer(size_t n);
    ~PinnedBuffer();
    PinnedBuffer(const PinnedBuffer&) = delete;
    PinnedBuffer& operator=(const PinnedBuffer&) = delete;
    PinnedBuffer(PinnedBuffer&& o) noexcept { swap(o); }
    PinnedBuffer& operator=(PinnedBuffer&& o) noexcept {
        swap(o);
        return *this;
    }
    void swap(PinnedBuffer& o) noexcept {
        std::swap(host, o.host);
        std::swap(dev, o.dev);
        std::swap(bytes, o.bytes);
        std::swap(huge, o.huge);
        std::swap(map_base, o.map_base);
        std::swap(map_bytes, o.map_bytes);
    }
    void reserve(size_t n);  // grow-only, contents not preserved
    void release();
};

// Device allocation (cudaMalloc), grow-only reserve.
// Allocator of mapped pinned host memory (cudaHostAlloc Mapped|Portable): a
// container's data() is then also a device address (UVA), so kernels read it
// over PCIe without a staging copy. Allocation and release are slow and can
// synchronize the device: such containers are pooled, not churned.
template <typename T>
struct PinnedAllocator {
    using value_type = T;
    PinnedAllocator() = default;
    template <typename U>
    PinnedAllocator(const PinnedAllocator<U>&) {}
    T* allocate(size_t n) {
        void* p = nullptr;
        TKV_CUDA(cudaHostAlloc(&p, std::max<size_t>(1, n) * sizeof(T), cudaHostAllocMapped | cudaHostAllocPortable));
        return static_cast<T*>(p);
    }
    void deallocate(T* p, size_t) { cudaFreeHost(p); }
    // resize() default-initialises (no zero fill: the buffer is overwritten)
    template <typename U>
    void construct(U* p) noexcept {
        ::new (static_cast<void*>(p)) U;
    }
    template <typename U, typename... A>
    void construct(U* p, A&&... a) {
        ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
    template <typename U>
    bool operator==(const PinnedAllocator<U>&) const { return true; }
};
using PinnedTokens = std::vector<TokenId, PinnedAllocator<TokenId>>;

struct DeviceBuffer {
    uint8_t* ptr = nullptr;
    size_t bytes = 0;
    DeviceBuffer() = default;
    explicit DeviceBuffer(size_t n);
    ~DeviceBuffer();
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept {
        std::swap(ptr, o.ptr);
        std::swap(bytes, o.bytes);
    }
    void reserve(size_t n);
};

// A pinned staging buffer paired with a device buffer of the same size, and
// a pool of them. cudaHostAlloc / cudaMalloc can synchronize the device, so
// nothing on the transfer path allocates once the pool is warm: per-batch
// plans and per-query page tables borrow blocks and return them.
struct DualBuffer {
    PinnedBuffer host;
    DeviceBuffer dev;
};

class DualPool {
public:
    std::unique_ptr<DualBuffer> acquire(size_t bytes);
    void release(std::unique_ptr<DualBuffer> b);
    size_t blocks() const;

private:
    mutable std::mutex mu_;
    std::vector<std::unique_ptr<DualBuffer>> free_;
    size_t created_ = 0;
};

struct Stream {
    cudaStream_t s = nullptr;
    bool owned = false;
    Stream() = default;
    static Stream create(int priority = 0);
    static Stream wrap(cudaStream_t s) { return Stream{s, false}; }
    Stream(cudaStream_t st, bool own) : s(st), owned(own) {}
    ~Stream();
    Stream(const Stream&) = delete;
    Stream& operator=(const Stream&) = delete;
    Stream(Stream&& o) noexcept {
        std::swap(s, o.s);
        std::swap(owned, o.owned);
    }
    Stream& operator=(Stream&& o) noexcept {
        std::swap(s, o.s);
        std::swap(owned, o.owned);
        return *this;
    }
    operator cudaStream_t() const { return s; }
};

struct Event {
    cudaEvent_t e = nullptr;
    Event();
    explicit Event(bool timing);
    ~Event();
    Event(const Event&) = delete;
    Event& operator=(const Event&) = delete;
    Event(Event&& o) noexcept { std::swap(e, o.e); }
    void record(cudaStream_t s) const;
    void wait_on(cudaStream_t s) const;  // s waits for this event
    void sync() const;
    operator cudaEvent_t() const { return e; }
};

}  // namespace tkv
