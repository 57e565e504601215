// Copy-engine piece transfers grouped into pitched runs (ce_copy.hpp).
#include "ce_copy.hpp"

#include <atomic>
#include <cstdlib>
#include <cstring>

namespace tkv {
namespace {

// Largest pitch a 2D copy accepts (cudaDevAttrMaxPitch), read once.
size_t max_pitch() {
    static std::atomic<long long> cached{-1};
    long long v = cached.load(std::memory_order_relaxed);
    if (v < 0) {
        int dev = 0, p = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&p, cudaDevAttrMaxPitch, dev) != cudaSuccess || p <= 0)
            p = 0;
        v = p;
        cached.store(v, std::memory_order_relaxed);
    }
    return size_t(v);
}

// TKV_CE_RUNS=0 issues one copy per piece (A/B measurement only).
bool runs_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TKV_CE_RUNS");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    return on;
}

inline std::ptrdiff_t delta(const void* a, const void* b) {
    return static_cast<const char*>(b) - static_cast<const char*>(a);
}

}  // namespace

size_t plan_copy_runs(void* const* dst, const void* const* src, const size_t* sizes, size_t n,
                      size_t pitch_max, CopyRun* runs) {
    size_t i = 0, k = 0;
    while (i < n) {
        const size_t w = sizes[i];
        size_t j = i + 1;  // run is [i, j)
        std::ptrdiff_t sp = 0, dp = 0;
        if (w > 0 && j < n && sizes[j] == w) {
            sp = delta(src[i], src[j]);
            dp = delta(dst[i], dst[j]);
            const std::ptrdiff_t sw = std::ptrdiff_t(w);
            // Both pitches the same sign and at least one piece wide (rows do
            // not overlap), within the 2D copy's pitch limit.
            const bool up = sp >= sw && dp >= sw;
            const bool down = sp <= -sw && dp <= -sw;
            const size_t asp = size_t(sp < 0 ? -sp : sp), adp = size_t(dp < 0 ? -dp : dp);
            if ((up || down) && asp <= pitch_max && adp <= pitch_max) {
                ++j;
                while (j < n && sizes[j] == w && delta(src[j - 1], src[j]) == sp &&
                       delta(dst[j - 1], dst[j]) == dp)
                    ++j;
            }
        }
        CopyRun r;
        r.rows = j - i;
        r.width = w;
        if (r.rows == 1) {
            r.first = i;
        } else {
            // A descending run is the same rows read from its last piece up.
            r.first = sp > 0 ? i : j - 1;
            r.src_pitch = size_t(sp < 0 ? -sp : sp);
            r.dst_pitch = size_t(dp < 0 ? -dp : dp);
        }
        if (runs) runs[k] = r;
        ++k;
        i = j;
    }
    return k;
}

cudaError_t ce_copy_pieces(void* const* dst, const void* const* src, const size_t* sizes, size_t n,
                           cudaMemcpyKind kind, cudaStream_t stream, CopyRunStats* stats) {
    const size_t pmax = runs_enabled() ? max_pitch() : 0;  // pitch limit 0: every piece alone
    thread_local std::vector<CopyRun> runs;
    runs.resize(n);
    const size_t k = plan_copy_runs(dst, src, sizes, n, pmax, runs.data());
    uint64_t issued = 0;
    for (size_t r = 0; r < k; ++r) {
        const CopyRun& c = runs[r];
        if (c.width == 0) continue;
        // A run's pitch x rows extent may reach past the slab by one pitch
        // less a width; the runtime accepts that for allocated and registered
        // pinned memory alike (tools/probe_pitch_extent.cu).
        cudaError_t e =
            c.rows == 1 ? cudaMemcpyAsync(dst[c.first], src[c.first], c.width, kind, stream)
                        : cudaMemcpy2DAsync(dst[c.first], c.dst_pitch, src[c.first], c.src_pitch,
                                            c.width, c.rows, kind, stream);
        if (e != cudaSuccess) return e;
        ++issued;
    }
    if (stats) {
        stats->pieces += n;
        stats->runs += issued;
    }
    return cudaSuccess;
}

}  // namespace tkv
