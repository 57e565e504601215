// Copy-engine transfers of many host<->device pieces on one stream.
//
// A layer of a load or store batch is one piece per chunk: the chunk's layer
// slice in its pinned slot (slab + slot * slot_bytes + l * T * bpt) and its
// place in the packed HBM staging ring. The pieces are grouped into runs of
// equal width whose source and destination addresses both advance by a
// constant pitch (consecutive slots of the slab against consecutive ring
// offsets), and each run goes to the copy engine as ONE pitched copy
// (cudaMemcpy2DAsync: width = piece bytes, height = run length); a lone piece
// is a plain cudaMemcpyAsync. Per-piece copies of 1 MiB pieces reach only
// 46 GB/s one way and 49-63 GB/s both ways on this box
// (profiles/r01_microbench_streams.txt), one large copy 55 / 94.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

namespace tkv {

struct CopyRunStats {
    uint64_t pieces = 0;  // pieces submitted
    uint64_t runs = 0;    // copies issued (pitched copies + plain copies)
};

// One copy: `rows` pieces of `width` bytes starting at piece `first`, the
// next row `src_pitch` / `dst_pitch` bytes further on (rows == 1: no pitch).
struct CopyRun {
    size_t first = 0, rows = 1, width = 0, src_pitch = 0, dst_pitch = 0;
};

// Groups pieces into runs, greedily in order: a run continues while the
// width is the same and both addresses move by the run's first step; the
// steps must have one sign (a descending run is issued from its last piece),
// be at least one width (rows do not overlap) and at most `pitch_max`.
// Writes the runs to `runs` (capacity n; may be null) and returns their count.
size_t plan_copy_runs(void* const* dst, const void* const* src, const size_t* sizes, size_t n,
                      size_t pitch_max, CopyRun* runs);

// Enqueues dst[i] <- src[i] (sizes[i] bytes) for i < n on `stream`, in runs.
// Returns the first CUDA error; `stats` (optional) accumulates the counts.
cudaError_t ce_copy_pieces(void* const* dst, const void* const* src, const size_t* sizes, size_t n,
                           cudaMemcpyKind kind, cudaStream_t stream, CopyRunStats* stats = nullptr);

}  // namespace tkv
