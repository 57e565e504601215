// Host copies of prompt-sized buffers (lookup packing and the query state's
// prompt copy: 512 KiB for a 128K-token document) split over a few
// persistent helper threads with streaming stores. One thread moves ~10-28
// GB/s into pinned memory; four move 60-110 GB/s on the B200 hosts
// (tools/microbench_promptcopy.cpp, profiles/r02_promptcopy.jsonl).
#pragma once
#include <cstddef>

namespace tkv {

// memcpy semantics (no overlap). Small copies, and copies issued while
// another thread's parallel copy is running, run on the calling thread alone;
// the caller always works on its own pieces too, so a helper that wakes late
// costs nothing but its share.
void host_copy(void* dst, const void* src, size_t n);

// Wakes the helpers ahead of a burst of copies (a lookup calls it on entry):
// they then spin for the next ~100 us instead of sleeping, so the copies
// that follow find them awake (a futex wake-up costs tens of microseconds).
void host_copy_prime();

}  // namespace tkv
