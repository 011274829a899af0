// Kernel timing (CUDA events on the launching stream) and launch counting,
// used by bench.py to report per-kernel durations inside the timed region.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace isoc {
enum ProfKind {
    PK_SIGMA = 0,
    PK_OMEGA = 1,
    PK_FILTER = 2,
    PK_DECIDE = 3,
    PK_RESCAN = 4,
    PK_BFS = 5,
    PK_COST = 6,
    PK_COUNT = 7
};
void note_launch(int k = 1);
// returns an event pair index (or -1 when profiling is off); record the end
// with prof_end(idx, stream) after the launch
int prof_begin(int kind, cudaStream_t st);
void prof_end(int idx, cudaStream_t st);
}  // namespace isoc
