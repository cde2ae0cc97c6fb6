// rng.h — device generator of the reference's synthetic weights.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pgmoe {

struct GenJob {
    void *out;
    uint64_t seed;
    int64_t n;
};

// core.py:22-28 substream tags
enum { kTagGate = 0, kTagPreGate = 1, kTagW1 = 2, kTagW2 = 3, kTagDense = 4, kTagInput = 5 };

uint64_t derive_seed(uint64_t base, const int64_t *tags, int ntags);
uint64_t matrix_seed(uint64_t seed, int tag, int block, int expert);
int gen_matrices(const GenJob *jobs_dev, int njobs, int wdtype, cudaStream_t s);

}  // namespace pgmoe
