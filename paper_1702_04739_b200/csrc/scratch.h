// Stream-ordered scratch freed on every return path (host side).
#pragma once
#include <cstddef>
#include <cuda_runtime.h>

namespace isoc {

cudaError_t isoc_malloc_async(void** p, size_t bytes, cudaStream_t st);   // alloc.cu
cudaError_t isoc_free_async(void* p, cudaStream_t st);

struct Scratch {
    cudaStream_t st;
    void* ptrs[16];
    int count = 0;
    explicit Scratch(cudaStream_t s) : st(s) {}
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    template <typename T>
    cudaError_t alloc(T** p, size_t elems) {
        if (count >= 16) return cudaErrorMemoryAllocation;
        cudaError_t e = isoc_malloc_async((void**)p, (elems ? elems : 1) * sizeof(T), st);
        if (e == cudaSuccess) ptrs[count++] = *p;
        return e;
    }
    ~Scratch() {
        for (int i = 0; i < count; ++i) isoc_free_async(ptrs[i], st);
    }
};

}  // namespace isoc
