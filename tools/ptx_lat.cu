// ptx_lat.cu -- single-thread latency of the memory-ordering primitives the
// resizing barrier is built from (clock64 cycles and ns via %globaltimer),
// measured on the GPU box:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 \
//   -o /tmp/ptx_lat tools/ptx_lat.cu && /tmp/ptx_lat
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

#define BODY(NAME, STMT)                                                        \
    {                                                                           \
        unsigned long long v = 0;                                               \
        long long c0 = clock64();                                               \
        uint64_t t0 = gt();                                                     \
        for (int i = 0; i < n; ++i) { STMT; }                                   \
        long long c1 = clock64();                                               \
        uint64_t t1 = gt();                                                     \
        sink[0] += v;                                                           \
        if (threadIdx.x == 0) printf("%-34s %8.1f cyc %8.1f ns\n", NAME, (double)(c1 - c0) / n, (double)(t1 - t0) / n); \
    }

__global__ void lat(unsigned long long *w, unsigned long long *sink, int n) {
    BODY("globaltimer read", v += gt())
    BODY("atom.relaxed add (dependent)", v = atomicAdd(w + (v >> 63), 1ull))
    BODY("atom.acq_rel.gpu add (dependent)", asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(v) : "l"(w + (v >> 63)) : "memory"))
    BODY("ld.acquire.gpu (dependent)", asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(w + 8 + (v >> 63)) : "memory"))
    BODY("ld.relaxed.gpu (dependent)", asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(w + 8 + (v >> 63)) : "memory"))
    BODY("fence.sc.gpu (__threadfence)", __threadfence())
    BODY("fence.acq_rel.gpu", asm volatile("fence.acq_rel.gpu;" ::: "memory"))
    BODY("st.relaxed + fence.sc", { w[16] = v + i; __threadfence(); })
    BODY("st.release.gpu", asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(w + 24), "l"((unsigned long long)i) : "memory"))
    BODY("st.release + ld.acquire same addr", { asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(w + 24), "l"((unsigned long long)i) : "memory"); asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(w + 24) : "memory"); })
    BODY("__syncthreads (1 warp)", __syncthreads())
}

int main() {
    unsigned long long *w, *sink;
    cudaMalloc(&w, 4096);
    cudaMalloc(&sink, 64);
    cudaMemset(w, 0, 4096);
    lat<<<1, 1>>>(w, sink, 2000);
    cudaDeviceSynchronize();
    lat<<<1, 1>>>(w, sink, 20000);
    cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
