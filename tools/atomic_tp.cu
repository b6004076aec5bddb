// atomic_tp.cu -- throughput of contended global atomics on B200: every warp
// of a 296 x 512 grid (the BFS launch shape) issues R atomics from lane 0 to
// one shared address (or to one line per warp), with and without a return
// value.  Tells how many same-address atomics a BFS level can afford.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/atomic_tp tools/atomic_tp.cu && /tmp/atomic_tp
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <bool RET, bool SPREAD>
__global__ void k(unsigned long long *w, unsigned long long *sink, int R) {
    if ((threadIdx.x & 31) != 0) return;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    unsigned long long *a = SPREAD ? w + (size_t)gw * 16 : w;
    unsigned long long v = 0;
    for (int i = 0; i < R; ++i) {
        if (RET) v += atomicAdd(a + (v >> 63), 1ull);
        else atomicAdd(a, 1ull);
    }
    if (RET && v == 42) sink[0] = v;
}

template <bool RET, bool SPREAD>
void run(const char *name, unsigned long long *w, unsigned long long *sink, int R) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<RET, SPREAD><<<296, 512>>>(w, sink, R);
    cudaEventRecord(e0);
    k<RET, SPREAD><<<296, 512>>>(w, sink, R);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double n = 296.0 * 16 * R;
    printf("%-28s R=%3d  %9.1f us  %7.3f ns/atomic  (%.0f atomics)\n", name, R, ms * 1e3, ms * 1e6 / n, n);
}

int main() {
    unsigned long long *w, *sink;
    cudaMalloc(&w, 296 * 16 * 16 * 8);
    cudaMalloc(&sink, 8);
    cudaMemset(w, 0, 296 * 16 * 16 * 8);
    for (int R : {1, 4, 16}) {
        run<true, false>("atom same address", w, sink, R);
        run<false, false>("red same address", w, sink, R);
        run<true, true>("atom line per warp", w, sink, R);
        run<false, true>("red line per warp", w, sink, R);
    }
    return 0;
}
