// Does __syncthreads() wait for thread 0 while it spins on an acquire load?  Plain vs cooperative launch.
#include <cstdio>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ unsigned ld_acq(const unsigned *p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__global__ void __launch_bounds__(256) k(unsigned *flag, unsigned *bad) {
    __shared__ unsigned bcast;
    if (threadIdx.x == 0) bcast = 0;
    __syncthreads();
    if (blockIdx.x == 0) {
        if (threadIdx.x == 0) {
            unsigned long long t0 = gt();
            while (gt() - t0 < 20000) __nanosleep(64);
            atomicExch(flag, 1u);
        }
        return;
    }
    if (threadIdx.x == 0) {
        for (;;) { if (ld_acq(flag)) break; __nanosleep(64); }
        bcast = 1;
    }
    __syncthreads();
    if (bcast == 0) atomicAdd(bad, 1u);
}
int main() {
    unsigned *b; cudaMalloc(&b, 8);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(b, 0, 8);
        if (mode == 0) k<<<8, 256>>>(b, b + 1);
        else {
            cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(8); cfg.blockDim = dim3(256);
            cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeCooperative; a[0].val.cooperative = 1;
            cfg.attrs = a; cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k, b, b + 1);
        }
        unsigned h[2] = {0, 0}; cudaMemcpy(h, b, 8, cudaMemcpyDeviceToHost);
        printf("%s launch: threads that passed the barrier early: %u of %d (err %s)\n", mode ? "cooperative" : "plain", h[1], 7 * 256, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
