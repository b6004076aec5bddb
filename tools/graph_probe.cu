#include <cstdio>
struct P { int a[64]; int *out; };
__global__ void k(P p) { if (threadIdx.x == 0 && blockIdx.x == 0) *p.out = p.a[0]; }
#define C(x) do { cudaError_t e = (x); if (e) printf("%s -> %s\n", #x, cudaGetErrorString(e)); } while (0)
int main() {
    int *d; cudaMalloc(&d, 4);
    cudaStream_t cs; cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int coop = 0; coop < 2; ++coop) for (int evs = 0; evs < 2; ++evs) {
        P p = {}; p.a[0] = 7; p.out = d;
        void *args[] = {&p};
        C(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        if (evs) C(cudaEventRecordWithFlags(e0, cs, cudaEventRecordExternal));
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(148); cfg.blockDim = dim3(256); cfg.stream = cs;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
        cfg.attrs = at; cfg.numAttrs = coop;
        C(cudaLaunchKernelExC(&cfg, (void *)k, args));
        if (evs) C(cudaEventRecordWithFlags(e1, cs, cudaEventRecordExternal));
        cudaGraph_t g; C(cudaStreamEndCapture(cs, &g));
        size_t n = 0; C(cudaGraphGetNodes(g, nullptr, &n)); cudaGraphNode_t nodes[8]; C(cudaGraphGetNodes(g, nodes, &n));
        cudaGraphNode_t kn = nullptr;
        for (size_t i = 0; i < n; ++i) { cudaGraphNodeType t; cudaGraphNodeGetType(nodes[i], &t); if (t == cudaGraphNodeTypeKernel) kn = nodes[i]; }
        cudaGraphExec_t ex; C(cudaGraphInstantiate(&ex, g, 0));
        p.a[0] = 42;
        cudaKernelNodeParams kp = {}; kp.func = (void *)k; kp.gridDim = dim3(148); kp.blockDim = dim3(256); kp.kernelParams = args;
        cudaError_t e = cudaGraphExecKernelNodeSetParams(ex, kn, &kp);
        C(cudaGraphLaunch(ex, 0)); C(cudaDeviceSynchronize());
        int h = 0; cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
        printf("coop %d events %d nodes %zu: setparams %s, result %d (want 42)\n", coop, evs, n, cudaGetErrorString(e), h);
    }
}
