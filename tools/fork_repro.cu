// Minimal reproduction: do all warps of a forked CTA run the body?
#include <cstdio>
#include <vector>

#include "coop_device.cuh"
#include "coop.h"

__global__ void __launch_bounds__(256) k(coop_dev *d, unsigned *cnt) {
    coop_run(d, [&](coop_ctx *c) {
        unsigned t = 0;
        if (coop_entry(c) == 0) {
            if (!coop_resizing_global_barrier(c, &t, sizeof t, 1)) return;
        }
        atomicAdd(&cnt[blockIdx.x], 1u);
        if (!coop_resizing_global_barrier(c, &t, sizeof t, 2)) return;
    });
}
int main() {
    unsigned *cnt; cudaMalloc(&cnt, 4096 * 4);
    for (int N : {8, 48, 148}) {
        std::vector<uint32_t> script = {(uint32_t)N};
        coop_dev_opts o = {};
        o.max_wgs = N; o.init_wgs = 1; o.policy = COOP_POLICY_SCRIPTED; o.script = script.data(); o.script_len = 1;
        coop_dev_handle *h; coop_dev_create(&o, &h);
        int bad = 0;
        for (int it = 0; it < 20; ++it) {
            cudaMemset(cnt, 0, 4096 * 4);
            coop_dev *dp; coop_dev_arm(h, N, 0, &dp);
            cudaError_t e = coop_dev_launch(k, N, 256, 0, 0, dp, cnt);
            coop_dev_stats st = {};
            int rc = coop_dev_collect(h, 0, &st);
            std::vector<unsigned> hc(N); cudaMemcpy(hc.data(), cnt, N * 4, cudaMemcpyDeviceToHost);
            for (int b = 0; b < N; ++b) if (hc[b] != 256) { ++bad; if (bad < 4) printf("N %d it %d cta %d count %u (rc %d e %d forks %u)\n", N, it, b, hc[b], rc, (int)e, st.forks); }
        }
        printf("N %d: bad CTAs %d\n", N, bad);
        coop_dev_destroy(h);
    }
}
