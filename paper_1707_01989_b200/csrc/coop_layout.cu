// coop_layout.cu -- graph-layout step for the bottom-up BFS levels (coop_csr_hub_first).
//
// Each neighbour list is reordered by descending neighbour degree, so a bottom-up
// candidate probes the hubs first: in an R-MAT graph the frontier of a dense level
// is mostly hubs, and a candidate with a frontier neighbour then finds it on the
// first probe instead of after a walk (537 -> 458 us mean kernel time
// on RMAT-24 in tools/hubfirst_probe.py).  Levels are unique, so results do not
// depend on the order.  Done once per graph, like building the CSR.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>

#include <cub/device/device_segmented_sort.cuh>

#include "../../include/coop.h"

char *coop_internal_errbuf();

namespace {

coop_status lfail(coop_status s, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(coop_internal_errbuf(), 512, fmt, ap);
    va_end(ap);
    return s;
}

// key[e] = degree of the neighbour col[e]
template <typename OffT>
__global__ void neighbour_degree_kernel(const OffT *ro, const int32_t *col, int64_t E, uint32_t *key) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = __ldg(col + e);
        key[e] = (uint32_t)(__ldg(ro + v + 1) - __ldg(ro + v));
    }
}

template <typename OffT>
cudaError_t hub_first(const OffT *ro, const int32_t *col, int64_t V, int64_t E, int32_t *col_out, cudaStream_t s) {
    uint32_t *keys = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    cudaError_t e = cudaMallocAsync(&keys, sizeof(uint32_t) * 2 * (size_t)E, s);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    neighbour_degree_kernel<<<sms * 8, 256, 0, s>>>(ro, col, E, keys);
    e = cudaGetLastError();
    if (e == cudaSuccess)
        e = cub::DeviceSegmentedSort::SortPairsDescending(nullptr, tmp_bytes, keys, keys + E, col, col_out, (int)E,
                                                          (int)V, ro, ro + 1, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&tmp, tmp_bytes ? tmp_bytes : 1, s);
    if (e == cudaSuccess)
        e = cub::DeviceSegmentedSort::SortPairsDescending(tmp, tmp_bytes, keys, keys + E, col, col_out, (int)E,
                                                          (int)V, ro, ro + 1, s);
    cudaFreeAsync(tmp, s);
    cudaFreeAsync(keys, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return e;
}

}  // namespace

extern "C" coop_status coop_csr_hub_first(const coop_csr *g, int32_t *col_out, void *stream) {
    if (!g || !col_out || !g->row_offsets || (!g->col_idx && g->num_edges > 0))
        return lfail(COOP_ERR_INVALID_ARG, "NULL graph / output");
    if (g->num_vertices < 1 || g->num_vertices > (int64_t)INT32_MAX) return lfail(COOP_ERR_INVALID_ARG, "bad V");
    if (g->num_edges < 0 || g->num_edges > (int64_t)INT32_MAX - 1)
        return lfail(COOP_ERR_INVALID_ARG, "num_edges %lld: the segmented sort takes < 2^31 entries",
                     (long long)g->num_edges);
    if (g->offset_bits != 32 && g->offset_bits != 64) return lfail(COOP_ERR_INVALID_ARG, "offset_bits must be 32 or 64");
    if (g->num_edges == 0) return COOP_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    if (g->offset_bits == 32)
        e = hub_first(static_cast<const uint32_t *>(g->row_offsets), g->col_idx, g->num_vertices, g->num_edges,
                      col_out, s);
    else
        e = hub_first(static_cast<const long long *>(g->row_offsets), g->col_idx, g->num_vertices, g->num_edges,
                      col_out, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return lfail(COOP_ERR_CUDA, "coop_csr_hub_first: %s", cudaGetErrorString(e));
    }
    return COOP_OK;
}
