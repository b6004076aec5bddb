/*
 * oracle/textbook.c -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * O1 of SURVEY.md §8(c): the plain definitions the cooperative kernels must
 * reproduce bit-exactly, written as the textbook algorithms.
 *
 *   oracle_bfs      -- FIFO-queue breadth-first search.  level[v] = minimum hop
 *                      count from the source, -1 if unreachable.  This is what
 *                      Fig. 4's frontier loop computes (PAPER.md:709-729,
 *                      "level" counter P:712/P:723); SPEC.md:357 names the
 *                      "textbook queue-based BFS" as the oracle.
 *   oracle_dijkstra -- binary-heap Dijkstra with lazy deletion.  dist[v] =
 *                      minimum over s->v paths of the sum of uint32 weights,
 *                      0xFFFFFFFF if unreachable.  This is the fixpoint the
 *                      worklist SSSP ("l-sssp", Table 1) converges to;
 *                      the paper gives no SSSP text (SURVEY §8(c) reading 8).
 *
 * No blocking, fusion or reordering: one queue / one heap, one thread.
 * Shares no code with the CUDA path.  Returns 0 on success, -1 on bad
 * arguments, -2 on allocation failure.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int oracle_bfs(int64_t V, const int64_t *row_offsets, const int32_t *col_idx,
               int64_t source, int32_t *level_out)
{
    if (V <= 0 || source < 0 || source >= V) return -1;
    for (int64_t v = 0; v < V; ++v) level_out[v] = -1;
    int64_t *queue = (int64_t *)malloc(sizeof(int64_t) * (size_t)V);
    if (!queue) return -2;
    int64_t head = 0, tail = 0;
    level_out[source] = 0;
    queue[tail++] = source;
    while (head < tail) {
        int64_t u = queue[head++];
        for (int64_t e = row_offsets[u]; e < row_offsets[u + 1]; ++e) {
            int64_t w = col_idx[e];
            if (level_out[w] == -1) {
                level_out[w] = level_out[u] + 1;
                queue[tail++] = w;
            }
        }
    }
    free(queue);
    return 0;
}

/* ---- binary min-heap of (dist, vertex) pairs, lazy deletion ---- */
typedef struct { uint64_t d; int64_t v; } item_t;

static void heap_push(item_t *h, int64_t *n, item_t x)
{
    int64_t i = (*n)++;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (h[p].d <= x.d) break;
        h[i] = h[p];
        i = p;
    }
    h[i] = x;
}

static item_t heap_pop(item_t *h, int64_t *n)
{
    item_t top = h[0];
    item_t last = h[--(*n)];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        uint64_t md = last.d;
        if (l < *n && h[l].d < md) { m = l; md = h[l].d; }
        if (r < *n && h[r].d < md) { m = r; }
        if (m == i) break;
        h[i] = h[m];
        i = m;
    }
    if (*n > 0) h[i] = last;
    return top;
}

int oracle_dijkstra(int64_t V, const int64_t *row_offsets, const int32_t *col_idx,
                    const uint32_t *weights, int64_t source, uint32_t *dist_out)
{
    if (V <= 0 || source < 0 || source >= V) return -1;
    int64_t E = row_offsets[V];
    /* 64-bit tentative distances so that no sum can wrap inside the oracle */
    uint64_t *dist = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)V);
    unsigned char *done = (unsigned char *)calloc((size_t)V, 1);
    item_t *heap = (item_t *)malloc(sizeof(item_t) * (size_t)(E + 1));
    if (!dist || !done || !heap) { free(dist); free(done); free(heap); return -2; }
    const uint64_t INF = UINT64_MAX;
    for (int64_t v = 0; v < V; ++v) dist[v] = INF;
    int64_t n = 0;
    dist[source] = 0;
    heap_push(heap, &n, (item_t){0, source});
    while (n > 0) {
        item_t it = heap_pop(heap, &n);
        if (done[it.v]) continue;
        done[it.v] = 1;
        for (int64_t e = row_offsets[it.v]; e < row_offsets[it.v + 1]; ++e) {
            int64_t w = col_idx[e];
            uint64_t nd = it.d + (uint64_t)weights[e];
            if (nd < dist[w]) {
                dist[w] = nd;
                heap_push(heap, &n, (item_t){nd, w});
            }
        }
    }
    int rc = 0;
    for (int64_t v = 0; v < V; ++v) {
        if (dist[v] == INF) dist_out[v] = 0xFFFFFFFFu;
        else if (dist[v] >= 0xFFFFFFFFull) { dist_out[v] = 0xFFFFFFFFu; rc = -3; } /* not representable */
        else dist_out[v] = (uint32_t)dist[v];
    }
    free(dist); free(done); free(heap);
    return rc;
}
