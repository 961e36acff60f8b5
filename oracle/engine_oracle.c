/*
 * TEST INFRASTRUCTURE ONLY -- C restatement of the reference engine.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg load
 * this library (oracle/build/libdfsim_oracle.so); the product never does.
 *
 * Restates, on rank-ordered CSR arrays (node index == rank of the id string,
 * device index == rank of the device string):
 *   oracle_simulate      engine.py:96-146 (heap of (finish, id, dev), per-device
 *                        FIFO, exact == batching) and _finalize 69-93
 *                        (entries sorted by (start, device, id); busy summed in
 *                        entry order; makespan = max finish)
 *   oracle_critical_path graph.py:424-485 (Kahn with an id heap, suffix DP,
 *                        min-id source among the max, greedy min-id walk)
 * Compiled with -ffp-contract=off so a*b+c is never fused.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef struct { double t; int32_t node; int32_t dev; } ev_t;

static int ev_less(const ev_t *a, const ev_t *b) {
    /* heap tuple order (finish, node id, device) -- engine.py:125 */
    if (a->t != b->t) return a->t < b->t;
    if (a->node != b->node) return a->node < b->node;
    return a->dev < b->dev;
}

static void ev_push(ev_t *h, int *n, ev_t e) {
    int i = (*n)++;
    h[i] = e;
    while (i > 0) {
        int p = (i - 1) / 2;
        if (!ev_less(&h[i], &h[p])) break;
        ev_t t = h[i]; h[i] = h[p]; h[p] = t; i = p;
    }
}

static ev_t ev_pop(ev_t *h, int *n) {
    ev_t top = h[0];
    h[0] = h[--(*n)];
    int i = 0;
    for (;;) {
        int l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && ev_less(&h[l], &h[m])) m = l;
        if (r < *n && ev_less(&h[r], &h[m])) m = r;
        if (m == i) break;
        ev_t t = h[i]; h[i] = h[m]; h[m] = t; i = m;
    }
    return top;
}

static int cmp_int(const void *a, const void *b) {
    int x = *(const int *)a, y = *(const int *)b;
    return (x > y) - (x < y);
}

/*
 * Returns 0 on success, 1 if some node was never placed (CycleError); in that
 * case start[v] is NaN for unplaced nodes.  entry_order (optional) receives the
 * node ranks in Schedule.entries order.
 */
int oracle_simulate(int32_t n, int32_t n_dev, const int32_t *succ_off, const int32_t *succ_idx,
                    const int32_t *indeg, const int32_t *dev, const double *dur,
                    double *start, double *finish, double *busy, double *makespan,
                    int32_t *entry_order, int32_t *n_placed_out) {
    int32_t *cnt = malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t *qbuf = malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t *qoff = calloc((size_t)n_dev + 1, sizeof(int32_t));
    int32_t *qhead = malloc(sizeof(int32_t) * (size_t)(n_dev + 1));
    int32_t *qtail = malloc(sizeof(int32_t) * (size_t)(n_dev + 1));
    int32_t *run = malloc(sizeof(int32_t) * (size_t)(n_dev + 1));
    double *devfree = malloc(sizeof(double) * (size_t)(n_dev + 1));
    double *ready = malloc(sizeof(double) * (size_t)(n + 1));
    int32_t *fresh = malloc(sizeof(int32_t) * (size_t)(n + 1));
    ev_t *heap = malloc(sizeof(ev_t) * (size_t)(n_dev + 1));
    int nheap = 0, nplaced = 0, nfresh = 0;

    for (int32_t v = 0; v < n; v++) { cnt[v] = indeg[v]; qoff[dev[v] + 1]++; start[v] = 0.0 / 0.0; finish[v] = 0.0 / 0.0; }
    for (int32_t d = 0; d < n_dev; d++) { qoff[d + 1] += qoff[d]; qhead[d] = qtail[d] = qoff[d]; run[d] = -1; devfree[d] = 0.0; }

    /* sources in id order (enqueue sorts, engine.py:112) */
    for (int32_t v = 0; v < n; v++)
        if (cnt[v] == 0) { ready[v] = 0.0; qbuf[qtail[dev[v]]++] = v; }

#define START_IDLE()                                                                  \
    for (int32_t d = 0; d < n_dev; d++) {                                             \
        if (run[d] >= 0 || qhead[d] == qtail[d]) continue;                            \
        int32_t v = qbuf[qhead[d]++];                                                 \
        double s = devfree[d] > ready[v] ? devfree[d] : ready[v];                     \
        double f = s + dur[v];                                                        \
        start[v] = s; finish[v] = f; nplaced++;                                       \
        run[d] = v;                                                                   \
        ev_t e = {f, v, d};                                                           \
        ev_push(heap, &nheap, e);                                                     \
    }

    START_IDLE();
    while (nheap > 0) {
        double now = heap[0].t;
        nfresh = 0;
        while (nheap > 0 && heap[0].t == now) {
            ev_t e = ev_pop(heap, &nheap);
            run[e.dev] = -1;
            devfree[e.dev] = now;
            for (int32_t j = succ_off[e.node]; j < succ_off[e.node + 1]; j++) {
                int32_t m = succ_idx[j];
                if (--cnt[m] == 0) fresh[nfresh++] = m;
            }
        }
        qsort(fresh, (size_t)nfresh, sizeof(int32_t), cmp_int);
        for (int i = 0; i < nfresh; i++) { ready[fresh[i]] = now; qbuf[qtail[dev[fresh[i]]]++] = fresh[i]; }
        START_IDLE();
    }
#undef START_IDLE

    int status = nplaced == n ? 0 : 1;
    if (n_placed_out) *n_placed_out = nplaced;
    double ms = 0.0;
    for (int32_t d = 0; d < n_dev; d++) busy[d] = 0.0;
    if (status == 0) {
        /* Schedule.entries order: (start, device, id) -- engine.py:88 */
        int32_t *ord = entry_order ? entry_order : fresh;
        for (int32_t v = 0; v < n; v++) ord[v] = v;
        /* bottom-up merge sort keyed by (start, dev, id) */
        int32_t *tmp = malloc(sizeof(int32_t) * (size_t)(n + 1));
        for (int32_t width = 1; width < n; width *= 2) {
            for (int32_t lo = 0; lo < n; lo += 2 * width) {
                int32_t mid = lo + width < n ? lo + width : n, hi = lo + 2 * width < n ? lo + 2 * width : n;
                int32_t i = lo, j = mid, k = lo;
                while (i < mid && j < hi) {
                    int32_t a = ord[i], b = ord[j];
                    int take_b = start[b] < start[a] || (start[b] == start[a] && (dev[b] < dev[a] || (dev[b] == dev[a] && b < a)));
                    tmp[k++] = take_b ? ord[j++] : ord[i++];
                }
                while (i < mid) tmp[k++] = ord[i++];
                while (j < hi) tmp[k++] = ord[j++];
            }
            memcpy(ord, tmp, sizeof(int32_t) * (size_t)n);
        }
        for (int32_t i = 0; i < n; i++) {
            int32_t v = ord[i];
            busy[dev[v]] = busy[dev[v]] + (finish[v] - start[v]);
            if (finish[v] > ms) ms = finish[v];
        }
        free(tmp);
    }
    *makespan = ms;
    free(cnt); free(qbuf); free(qoff); free(qhead); free(qtail); free(run); free(devfree);
    free(ready); free(fresh); free(heap);
    return status;
}

/* min-heap of node ranks for Kahn's order (graph.py:430-439) */
static void ih_push(int32_t *h, int *n, int32_t x) {
    int i = (*n)++;
    h[i] = x;
    while (i > 0) { int p = (i - 1) / 2; if (h[p] <= h[i]) break; int32_t t = h[i]; h[i] = h[p]; h[p] = t; i = p; }
}
static int32_t ih_pop(int32_t *h, int *n) {
    int32_t top = h[0];
    h[0] = h[--(*n)];
    int i = 0;
    for (;;) {
        int l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && h[l] < h[m]) m = l;
        if (r < *n && h[r] < h[m]) m = r;
        if (m == i) break;
        int32_t t = h[i]; h[i] = h[m]; h[m] = t; i = m;
    }
    return top;
}

/* Returns 0, or 1 on a cycle.  path must hold n entries. */
int oracle_critical_path(int32_t n, const int32_t *succ_off, const int32_t *succ_idx, const int32_t *indeg,
                         const double *d, double *length, int32_t *path, int32_t *path_len) {
    if (n == 0) { *length = 0.0; *path_len = 0; return 0; }
    int32_t *left = malloc(sizeof(int32_t) * (size_t)n);
    int32_t *order = malloc(sizeof(int32_t) * (size_t)n);
    int32_t *heap = malloc(sizeof(int32_t) * (size_t)n);
    double *suffix = malloc(sizeof(double) * (size_t)n);
    int nh = 0, no = 0;
    for (int32_t v = 0; v < n; v++) { left[v] = indeg[v]; if (left[v] == 0) ih_push(heap, &nh, v); }
    while (nh > 0) {
        int32_t v = ih_pop(heap, &nh);
        order[no++] = v;
        for (int32_t j = succ_off[v]; j < succ_off[v + 1]; j++)
            if (--left[succ_idx[j]] == 0) ih_push(heap, &nh, succ_idx[j]);
    }
    int status = 0;
    if (no != n) { status = 1; goto done; }
    for (int i = n - 1; i >= 0; i--) {
        int32_t v = order[i];
        double best = 0.0;
        for (int32_t j = succ_off[v]; j < succ_off[v + 1]; j++)
            if (suffix[succ_idx[j]] > best) best = suffix[succ_idx[j]];
        suffix[v] = d[v] + best;
    }
    double len = 0.0; int32_t src = -1;
    for (int i = 0; i < n; i++) {
        int32_t v = order[i];
        if (indeg[v] != 0) continue;
        if (src < 0 || suffix[v] > len) { len = suffix[v]; src = v; }
    }
    for (int32_t v = 0; v < n; v++)  /* min id among sources achieving the max */
        if (indeg[v] == 0 && suffix[v] == len) { src = v; break; }
    *length = len;
    int32_t k = 0, v = src;
    path[k++] = v;
    while (succ_off[v + 1] > succ_off[v]) {
        double top = suffix[succ_idx[succ_off[v]]];
        for (int32_t j = succ_off[v]; j < succ_off[v + 1]; j++) if (suffix[succ_idx[j]] > top) top = suffix[succ_idx[j]];
        int32_t nxt = -1;
        for (int32_t j = succ_off[v]; j < succ_off[v + 1]; j++)
            if (suffix[succ_idx[j]] == top) { nxt = succ_idx[j]; break; }  /* successors sorted by id */
        v = nxt;
        path[k++] = v;
    }
    *path_len = k;
done:
    free(left); free(order); free(heap); free(suffix);
    return status;
}

/* Batch driver for the CPU baseline and the full-grid parity tests: S independent
 * simulations + CP lengths, spread over n_threads pthreads (each owns a contiguous slice of
 * sims).  Optional outputs (NULL: not written): start/finish [S][n], busy [S][n_dev],
 * cp_src [S] (rank of the critical path's first node). */
typedef struct {
    int32_t n, n_dev; const int32_t *succ_off, *succ_idx, *indeg, *dev;
    int64_t s0, s1; const double *dur; double *makespan, *cp_len;
    double *start_out, *finish_out, *busy_out; int32_t *cp_src; int status;
} batch_arg_t;

static void *batch_worker(void *p) {
    batch_arg_t *a = p;
    int32_t n = a->n;
    double *st = malloc(sizeof(double) * (size_t)(n + 1));
    double *fi = malloc(sizeof(double) * (size_t)(n + 1));
    double *busy = malloc(sizeof(double) * (size_t)(a->n_dev + 1));
    int32_t *path = malloc(sizeof(int32_t) * (size_t)(n + 1));
    for (int64_t s = a->s0; s < a->s1; s++) {
        int32_t np = 0, pl = 0;
        int rc = oracle_simulate(n, a->n_dev, a->succ_off, a->succ_idx, a->indeg, a->dev,
                                 a->dur + (size_t)s * (size_t)n, st, fi, busy, &a->makespan[s], NULL, &np);
        if (a->start_out) memcpy(a->start_out + (size_t)s * (size_t)n, st, sizeof(double) * (size_t)n);
        if (a->finish_out) memcpy(a->finish_out + (size_t)s * (size_t)n, fi, sizeof(double) * (size_t)n);
        if (a->busy_out) memcpy(a->busy_out + (size_t)s * (size_t)a->n_dev, busy, sizeof(double) * (size_t)a->n_dev);
        a->cp_len[s] = 0.0;
        if (a->cp_src) a->cp_src[s] = -1;
        if (rc == 0) {
            for (int32_t v = 0; v < n; v++) fi[v] = fi[v] - st[v];
            rc = oracle_critical_path(n, a->succ_off, a->succ_idx, a->indeg, fi, &a->cp_len[s], path, &pl);
            if (a->cp_src && pl > 0) a->cp_src[s] = path[0];
        }
        a->status |= rc;
    }
    free(st); free(fi); free(busy); free(path);
    return NULL;
}

int oracle_simulate_batch_full(int32_t n, int32_t n_dev, const int32_t *succ_off, const int32_t *succ_idx,
                               const int32_t *indeg, const int32_t *dev, int64_t n_sims, const double *dur,
                               double *makespan, double *cp_len, double *start_out, double *finish_out,
                               double *busy_out, int32_t *cp_src, int32_t n_threads) {
    if (n_threads < 1) n_threads = 1;
    pthread_t tid[256];
    batch_arg_t arg[256];
    if (n_threads > 256) n_threads = 256;
    int status = 0;
    for (int t = 0; t < n_threads; t++) {
        arg[t] = (batch_arg_t){n, n_dev, succ_off, succ_idx, indeg, dev,
                               n_sims * t / n_threads, n_sims * (t + 1) / n_threads, dur, makespan, cp_len,
                               start_out, finish_out, busy_out, cp_src, 0};
        pthread_create(&tid[t], NULL, batch_worker, &arg[t]);
    }
    for (int t = 0; t < n_threads; t++) { pthread_join(tid[t], NULL); status |= arg[t].status; }
    return status;
}

int oracle_simulate_batch(int32_t n, int32_t n_dev, const int32_t *succ_off, const int32_t *succ_idx,
                          const int32_t *indeg, const int32_t *dev, int64_t n_sims, const double *dur,
                          double *makespan, double *cp_len, int32_t n_threads) {
    return oracle_simulate_batch_full(n, n_dev, succ_off, succ_idx, indeg, dev, n_sims, dur, makespan, cp_len,
                                      NULL, NULL, NULL, NULL, n_threads);
}
