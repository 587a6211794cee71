/*
 * mfx_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference `dynmaxflow`
 * algorithms on the hot path, used as the parity checker for the CUDA engine
 * (tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg only).
 * Nothing in the product package links or calls this file.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/pkg/src/dynmaxflow/).  Arrays use the
 * reference's int64 layout so results compare byte-for-byte with the
 * reference's numpy arrays.  Parity is pinned against fixtures produced by
 * the live reference (tests/golden/make_golden.py).
 *
 * Concurrency: the reference runs push/repair phases on a thread pool with
 * relaxed atomics; this restatement runs them sequentially in worklist order,
 * which is the reference's `deterministic=True` schedule (solver.py:56-58,
 * 70-73).  Flow values are schedule independent (unique max-flow value).
 */
#define _POSIX_C_SOURCE 199309L
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* Wall-clock cap for bounded CPU-baseline samples (bench.py cpu_baseline):
 * push_rounds stops at a round boundary once it is past, and the solve
 * reports status 5 ("capped") with the rounds it completed.  0 = no cap. */
static double g_deadline = 0.0;

static double now_s(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

void orc_set_time_cap(double seconds) { g_deadline = seconds > 0 ? now_s() + seconds : 0.0; }

/* ------------------------------------------------------------------ */
/* radix sort of (uint64 key, int64 payload) pairs, LSD, 16-bit digits  */
/* ------------------------------------------------------------------ */
static void radix_sort_pairs(uint64_t *key, int64_t *val, int64_t cnt)
{
    if (cnt <= 1) return;
    uint64_t *k2 = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)cnt);
    int64_t *v2 = (int64_t *)malloc(sizeof(int64_t) * (size_t)cnt);
    int64_t *hist = (int64_t *)malloc(sizeof(int64_t) * 65536);
    uint64_t all_or = 0, all_and = ~(uint64_t)0;
    for (int64_t i = 0; i < cnt; i++) { all_or |= key[i]; all_and &= key[i]; }
    for (int pass = 0; pass < 4; pass++) {
        int sh = pass * 16;
        /* skip a pass whose digit is identical for every key */
        if ((((all_or ^ all_and) >> sh) & 0xFFFF) == 0) continue;
        memset(hist, 0, sizeof(int64_t) * 65536);
        for (int64_t i = 0; i < cnt; i++) hist[(key[i] >> sh) & 0xFFFF]++;
        int64_t acc = 0;
        for (int d = 0; d < 65536; d++) { int64_t c = hist[d]; hist[d] = acc; acc += c; }
        for (int64_t i = 0; i < cnt; i++) {
            int64_t p = hist[(key[i] >> sh) & 0xFFFF]++;
            k2[p] = key[i]; v2[p] = val[i];
        }
        memcpy(key, k2, sizeof(uint64_t) * (size_t)cnt);
        memcpy(val, v2, sizeof(int64_t) * (size_t)cnt);
    }
    free(k2); free(v2); free(hist);
}

/* ------------------------------------------------------------------ */
/* graph build                                                          */
/* ------------------------------------------------------------------ */

/* EdgeListGraph.validate, graph.py:48-61.  Returns 0, or an error code with
 * err_index = offending edge: -1 n<=0, -2 source out of range,
 * -3 target out of range, -4 negative capacity. */
int orc_validate_edges(int64_t n, int64_t m, const int64_t *us, const int64_t *vs,
                       const int64_t *caps, int64_t *err_index)
{
    *err_index = -1;
    if (n <= 0) return -1;
    for (int64_t i = 0; i < m; i++)
        if (us[i] < 0 || us[i] >= n) { *err_index = i; return -2; }
    for (int64_t i = 0; i < m; i++)
        if (vs[i] < 0 || vs[i] >= n) { *err_index = i; return -3; }
    for (int64_t i = 0; i < m; i++)
        if (caps[i] < 0) { *err_index = i; return -4; }
    return 0;
}

/* build_bicsr, graph.py:126-174.  Output arrays are caller-allocated with
 * capacity 2*m slots (offsets: n+1).  Returns the slot count S >= 0, or a
 * negative orc_validate_edges code.  diag = {self_loops_dropped,
 * parallel_edges_merged, reverse_stubs_added} (graph.py:64-68). */
int64_t orc_build_bicsr(int64_t n, int64_t m, const int64_t *us, const int64_t *vs,
                        const int64_t *caps, int64_t *offsets, int64_t *adj,
                        int64_t *src, int64_t *rev, int64_t *cap0, uint8_t *is_original,
                        int64_t *diag, int64_t *err_index)
{
    int rc = orc_validate_edges(n, m, us, vs, caps, err_index);
    if (rc) return rc;
    uint64_t N = (uint64_t)n;
    /* drop self-loops (graph.py:138-140) */
    uint64_t *key = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(2 * m + 1));
    int64_t *val = (int64_t *)malloc(sizeof(int64_t) * (size_t)(2 * m + 1));
    int64_t kept = 0;
    for (int64_t i = 0; i < m; i++) {
        if (us[i] == vs[i]) continue;
        key[kept] = (uint64_t)us[i] * N + (uint64_t)vs[i];
        val[kept] = caps[i];
        kept++;
    }
    diag[0] = m - kept;
    /* merge parallel edges: unique keys, summed caps (graph.py:143-147) */
    radix_sort_pairs(key, val, kept);
    int64_t m1 = 0;
    for (int64_t i = 0; i < kept; i++) {
        if (m1 > 0 && key[m1 - 1] == key[i]) { val[m1 - 1] += val[i]; continue; }
        key[m1] = key[i]; val[m1] = val[i]; m1++;
    }
    diag[1] = kept - m1;
    /* symmetric closure with zero-cap candidates (graph.py:152-163).
     * payload = cap*2 + origin flag; each key has at most one original
     * contribution, so summing payloads sums caps and ORs the flag. */
    for (int64_t i = 0; i < m1; i++) {
        uint64_t u = key[i] / N, v = key[i] % N;
        key[m1 + i] = v * N + u;
        val[m1 + i] = 0;
        val[i] = val[i] * 2 + 1;
    }
    int64_t tot = 2 * m1;
    radix_sort_pairs(key, val, tot);
    int64_t S = 0;
    for (int64_t i = 0; i < tot; i++) {
        if (S > 0 && key[S - 1] == key[i]) { val[S - 1] += val[i]; continue; }
        key[S] = key[i]; val[S] = val[i]; S++;
    }
    diag[2] = S - m1;
    /* src/adj/offsets (graph.py:165-168) */
    for (int64_t v = 0; v <= n; v++) offsets[v] = 0;
    for (int64_t i = 0; i < S; i++) {
        src[i] = (int64_t)(key[i] / N);
        adj[i] = (int64_t)(key[i] % N);
        cap0[i] = val[i] >> 1;
        is_original[i] = (uint8_t)(val[i] & 1);
        offsets[src[i] + 1]++;
    }
    for (int64_t v = 0; v < n; v++) offsets[v + 1] += offsets[v];
    /* rev = searchsorted(skeys, adj*n+src) (graph.py:171) */
    for (int64_t i = 0; i < S; i++) {
        uint64_t want = (uint64_t)adj[i] * N + (uint64_t)src[i];
        int64_t lo = 0, hi = S;
        while (lo < hi) {
            int64_t mid = lo + (hi - lo) / 2;
            if (key[mid] < want) lo = mid + 1; else hi = mid;
        }
        rev[i] = lo;
    }
    free(key); free(val);
    return S;
}

/* ------------------------------------------------------------------ */
/* state primitives                                                     */
/* ------------------------------------------------------------------ */

/* saturate_source, state.py:42-59 */
void orc_saturate_source(int64_t s, const int64_t *offsets, const int64_t *adj,
                         const int64_t *rev, int64_t *cf, int64_t *excess)
{
    int64_t total = 0;
    for (int64_t i = offsets[s]; i < offsets[s + 1]; i++) {
        int64_t d = cf[i];
        cf[i] = 0;
        cf[rev[i]] += d;
        excess[adj[i]] += d;
        total += d;
    }
    excess[s] -= total;
}

/* _bfs_heights, kernels.py:168-215 (backward mode, no region masking).
 * Returns the number of reached vertices (queue tail). */
int64_t orc_bfs_heights(int64_t n, const int64_t *offsets, const int64_t *adj,
                        const int64_t *rev, const int64_t *cf, int64_t *height,
                        const int64_t *bases, int64_t nb, int64_t forbidden)
{
    int64_t *queue = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + nb + 1));
    for (int64_t v = 0; v < n; v++) height[v] = n;
    int64_t tail = 0;
    for (int64_t b = 0; b < nb; b++) { height[bases[b]] = 0; queue[tail++] = bases[b]; }
    if (forbidden >= 0) height[forbidden] = n;
    int64_t head = 0;
    while (head < tail) {
        int64_t u = queue[head++];
        int64_t du = height[u];
        for (int64_t i = offsets[u]; i < offsets[u + 1]; i++) {
            int64_t v = adj[i];
            if (v == forbidden || height[v] != n) continue;
            if (cf[rev[i]] > 0) { height[v] = du + 1; queue[tail++] = v; }
        }
    }
    free(queue);
    return tail;
}

/* _push_relabel_chunk, kernels.py:19-67, run over the whole worklist in
 * order.  Writes (pushes, relabels) into counts[0..1]. */
void orc_push_relabel(const int64_t *work, int64_t nw, const int64_t *offsets,
                      const int64_t *adj, const int64_t *rev, int64_t *cf,
                      int64_t *excess, int64_t *height, int64_t n,
                      int64_t kernel_cycles, int64_t *counts)
{
    int64_t pushes = 0, relabels = 0;
    for (int64_t w = 0; w < nw; w++) {
        int64_t u = work[w];
        for (int64_t cnt = 0; cnt < kernel_cycles; cnt++) {
            int64_t e = excess[u];
            if (e <= 0 || height[u] >= n) break;
            int64_t best_i = -1, best_h = n + 1;
            for (int64_t i = offsets[u]; i < offsets[u + 1]; i++) {
                if (cf[i] > 0) {
                    int64_t hv = height[adj[i]];
                    if (hv < best_h) { best_h = hv; best_i = i; }
                }
            }
            if (best_i < 0) { height[u] = n; relabels++; break; }
            if (height[u] > best_h) {
                int64_t d = e < cf[best_i] ? e : cf[best_i];
                cf[best_i] -= d;
                cf[rev[best_i]] += d;
                excess[u] -= d;
                excess[adj[best_i]] += d;
                pushes++;
            } else {
                int64_t nh = best_h + 1;
                height[u] = nh > n ? n : nh;
                relabels++;
            }
        }
    }
    counts[0] += pushes;
    counts[1] += relabels;
}

/* _remove_invalid_chunk, kernels.py:70-93.  Returns repairs. */
int64_t orc_remove_invalid(const int64_t *work, int64_t nw, const int64_t *offsets,
                           const int64_t *adj, const int64_t *rev, int64_t *cf,
                           int64_t *excess, const int64_t *height)
{
    int64_t repaired = 0;
    for (int64_t w = 0; w < nw; w++) {
        int64_t u = work[w];
        int64_t hu = height[u];
        for (int64_t i = offsets[u]; i < offsets[u + 1]; i++) {
            int64_t v = adj[i];
            if (cf[i] > 0 && hu > height[v] + 1) {
                int64_t amt = cf[i];
                cf[i] = 0;
                cf[rev[i]] += amt;
                excess[u] -= amt;
                excess[v] += amt;
                repaired++;
            }
        }
    }
    return repaired;
}

/* _recompute_excess, kernels.py:218-231 */
void orc_recompute_excess(int64_t n, const int64_t *offsets, const int64_t *rev,
                          const int64_t *cf, const int64_t *cap0, int64_t *excess)
{
    for (int64_t u = 0; u < n; u++) {
        int64_t acc = 0;
        for (int64_t i = offsets[u]; i < offsets[u + 1]; i++) {
            int64_t ri = rev[i];
            int64_t fin = cap0[ri] - cf[ri];
            if (fin > 0) acc += fin;
            int64_t fout = cap0[i] - cf[i];
            if (fout > 0) acc -= fout;
        }
        excess[u] = acc;
    }
}

/* BiCsrGraph.edge_indices, graph.py:101-108: key = u*n+v looked up in the
 * sorted key order (row u, ascending neighbour).  Keys outside [0, n*n)
 * are not found, exactly as searchsorted cannot match them. */
static int64_t edge_index(int64_t n, const int64_t *offsets, const int64_t *adj,
                          int64_t u, int64_t v)
{
    int64_t want = u * n + v;
    if (want < 0 || want >= n * n) return -1;
    int64_t uu = want / n, vv = want % n;
    int64_t lo = offsets[uu], hi = offsets[uu + 1];
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (adj[mid] < vv) lo = mid + 1; else hi = mid;
    }
    return (lo < offsets[uu + 1] && adj[lo] == vv) ? lo : -1;
}

static int cmp_pair(const void *a, const void *b)
{
    const int64_t *x = (const int64_t *)a, *y = (const int64_t *)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    return x[1] < y[1] ? -1 : (x[1] > y[1]);
}

/* _resolve_batch, dynamic.py:63-88.  Returns 0 or a BatchError kind
 * (1 negative capacity, 2 unknown/stub edge, 3 duplicate) with *bad = the
 * reference's reported update index.  idx receives the slots. */
int orc_resolve_batch(int64_t n, const int64_t *offsets, const int64_t *adj,
                      const uint8_t *is_original, int64_t k, const int64_t *us,
                      const int64_t *vs, const int64_t *new_caps, int64_t *idx,
                      int64_t *bad)
{
    *bad = -1;
    for (int64_t j = 0; j < k; j++)
        if (new_caps[j] < 0) { *bad = j; return 1; }
    for (int64_t j = 0; j < k; j++) {
        idx[j] = edge_index(n, offsets, adj, us[j], vs[j]);
    }
    for (int64_t j = 0; j < k; j++)
        if (idx[j] < 0 || !is_original[idx[j]]) { *bad = j; return 2; }
    /* stable argsort by slot: sort (slot, j) pairs */
    int64_t *pr = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)(k + 1));
    for (int64_t j = 0; j < k; j++) { pr[2 * j] = idx[j]; pr[2 * j + 1] = j; }
    qsort(pr, (size_t)k, 2 * sizeof(int64_t), cmp_pair);
    int rc = 0;
    for (int64_t p = 1; p < k; p++)
        if (pr[2 * p] == pr[2 * (p - 1)]) { *bad = pr[2 * p + 1]; rc = 3; break; }
    free(pr);
    return rc;
}

/* apply_updates, dynamic.py:91-111.  Returns 0, a BatchError kind (1-3)
 * or 4 when a negative residual survives (SolverError). */
int orc_apply_updates(int64_t n, const int64_t *offsets, const int64_t *adj,
                      const int64_t *rev, int64_t *cap0, const uint8_t *is_original,
                      int64_t *cf, int64_t k, const int64_t *us, const int64_t *vs,
                      const int64_t *new_caps, int64_t *bad)
{
    int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)(k + 1));
    int rc = orc_resolve_batch(n, offsets, adj, is_original, k, us, vs, new_caps, idx, bad);
    if (rc) { free(idx); return rc; }
    for (int64_t j = 0; j < k; j++) {
        cf[idx[j]] += new_caps[j] - cap0[idx[j]];
        cap0[idx[j]] = new_caps[j];
    }
    /* negative residuals: amounts captured first, then applied (numpy
     * fancy-index semantics of dynamic.py:105-109) */
    int64_t *amt = (int64_t *)malloc(sizeof(int64_t) * (size_t)(k + 1));
    for (int64_t j = 0; j < k; j++) amt[j] = cf[idx[j]] < 0 ? cf[idx[j]] : 0;
    for (int64_t j = 0; j < k; j++) if (amt[j] < 0) cf[rev[idx[j]]] += amt[j];
    for (int64_t j = 0; j < k; j++) if (amt[j] < 0) cf[idx[j]] = 0;
    for (int64_t j = 0; j < k; j++)
        if (cf[idx[j]] < 0 || cf[rev[idx[j]]] < 0) rc = 4;
    free(amt); free(idx);
    return rc;
}

/* extract_certificate, solver.py:178-184: cut over original slots A->B with
 * A = {h == n}.  Returns -1 if an active vertex remains. */
int64_t orc_cut_capacity(int64_t n, const int64_t *offsets, const int64_t *adj,
                         const int64_t *cap0, const uint8_t *is_original,
                         const int64_t *excess, const int64_t *height,
                         int64_t s, int64_t t)
{
    for (int64_t v = 0; v < n; v++)
        if (v != s && v != t && excess[v] > 0 && height[v] < n) return -1;
    int64_t cut = 0;
    for (int64_t u = 0; u < n; u++) {
        if (height[u] != n) continue;
        for (int64_t i = offsets[u]; i < offsets[u + 1]; i++)
            if (is_original[i] && height[adj[i]] != n) cut += cap0[i];
    }
    return cut;
}

/* ------------------------------------------------------------------ */
/* solvers                                                              */
/* ------------------------------------------------------------------ */
typedef struct {
    int64_t flow, cut, rounds, pushes, relabels, repairs;
    int64_t status; /* 0 ok, 2 batch error kind in bad, 3 solver error, 5 time cap hit */
    int64_t bad;    /* batch error: kind*2^32 + index */
} orc_result;

/* active_mask, state.py:62-67 */
static int is_active(int64_t v, int64_t n, const int64_t *excess, const int64_t *height,
                     int64_t s, int64_t t)
{
    return v != s && v != t && excess[v] > 0 && height[v] < n;
}

/* _push_rounds, solver.py:204-241 (deterministic single-worker schedule).
 * dynamic != 0 selects _dynamic_bases/forbidden=s (dynamic.py:119-133,
 * 162-168); topology != 0 selects the all-vertex worklist (solver.py:170-174). */
static void push_rounds(int64_t n, const int64_t *offsets, const int64_t *adj,
                        const int64_t *rev, int64_t *cf, int64_t *excess,
                        int64_t *height, int64_t s, int64_t t, int64_t kc,
                        int dynamic, int topology, orc_result *r)
{
    int64_t *bases = (int64_t *)calloc((size_t)(n + 1), sizeof(int64_t));
    int64_t *work = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    int64_t counts[2] = {0, 0};
    for (;;) {
        int64_t nb = 0;
        if (dynamic) {
            for (int64_t v = 0; v < n; v++)
                if (v == t || (v != s && excess[v] < 0)) bases[nb++] = v;
        } else {
            bases[nb++] = t;
        }
        orc_bfs_heights(n, offsets, adj, rev, cf, height, bases, nb, dynamic ? s : -1);
        int64_t nw = 0;
        for (int64_t v = 0; v < n; v++)
            if (is_active(v, n, excess, height, s, t)) work[nw++] = v;
        if (nw == 0) break;
        if (topology) {
            nw = 0;
            for (int64_t v = 0; v < n; v++) if (v != s && v != t) work[nw++] = v;
        }
        orc_push_relabel(work, nw, offsets, adj, rev, cf, excess, height, n, kc, counts);
        r->repairs += orc_remove_invalid(work, nw, offsets, adj, rev, cf, excess, height);
        r->rounds++;
        if (g_deadline > 0 && now_s() > g_deadline) { r->status = 5; break; }
    }
    r->pushes += counts[0];
    r->relabels += counts[1];
    free(bases); free(work);
}

/* solve_static, solver.py:253-283 (state arrays caller-allocated) */
void orc_solve_static(int64_t n, const int64_t *offsets, const int64_t *adj,
                      const int64_t *rev, const int64_t *cap0, const uint8_t *is_original,
                      int64_t *cf, int64_t *excess, int64_t *height, int64_t s,
                      int64_t t, int64_t kc, int topology, orc_result *r)
{
    memset(r, 0, sizeof(*r));
    int64_t S = offsets[n];
    memcpy(cf, cap0, sizeof(int64_t) * (size_t)S);
    memset(excess, 0, sizeof(int64_t) * (size_t)n);
    memset(height, 0, sizeof(int64_t) * (size_t)n);
    orc_saturate_source(s, offsets, adj, rev, cf, excess);
    push_rounds(n, offsets, adj, rev, cf, excess, height, s, t, kc, 0, topology, r);
    if (r->status == 5) return;
    r->flow = excess[t];
    r->cut = orc_cut_capacity(n, offsets, adj, cap0, is_original, excess, height, s, t);
    if (r->cut != r->flow) r->status = 3;
}

/* solve_dynamic, dynamic.py:146-175 */
void orc_solve_dynamic(int64_t n, const int64_t *offsets, const int64_t *adj,
                       const int64_t *rev, int64_t *cap0, const uint8_t *is_original,
                       int64_t *cf, int64_t *excess, int64_t *height, int64_t s,
                       int64_t t, int64_t kc, int topology, int64_t k,
                       const int64_t *us, const int64_t *vs, const int64_t *new_caps,
                       orc_result *r)
{
    memset(r, 0, sizeof(*r));
    for (int64_t v = 0; v < n; v++)
        if (is_active(v, n, excess, height, s, t)) { r->status = 3; return; }
    int64_t bad = -1;
    int rc = orc_apply_updates(n, offsets, adj, rev, cap0, is_original, cf, k, us, vs,
                               new_caps, &bad);
    if (rc == 4) { r->status = 3; return; }
    if (rc) { r->status = 2; r->bad = ((int64_t)rc << 32) | bad; return; }
    orc_recompute_excess(n, offsets, rev, cf, cap0, excess);
    orc_saturate_source(s, offsets, adj, rev, cf, excess);
    push_rounds(n, offsets, adj, rev, cf, excess, height, s, t, kc, 1, topology, r);
    if (r->status == 5) return;
    int64_t flow = 0;
    for (int64_t v = 0; v < n; v++) if (height[v] == 0) flow += excess[v];
    r->flow = flow;
    r->cut = orc_cut_capacity(n, offsets, adj, cap0, is_original, excess, height, s, t);
    if (r->cut != r->flow) r->status = 3;
}

/* dinic_maxflow, oracle.py:20-55 + _augment_in_level_graph oracle.py:58-84,
 * restated on the Bi-CSR residual layout: the reference builds its own
 * per-vertex [head, residual, reverse] lists from the edge list, and a
 * Bi-CSR slot pair (i, rev i) with cf = cap0 is exactly that residual
 * graph with parallel edges merged.  Level graph by BFS from s over cf > 0;
 * blocking flow by iterative current-arc DFS, dead ends get level -1.
 * Leaves the final residuals in cf (cf = cap0 on entry is the caller's job)
 * and returns the flow value.  Test infrastructure: it produces terminated
 * states for the capped CPU baselines and checks flow values. */
int64_t orc_dinic(int64_t n, const int64_t *offsets, const int64_t *adj, const int64_t *rev,
                  int64_t *cf, int64_t s, int64_t t)
{
    if (s == t) return -1;
    int64_t *level = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *queue = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *it = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *path = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1)); /* slots */
    int64_t total = 0;
    for (;;) {
        for (int64_t v = 0; v < n; v++) level[v] = -1;
        level[s] = 0;
        int64_t head = 0, tail = 0;
        queue[tail++] = s;
        while (head < tail) {
            int64_t u = queue[head++];
            for (int64_t i = offsets[u]; i < offsets[u + 1]; i++) {
                int64_t v = adj[i];
                if (cf[i] > 0 && level[v] < 0) { level[v] = level[u] + 1; queue[tail++] = v; }
            }
        }
        if (level[t] < 0) break;
        for (int64_t v = 0; v < n; v++) it[v] = offsets[v];
        for (;;) { /* augmenting paths inside the level graph */
            int64_t depth = 0, u = s, pushed = 0;
            for (;;) {
                if (u == t) {
                    int64_t amt = INT64_MAX;
                    for (int64_t d = 0; d < depth; d++) if (cf[path[d]] < amt) amt = cf[path[d]];
                    for (int64_t d = 0; d < depth; d++) { cf[path[d]] -= amt; cf[rev[path[d]]] += amt; }
                    pushed = amt;
                    break;
                }
                int advanced = 0;
                while (it[u] < offsets[u + 1]) {
                    int64_t i = it[u];
                    if (cf[i] > 0 && level[adj[i]] == level[u] + 1) {
                        path[depth++] = i;
                        u = adj[i];
                        advanced = 1;
                        break;
                    }
                    it[u]++;
                }
                if (!advanced) {
                    level[u] = -1;
                    if (depth == 0) break;
                    u = (depth >= 2) ? adj[path[depth - 2]] : s;
                    depth--;
                }
            }
            if (pushed == 0) break;
            total += pushed;
        }
    }
    free(level); free(queue); free(it); free(path);
    return total;
}
