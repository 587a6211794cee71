// state.cu -- state primitives, the O(k) dynamic batch pre-phase, and the
// device verifiers.
//
// Batch pre-phase (replaces apply_updates + recompute_excess + saturate_source,
// dynamic.py:91-116 and state.py:42-59):
//   resolve   slot lookup by binary search in row u, validation exactly in the
//             reference order: negative capacity, unknown/stub edge, duplicate
//             (dynamic.py:63-88); nothing is mutated if any check fails.
//   apply     cf += new - cap0, cap0 = new (dynamic.py:103-104)
//   repair    negative residual -> flow reversal (dynamic.py:105-109); the
//             excess moves only at the repaired endpoints, which is what the
//             reference's O(n + S) recompute_excess yields (SURVEY 8a A14:
//             excess[u] == sum_row(u) (cf - cap0) is invariant under the delta)
//   pc        refresh pair capacities of the touched pairs
//   saturate  the source row (state.py:42-59)
#include <limits.h>

#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "engine.h"

namespace mfx {

static inline int grid_for(long long work, int num_sms, int per_sm = 8) {
  long long g = (work + kBlock - 1) / kBlock;
  long long cap = (long long)num_sms * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ bool batch_failed(const long long *err);

template <typename CapT>
__global__ void saturate_kernel(const int *__restrict__ off, const int *__restrict__ adj,
                                const int *__restrict__ rev, CapT *cf, long long *ex, int s,
                                const long long *gate) {
  pdl_wait();
  __shared__ long long scr[kWarps];
  if (gate && batch_failed(gate)) return;
  int lo = off[s], hi = off[s + 1];
  long long sum = 0;
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x) {
    CapT d = cf[i];
    if (d > 0) {
      cf[i] = 0;
      // rev[i] and adj[i] are distinct across the row: plain read-modify-write
      cf[rev[i]] += d;
      ex[adj[i]] += (long long)d;
      sum += (long long)d;
    }
  }
  sum = warp_sum(sum);
  if ((threadIdx.x & 31) == 0) scr[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < kWarps; ++w) t += scr[w];
    if (t) atomicAdd((unsigned long long *)(ex + s), (unsigned long long)(-t));
  }
}

template <typename CapT>
static cudaError_t saturate_t(const GraphObj &g, StateObj &st, const long long *gate) {
  Topology &T = *g.topo;
  cudaError_t e = pdl_launch(saturate_kernel<CapT>, grid_for(1 << 22, T.num_sms, 2), kBlock,
                             T.stream, (const int *)T.off, (const int *)T.adj, (const int *)T.rev,
                             (CapT *)st.cf, st.ex, st.s, gate);
  count_launch();
  return e ? e : cudaGetLastError();
}

cudaError_t launch_saturate(const GraphObj &g, StateObj &st, const long long *gate) {
  return g.topo->cap_bytes == 8 ? saturate_t<long long>(g, st, gate)
                                : saturate_t<int>(g, st, gate);
}

cudaError_t launch_init_state(const GraphObj &g, StateObj &st) {
  Topology &T = *g.topo;
  cudaError_t e = cudaMemcpyAsync(st.cf, g.cap0, (size_t)T.S * T.cap_bytes,
                                  cudaMemcpyDeviceToDevice, T.stream);
  if (e) return e;
  if ((e = cudaMemsetAsync(st.ex, 0, sizeof(long long) * (size_t)T.n, T.stream))) return e;
  e = cudaMemsetAsync(st.h, 0, sizeof(int) * (size_t)T.n, T.stream);
  st.tl_ok = false;
  st.excess_consistent = true;
  st.terminated_known = false;
  return e;
}

__global__ void vbin_kernel(const int *off, int n, uint8_t *vbin) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    vbin[v] = (uint8_t)bin_of(off[v + 1] - off[v]);
}

__global__ void long_rows_kernel(const int *off, int n, unsigned long long *acc) {
  unsigned long long x = 0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int d = off[v + 1] - off[v];
    if (d > kBin0Max) x += (unsigned long long)d;
  }
  x = warp_sum(x);
  if ((threadIdx.x & 31) == 0 && x) atomicAdd(acc, x);
}

cudaError_t long_row_permille(const Topology &t, int *permille) {
  *permille = 0;
  if (t.S <= 0) return cudaSuccess;
  unsigned long long *d = nullptr, h = 0;
  cudaError_t e = cudaMalloc(&d, sizeof(h));
  if (e) return e;
  cudaMemsetAsync(d, 0, sizeof(h), t.stream);
  long_rows_kernel<<<grid_for(t.n, t.num_sms), kBlock, 0, t.stream>>>(t.off, t.n, d);
  count_launch();
  e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, t.stream);
  if (!e) e = cudaStreamSynchronize(t.stream);
  cudaFree(d);
  *permille = (int)(1000.0 * (double)h / (double)t.S);
  return e;
}

cudaError_t launch_vbin(const Topology &t, uint8_t *vbin) {
  if (t.n == 0) return cudaSuccess;
  vbin_kernel<<<grid_for(t.n, t.num_sms), kBlock, 0, t.stream>>>(t.off, t.n, vbin);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
__global__ void mask_kernel(const long long *ex, const int *h, int n, int s, int t, int which,
                            uint8_t *out) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    bool m;
    if (which == 0) m = v != s && v != t && ex[v] > 0 && h[v] < n;       // active_mask
    else if (which == 1) m = v != s && v != t && ex[v] < 0;              // deficient_mask
    else m = h[v] == n;                                                   // cut side A
    out[v] = m;
  }
}

cudaError_t launch_mask(const StateObj &st, int which, uint8_t *d_out) {
  Topology &T = *st.topo;
  mask_kernel<<<grid_for(T.n, T.num_sms), kBlock, 0, T.stream>>>(st.ex, st.h, T.n, st.s, st.t,
                                                                  which, d_out);
  count_launch();
  return cudaGetLastError();
}

__global__ void count_active_kernel(const long long *ex, const int *h, int n, int s, int t,
                                    unsigned long long *out) {
  unsigned long long c = 0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    c += (v != s && v != t && ex[v] > 0 && h[v] < n);
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

cudaError_t launch_count_active(const StateObj &st, unsigned long long *d_out) {
  Topology &T = *st.topo;
  cudaError_t e = cudaMemsetAsync(d_out, 0, sizeof(unsigned long long), T.stream);
  if (e) return e;
  count_active_kernel<<<grid_for(T.n, T.num_sms), kBlock, 0, T.stream>>>(st.ex, st.h, T.n, st.s,
                                                                          st.t, d_out);
  count_launch();
  return cudaGetLastError();
}

// recompute_excess (kernels.py:218-231), warp per vertex
template <typename CapT>
__global__ void recompute_excess_kernel(const int *__restrict__ off, const int *__restrict__ rev,
                                        const CapT *__restrict__ cf, const CapT *__restrict__ cap0,
                                        long long *ex, int n) {
  int lane = threadIdx.x & 31;
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int u = w; u < n; u += nw) {
    long long acc = 0;
    for (int i = off[u] + lane; i < off[u + 1]; i += 32) {
      int ri = rev[i];
      long long fin = (long long)cap0[ri] - (long long)cf[ri];
      if (fin > 0) acc += fin;
      long long fout = (long long)cap0[i] - (long long)cf[i];
      if (fout > 0) acc -= fout;
    }
    acc = warp_sum(acc);
    if (lane == 0) ex[u] = acc;
  }
}

cudaError_t launch_recompute_excess(const GraphObj &g, StateObj &st) {
  Topology &T = *g.topo;
  int grid = grid_for((long long)T.n * 32, T.num_sms);
  if (T.cap_bytes == 8)
    recompute_excess_kernel<long long><<<grid, kBlock, 0, T.stream>>>(
        T.off, T.rev, (const long long *)st.cf, (const long long *)g.cap0, st.ex, T.n);
  else
    recompute_excess_kernel<int><<<grid, kBlock, 0, T.stream>>>(
        T.off, T.rev, (const int *)st.cf, (const int *)g.cap0, st.ex, T.n);
  count_launch();
  st.excess_consistent = true;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// batch pre-phase
// ---------------------------------------------------------------------------
// d_err layout (int64): 0 first negative-capacity update, 1 first unknown/stub
// update, 2 smallest duplicated slot, 3 reported duplicate update, 4 first
// update overflowing int32 residual storage.  LLONG_MAX = none.
enum { E_NEG = 0, E_UNKNOWN = 1, E_DUPSLOT = 2, E_DUPK = 3, E_OVER = 4, E_N = 8 };

__device__ __forceinline__ bool batch_failed(const long long *err) {
  return err[E_NEG] != LLONG_MAX || err[E_UNKNOWN] != LLONG_MAX || err[E_DUPK] != LLONG_MAX ||
         err[E_OVER] != LLONG_MAX;
}

// BiCsrGraph.edge_indices (graph.py:101-108): key u*n+v with numpy's wrapping
// int64 arithmetic, looked up in the (u, v)-sorted slot order.
__device__ __forceinline__ int find_slot(const int *__restrict__ off, const int *__restrict__ adj,
                                         int n, long long u, long long v, int *uu_out, int *vv_out) {
  long long want = (long long)((unsigned long long)u * (unsigned long long)n + (unsigned long long)v);
  long long nn = (long long)n * (long long)n;
  if (want < 0 || want >= nn) return -1;
  int uu = (int)(want / n), vv = (int)(want % n);
  *uu_out = uu;
  *vv_out = vv;
  int lo = off[uu], hi = off[uu + 1];
  while (lo < hi) {
    int mid = lo + ((hi - lo) >> 1);
    if (adj[mid] < vv) lo = mid + 1;
    else hi = mid;
  }
  return (lo < off[uu + 1] && adj[lo] == vv) ? lo : -1;
}

template <typename CapT>
__global__ void batch_resolve_kernel(const int *__restrict__ off, const int *__restrict__ adj,
                                     const int *__restrict__ rev, const uint8_t *__restrict__ orig,
                                     const CapT *__restrict__ cap0, int n, long long k,
                                     const long long *us, const long long *vs, const long long *caps,
                                     int *slot, int *uv, long long *err) {
  pdl_wait();
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < k;
       j += (long long)gridDim.x * blockDim.x) {
    long long c = caps[j];
    if (c < 0) atomicMin(err + E_NEG, j);
    int uu = 0, vv = 0;
    int i = find_slot(off, adj, n, us[j], vs[j], &uu, &vv);
    slot[j] = i;
    uv[2 * j] = uu;
    uv[2 * j + 1] = vv;
    if (i < 0 || !orig[i]) atomicMin(err + E_UNKNOWN, j);
  }
}

// int32 residual storage needs every post-batch pair sum below 2^31: the new
// capacity plus the partner slot's capacity after the batch (its own update
// if it is in the batch, found through slot_first, else its cap0).
template <typename CapT>
__global__ void batch_over_kernel(long long k, const int *slot, const int *first,
                                  const int *__restrict__ rev, const CapT *cap0,
                                  const long long *caps, long long *err) {
  pdl_wait();
  if (err[E_NEG] != LLONG_MAX || err[E_UNKNOWN] != LLONG_MAX) return;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < k;
       j += (long long)gridDim.x * blockDim.x) {
    int r = rev[slot[j]];
    int jr = first[r];
    long long partner = jr != kFirstNone ? caps[jr] : (long long)cap0[r];
    if (caps[j] + partner >= (1ll << 31)) atomicMin(err + E_OVER, j);
  }
}

__global__ void batch_first_kernel(long long k, const int *slot, int *first, const long long *err) {
  pdl_wait();
  if (err[E_NEG] != LLONG_MAX || err[E_UNKNOWN] != LLONG_MAX) return;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < k;
       j += (long long)gridDim.x * blockDim.x)
    atomicMin(first + slot[j], (int)j);
}

__global__ void batch_dup_kernel(long long k, const int *slot, const int *first, long long *err) {
  pdl_wait();
  if (err[E_NEG] != LLONG_MAX || err[E_UNKNOWN] != LLONG_MAX) return;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < k;
       j += (long long)gridDim.x * blockDim.x)
    if (first[slot[j]] != (int)j) atomicMin(err + E_DUPSLOT, (long long)slot[j]);
}

// reference reports order[p] of the first equal pair in the stable (slot, j)
// order: the second-smallest update index on the smallest duplicated slot
__global__ void batch_dupidx_kernel(long long k, const int *slot, const int *first, long long *err) {
  pdl_wait();
  if (err[E_NEG] != LLONG_MAX || err[E_UNKNOWN] != LLONG_MAX || err[E_DUPSLOT] == LLONG_MAX) return;
  long long ds = err[E_DUPSLOT];
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < k;
       j += (long long)gridDim.x * blockDim.x)
    if (slot[j] == ds && first[slot[j]] != (int)j) atomicMin(err + E_DUPK, j);
}

template <typename CapT>
__global__ void batch_apply_kernel(long long k, const int *slot, int *first, const long long *caps,
                                   CapT *cap0, CapT *cf, const long long *err, int apply) {
  pdl_wait();
  bool ok = apply && !batch_failed(err);
  bool resolved = err[E_NEG] == LLONG_MAX && err[E_UNKNOWN] == LLONG_MAX;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < k;
       j += (long long)gridDim.x * blockDim.x) {
    int i = slot[j];
    if (resolved) first[i] = kFirstNone;  // restore the scratch invariant
    if (ok) {
      CapT nc = (CapT)caps[j];
      if (cf) cf[i] += nc - cap0[i];
      cap0[i] = nc;
    }
  }
}

template <typename CapT>
__global__ void batch_repair_kernel(long long k, const int *slot, const int *uv,
                                    const int *__restrict__ rev, CapT *cf, long long *ex,
                                    const long long *err) {
  pdl_wait();
  if (batch_failed(err)) return;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < k;
       j += (long long)gridDim.x * blockDim.x) {
    int i = slot[j];
    CapT c = cf[i];
    if (c < 0) {  // new capacity below the committed flow: reverse the surplus
      cf[i] = 0;
      atomic_add(cf + rev[i], c);
      if (ex) {
        atomic_add(ex + uv[2 * j], -(long long)c);
        atomic_add(ex + uv[2 * j + 1], (long long)c);
      }
    }
  }
}

template <typename CapT>
__global__ void batch_pc_kernel(long long k, const int *slot, const int *__restrict__ rev,
                                const CapT *cap0, CapT *pc, const long long *err) {
  pdl_wait();
  if (batch_failed(err)) return;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < k;
       j += (long long)gridDim.x * blockDim.x) {
    int i = slot[j], r = rev[i];
    CapT p = cap0[i] + cap0[r];
    pc[i] = p;
    pc[r] = p;
  }
}

__global__ void fill_ll_kernel(long long *p, int cnt, long long v) {
  pdl_wait();
  if (threadIdx.x < cnt) p[threadIdx.x] = v;
}

template <typename CapT>
static cudaError_t batch_t(GraphObj &g, StateObj *st, int64_t k, const int64_t *d_us,
                           const int64_t *d_vs, const int64_t *d_caps, bool apply,
                           bool update_excess, int *launches) {
  Topology &T = *g.topo;
  Workspace &W = T.ws;
  cudaError_t e = pdl_launch(fill_ll_kernel, 1, 32, T.stream, W.d_err, (int)E_N, (long long)LLONG_MAX);
  count_launch();
  if (launches) *launches += 1;
  if (e || k == 0) return e ? e : cudaGetLastError();
  int grid = grid_for(k, T.num_sms);
  const long long *us = (const long long *)d_us, *vs = (const long long *)d_vs,
                  *cs = (const long long *)d_caps;
  const long long kk = k;
#define PDL(...) \
  if ((e = pdl_launch(__VA_ARGS__))) return e
  PDL(batch_resolve_kernel<CapT>, grid, kBlock, T.stream, (const int *)T.off, (const int *)T.adj,
      (const int *)T.rev, (const uint8_t *)T.orig, (const CapT *)g.cap0, T.n, kk, us, vs, cs,
      W.d_slot, W.d_uv, W.d_err);
  PDL(batch_first_kernel, grid, kBlock, T.stream, kk, (const int *)W.d_slot, W.slot_first,
      (const long long *)W.d_err);
  if (sizeof(CapT) == 4) {
    PDL(batch_over_kernel<CapT>, grid, kBlock, T.stream, kk, (const int *)W.d_slot,
        (const int *)W.slot_first, (const int *)T.rev, (const CapT *)g.cap0, cs, W.d_err);
    count_launch();
    if (launches) *launches += 1;
  }
  PDL(batch_dup_kernel, grid, kBlock, T.stream, kk, (const int *)W.d_slot,
      (const int *)W.slot_first, W.d_err);
  PDL(batch_dupidx_kernel, grid, kBlock, T.stream, kk, (const int *)W.d_slot,
      (const int *)W.slot_first, W.d_err);
  PDL(batch_apply_kernel<CapT>, grid, kBlock, T.stream, kk, (const int *)W.d_slot, W.slot_first,
      cs, (CapT *)g.cap0, st ? (CapT *)st->cf : (CapT *)nullptr, (const long long *)W.d_err,
      apply ? 1 : 0);
  int nl = 5;
  if (apply && st) {
    PDL(batch_repair_kernel<CapT>, grid, kBlock, T.stream, kk, (const int *)W.d_slot,
        (const int *)W.d_uv, (const int *)T.rev, (CapT *)st->cf,
        update_excess ? st->ex : (long long *)nullptr, (const long long *)W.d_err);
    ++nl;
  }
  if (apply) {
    PDL(batch_pc_kernel<CapT>, grid, kBlock, T.stream, kk, (const int *)W.d_slot,
        (const int *)T.rev, (const CapT *)g.cap0, (CapT *)g.pc, (const long long *)W.d_err);
    ++nl;
  }
#undef PDL
  if (launches) *launches += nl;
  count_launch(nl);
  return cudaGetLastError();
}

cudaError_t launch_batch(GraphObj &g, StateObj *st, int64_t k, const int64_t *d_us,
                         const int64_t *d_vs, const int64_t *d_caps, bool apply,
                         bool update_excess, int *launches) {
  if (g.topo->cap_bytes == 8)
    return batch_t<long long>(g, st, k, d_us, d_vs, d_caps, apply, update_excess, launches);
  return batch_t<int>(g, st, k, d_us, d_vs, d_caps, apply, update_excess, launches);
}

__global__ void edge_indices_kernel(const int *__restrict__ off, const int *__restrict__ adj, int n,
                                    long long k, const long long *us, const long long *vs,
                                    long long *out) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < k;
       j += (long long)gridDim.x * blockDim.x) {
    int uu, vv;
    out[j] = find_slot(off, adj, n, us[j], vs[j], &uu, &vv);
  }
}

cudaError_t launch_edge_indices(const GraphObj &g, int64_t k, const int64_t *d_us,
                                const int64_t *d_vs, int64_t *d_out) {
  Topology &T = *g.topo;
  if (k == 0) return cudaSuccess;
  edge_indices_kernel<<<grid_for(k, T.num_sms), kBlock, 0, T.stream>>>(
      T.off, T.adj, T.n, k, (const long long *)d_us, (const long long *)d_vs, (long long *)d_out);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// capacity width conversion and pair sums
// ---------------------------------------------------------------------------
__global__ void narrow_kernel(const long long *src, int *dst, long long cnt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = (int)src[i];
}
__global__ void widen_kernel(const int *src, long long *dst, long long cnt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

cudaError_t launch_convert_cap(const int64_t *src, void *dst, int cap_bytes, int64_t cnt,
                               cudaStream_t s) {
  if (cnt == 0) return cudaSuccess;
  if (cap_bytes == 8)
    return cudaMemcpyAsync(dst, src, sizeof(int64_t) * cnt, cudaMemcpyDeviceToDevice, s);
  narrow_kernel<<<grid_for(cnt, 148), kBlock, 0, s>>>((const long long *)src, (int *)dst, cnt);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_widen_cap(const void *src, int64_t *dst, int cap_bytes, int64_t cnt,
                             cudaStream_t s) {
  if (cnt == 0) return cudaSuccess;
  if (cap_bytes == 8)
    return cudaMemcpyAsync(dst, src, sizeof(int64_t) * cnt, cudaMemcpyDeviceToDevice, s);
  widen_kernel<<<grid_for(cnt, 148), kBlock, 0, s>>>((const int *)src, (long long *)dst, cnt);
  count_launch();
  return cudaGetLastError();
}

template <typename CapT>
__global__ void pc_full_kernel(const int *__restrict__ rev, const CapT *cap0, CapT *pc, int S) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x)
    pc[i] = cap0[i] + cap0[rev[i]];
}

cudaError_t launch_refresh_pc(const GraphObj &g) {
  Topology &T = *g.topo;
  if (T.S == 0) return cudaSuccess;
  int grid = grid_for(T.S, T.num_sms);
  if (T.cap_bytes == 8)
    pc_full_kernel<long long><<<grid, kBlock, 0, T.stream>>>(T.rev, (const long long *)g.cap0,
                                                             (long long *)g.pc, T.S);
  else
    pc_full_kernel<int><<<grid, kBlock, 0, T.stream>>>(T.rev, (const int *)g.cap0, (int *)g.pc, T.S);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// verification (oracle.py:111-225 on the device) and certificate
// ---------------------------------------------------------------------------
enum {
  V_NEG = 0, V_PAIR, V_EXMIS, V_EXSUM, V_ACTIVE, V_UNSAT, V_LOADED, V_CUT, V_FLOW, V_SB, V_TA,
  V_FIRSTBAD, V_N = 16
};

template <typename CapT>
__global__ void verify_kernel(const int *__restrict__ off, const int *__restrict__ adj,
                              const int *__restrict__ rev, const uint8_t *__restrict__ orig,
                              const CapT *__restrict__ cap0, const CapT *__restrict__ cf,
                              const long long *__restrict__ ex, const int *__restrict__ h, int n,
                              int s, int t, long long *rep) {
  int lane = threadIdx.x & 31;
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  long long neg = 0, pair = 0, exmis = 0, exsum = 0, active = 0, unsat = 0, loaded = 0, cut = 0,
            flow = 0;
  for (int u = w; u < n; u += nw) {
    int hu = h[u];
    bool au = hu == n;
    long long rowsum = 0;
    for (int i = off[u] + lane; i < off[u + 1]; i += 32) {
      long long c = cf[i], k0 = cap0[i];
      int r = rev[i];
      if (c < 0) {
        ++neg;
        atomicMin(rep + V_FIRSTBAD, (long long)i);
      }
      if (c + (long long)cf[r] != k0 + (long long)cap0[r]) {
        ++pair;
        atomicMin(rep + V_FIRSTBAD, (long long)i);
      }
      rowsum += c - k0;
      bool av = h[adj[i]] == n;
      if (orig[i] && au && !av) {
        cut += k0;
        if (c != 0) ++unsat;
      }
      if (orig[i] && !au && av) {
        long long f = k0 - c;
        if (f > 0) ++loaded;
      }
    }
    rowsum = warp_sum(rowsum);
    if (lane == 0) {
      long long e = ex[u];
      if (e != rowsum) ++exmis;
      exsum += e;
      if (u != s && u != t && e > 0 && hu < n) ++active;
      if (hu == 0) flow += e;
    }
  }
  neg = warp_sum(neg);
  pair = warp_sum(pair);
  unsat = warp_sum(unsat);
  loaded = warp_sum(loaded);
  cut = warp_sum(cut);
  if (lane == 0) {
    if (neg) atomicAdd((unsigned long long *)(rep + V_NEG), (unsigned long long)neg);
    if (pair) atomicAdd((unsigned long long *)(rep + V_PAIR), (unsigned long long)pair);
    if (exmis) atomicAdd((unsigned long long *)(rep + V_EXMIS), (unsigned long long)exmis);
    if (exsum) atomicAdd((unsigned long long *)(rep + V_EXSUM), (unsigned long long)exsum);
    if (active) atomicAdd((unsigned long long *)(rep + V_ACTIVE), (unsigned long long)active);
    if (unsat) atomicAdd((unsigned long long *)(rep + V_UNSAT), (unsigned long long)unsat);
    if (loaded) atomicAdd((unsigned long long *)(rep + V_LOADED), (unsigned long long)loaded);
    if (cut) atomicAdd((unsigned long long *)(rep + V_CUT), (unsigned long long)cut);
    if (flow) atomicAdd((unsigned long long *)(rep + V_FLOW), (unsigned long long)flow);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    rep[V_SB] = h[s] != n;
    rep[V_TA] = h[t] == n;
  }
}

cudaError_t launch_verify(const GraphObj &g, const StateObj &st, long long *d_rep) {
  Topology &T = *g.topo;
  fill_ll_kernel<<<1, 32, 0, T.stream>>>(d_rep, V_N, 0);
  fill_ll_kernel<<<1, 32, 0, T.stream>>>(d_rep + V_FIRSTBAD, 1, LLONG_MAX);
  count_launch(2);
  int grid = grid_for((long long)T.n * 32, T.num_sms);
  if (T.cap_bytes == 8)
    verify_kernel<long long><<<grid, kBlock, 0, T.stream>>>(
        T.off, T.adj, T.rev, T.orig, (const long long *)g.cap0, (const long long *)st.cf, st.ex,
        st.h, T.n, st.s, st.t, d_rep);
  else
    verify_kernel<int><<<grid, kBlock, 0, T.stream>>>(T.off, T.adj, T.rev, T.orig,
                                                      (const int *)g.cap0, (const int *)st.cf,
                                                      st.ex, st.h, T.n, st.s, st.t, d_rep);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// capacity consistency checks
// ---------------------------------------------------------------------------
// cf[i] + cf[rev i] == pc[i] on every slot (residual-sum conservation,
// oracle.py:118): out[0] = violations, out[1] = first violating slot.
template <typename CapT>
__global__ void pair_check_kernel(const CapT *cf, const CapT *pc, const int *__restrict__ rev,
                                  int S, unsigned long long *out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x)
    if ((long long)cf[i] + (long long)cf[rev[i]] != (long long)pc[i]) {
      atomicAdd(out, 1ull);
      atomicMin(out + 1, (unsigned long long)i);
    }
}

cudaError_t launch_pair_check(const GraphObj &g, const StateObj &st, unsigned long long *d_out) {
  const Topology &T = *g.topo;
  unsigned long long init[2] = {0ull, ~0ull};
  cudaError_t e = cudaMemcpyAsync(d_out, init, sizeof(init), cudaMemcpyHostToDevice, T.stream);
  if (e || T.S == 0) return e;
  if (T.cap_bytes == 8)
    pair_check_kernel<long long><<<grid_for(T.S, T.num_sms), kBlock, 0, T.stream>>>(
        (const long long *)st.cf, (const long long *)g.pc, T.rev, T.S, d_out);
  else
    pair_check_kernel<int><<<grid_for(T.S, T.num_sms), kBlock, 0, T.stream>>>(
        (const int *)st.cf, (const int *)g.pc, T.rev, T.S, d_out);
  count_launch();
  return cudaGetLastError();
}

// capacities staged as int64 for set_cap0: out[0] = first negative slot,
// out[1] = first slot whose pair sum reaches 2^31 (int32 storage only).
__global__ void cap_check_kernel(const long long *cap, const int *__restrict__ rev, int S,
                                 int narrow, unsigned long long *out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
    long long c = cap[i];
    if (c < 0) atomicMin(out, (unsigned long long)i);
    else if (narrow && c + cap[rev[i]] >= (1ll << 31)) atomicMin(out + 1, (unsigned long long)i);
  }
}

cudaError_t launch_cap_check(const Topology &T, const int64_t *d_cap, unsigned long long *d_out) {
  unsigned long long init[2] = {~0ull, ~0ull};
  cudaError_t e = cudaMemcpyAsync(d_out, init, sizeof(init), cudaMemcpyHostToDevice, T.stream);
  if (e || T.S == 0) return e;
  cap_check_kernel<<<grid_for(T.S, T.num_sms), kBlock, 0, T.stream>>>(
      (const long long *)d_cap, T.rev, T.S, T.cap_bytes == 4, d_out);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// device batch sampler on one graph (gen.py fast_batch semantics, the law of
// the partitioned engine's mfx_part_sample_batch): k_dec decrements among the
// original slots with capacity (new in [0, old)), then k_inc increments among
// the rest (new in [old + 1, 2 old + 10]), drawn without replacement by
// exponential-race keys with weight `bias` on the source row and on slots
// into the sink; emitted in slot order = (u, v) order.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long smix_s(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void sample_weight_kernel(const int *__restrict__ adj, const uint8_t *__restrict__ orig,
                                     long long S, long long s_lo, long long s_hi, int t, double bias,
                                     unsigned long long *acc) {
  unsigned long long w = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < S;
       i += (long long)gridDim.x * blockDim.x)
    if (orig[i]) w += (adj[i] == t || (i >= s_lo && i < s_hi)) ? (unsigned long long)bias : 1ull;
  w = warp_sum(w);
  if ((threadIdx.x & 31) == 0 && w) atomicAdd(acc, w);
}

template <typename CapT>
__global__ void sample_kernel(const int *__restrict__ adj, const uint8_t *__restrict__ orig,
                              const CapT *__restrict__ cap0, const uint8_t *taken, long long S,
                              long long s_lo, long long s_hi, int t, double bias,
                              unsigned long long seed, int dec, double tau, int cap,
                              unsigned long long *cand, int *cnt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < S;
       i += (long long)gridDim.x * blockDim.x) {
    if (!orig[i] || taken[i] || (dec && cap0[i] <= 0)) continue;
    const unsigned long long h = smix_s(seed ^ smix_s((unsigned long long)i));
    const double u = ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    const double w = (adj[i] == t || (i >= s_lo && i < s_hi)) ? bias : 1.0;
    const double key = -log(u) / w;
    if (key < tau) {
      const int q = atomicAdd(cnt, 1);
      if (q < cap) cand[q] = ((unsigned long long)__float_as_uint((float)key) << 32) | (unsigned)i;
    }
  }
}

template <typename CapT>
__global__ void sample_emit_kernel(const int *__restrict__ off, int n, const int *__restrict__ adj,
                                   const CapT *__restrict__ cap0, const int *slots, int k, int dec,
                                   unsigned long long seed, uint8_t *taken, long long *ou,
                                   long long *ov, long long *oc) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    const int i = slots[j];
    taken[i] = 1;
    const long long old = (long long)cap0[i];
    const unsigned long long h = smix_s(seed ^ 0xD1B54A32D192ED03ull ^ smix_s((unsigned long long)i + 1));
    int a = 0, b = n;  // row of slot i
    while (b - a > 1) {
      const int mid = (a + b) >> 1;
      if (off[mid] <= i) a = mid;
      else b = mid;
    }
    ou[j] = a;
    ov[j] = adj[i];
    oc[j] = dec ? (long long)(h % (unsigned long long)old)
                : old + 1 + (long long)(h % (unsigned long long)(old + 10));
  }
}

cudaError_t sample_batch(const GraphObj &g, int s, int t, long long k_dec, long long k_inc,
                         unsigned long long seed, double bias, long long *us, long long *vs,
                         long long *caps, long long *got) {
  const Topology &T = *g.topo;
  cudaStream_t st = T.stream;
  *got = 0;
  const long long S = T.S;
  if (S == 0 || k_dec + k_inc == 0) return cudaSuccess;
  int s_lo = 0, s_hi = 0;
  cudaError_t e = cudaMemcpyAsync(&s_lo, T.off + s, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (!e) e = cudaMemcpyAsync(&s_hi, T.off + s + 1, sizeof(int), cudaMemcpyDeviceToHost, st);
  uint8_t *taken = nullptr;
  unsigned long long *acc = nullptr;
  if (!e) e = cudaMalloc(&taken, (size_t)S);
  if (!e) e = cudaMalloc(&acc, sizeof(unsigned long long));
  if (!e) e = cudaMemsetAsync(taken, 0, (size_t)S, st);
  if (!e) e = cudaMemsetAsync(acc, 0, sizeof(unsigned long long), st);
  if (!e) e = cudaStreamSynchronize(st);
  const int grid = grid_for(S, T.num_sms);
  unsigned long long W = 0;
  if (!e) {
    sample_weight_kernel<<<grid, kBlock, 0, st>>>(T.adj, T.orig, S, s_lo, s_hi, t, bias, acc);
    count_launch();
    e = cudaMemcpyAsync(&W, acc, sizeof(W), cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaStreamSynchronize(st);
  }
  long long done = 0;
  for (int kind = 0; kind < 2 && !e; ++kind) {
    const long long want = kind == 0 ? k_dec : k_inc;
    if (want <= 0) continue;
    const int cap = (int)(8 * want + 4096 < S ? 8 * want + 4096 : S);
    unsigned long long *cand = nullptr, *sorted = nullptr;
    int *cnt = nullptr, *d_slots = nullptr;
    long long *d_out = nullptr;
    void *tmp = nullptr;
    e = cudaMalloc(&cand, sizeof(unsigned long long) * cap);
    if (!e) e = cudaMalloc(&sorted, sizeof(unsigned long long) * cap);
    if (!e) e = cudaMalloc(&cnt, sizeof(int));
    double tau = 3.0 * (double)want / (double)(W > 0 ? W : 1) + 1e-12;
    int c = 0;
    for (int it = 0; it < 60 && !e; ++it) {
      e = cudaMemsetAsync(cnt, 0, sizeof(int), st);
      if (T.cap_bytes == 8)
        sample_kernel<long long><<<grid, kBlock, 0, st>>>(
            T.adj, T.orig, (const long long *)g.cap0, taken, S, s_lo, s_hi, t, bias,
            seed * 2 + kind, kind == 0, tau, cap, cand, cnt);
      else
        sample_kernel<int><<<grid, kBlock, 0, st>>>(T.adj, T.orig, (const int *)g.cap0, taken, S,
                                                    s_lo, s_hi, t, bias, seed * 2 + kind,
                                                    kind == 0, tau, cap, cand, cnt);
      count_launch();
      if (!e) e = cudaMemcpyAsync(&c, cnt, sizeof(int), cudaMemcpyDeviceToHost, st);
      if (!e) e = cudaStreamSynchronize(st);
      if (c > cap) tau *= 0.5;                       // too many candidates
      else if (c < want && tau < 1e30) tau *= 4.0;  // too few: widen (or nothing left)
      else break;
      if (c < want && tau >= 1e30) break;
    }
    if (c > cap) c = cap;
    size_t tb = 0;
    if (!e) e = cub::DeviceRadixSort::SortKeys(nullptr, tb, cand, sorted, c, 0, 64, st);
    if (!e) e = cudaMalloc(&tmp, tb > 0 ? tb : 1);
    if (!e) e = cub::DeviceRadixSort::SortKeys(tmp, tb, cand, sorted, c, 0, 64, st);
    std::vector<unsigned long long> h((size_t)c);
    if (!e && c > 0)
      e = cudaMemcpyAsync(h.data(), sorted, sizeof(unsigned long long) * (size_t)c,
                          cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaStreamSynchronize(st);
    const long long take = want < c ? want : c;
    std::vector<int> slots((size_t)(take > 0 ? take : 0));
    for (long long j = 0; j < take; ++j) slots[j] = (int)(h[j] & 0xFFFFFFFFull);
    std::sort(slots.begin(), slots.end());
    if (!e) e = cudaMalloc(&d_slots, sizeof(int) * (size_t)(take > 0 ? take : 1));
    if (!e) e = cudaMalloc(&d_out, sizeof(long long) * 3 * (size_t)(take > 0 ? take : 1));
    if (!e && take > 0) {
      e = cudaMemcpyAsync(d_slots, slots.data(), sizeof(int) * take, cudaMemcpyHostToDevice, st);
      const int eg = grid_for(take, T.num_sms);
      if (T.cap_bytes == 8)
        sample_emit_kernel<long long><<<eg, kBlock, 0, st>>>(
            T.off, T.n, T.adj, (const long long *)g.cap0, d_slots, (int)take, kind == 0,
            seed * 2 + kind, taken, d_out, d_out + take, d_out + 2 * take);
      else
        sample_emit_kernel<int><<<eg, kBlock, 0, st>>>(T.off, T.n, T.adj, (const int *)g.cap0,
                                                       d_slots, (int)take, kind == 0,
                                                       seed * 2 + kind, taken, d_out, d_out + take,
                                                       d_out + 2 * take);
      count_launch();
      if (!e) e = cudaMemcpyAsync(us + done, d_out, sizeof(long long) * take, cudaMemcpyDeviceToHost, st);
      if (!e) e = cudaMemcpyAsync(vs + done, d_out + take, sizeof(long long) * take,
                                  cudaMemcpyDeviceToHost, st);
      if (!e) e = cudaMemcpyAsync(caps + done, d_out + 2 * take, sizeof(long long) * take,
                                  cudaMemcpyDeviceToHost, st);
      if (!e) e = cudaStreamSynchronize(st);
    }
    if (!e) done += take > 0 ? take : 0;
    cudaFree(tmp);
    cudaFree(cand);
    cudaFree(sorted);
    cudaFree(cnt);
    cudaFree(d_slots);
    cudaFree(d_out);
  }
  cudaFree(taken);
  cudaFree(acc);
  *got = done;
  return e;
}

}  // namespace mfx
