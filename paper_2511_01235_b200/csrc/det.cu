// det.cu -- SolverParams(deterministic=True) on the device.
//
// The reference's deterministic mode runs each phase on one worker in
// worklist (vertex-id) order (solver.py:56-58, 70-73), so its whole final
// state -- cf, excess, height -- is reproducible.  Here the global relabel
// is the ordinary device BFS (its heights are unique, hence identical), and
// one round's worklist + push phase + repair phase run as a single-thread
// kernel in exactly the reference's order (kernels.py:19-93, solver.py:
// 204-241).  The resulting states are byte-identical to the reference's
// deterministic runs (tests/golden state_sha), which pins the device
// arithmetic of every push, relabel and repair, not just the flow value.
// It is a parity / tracing mode: the push phase is serial by definition.
#include "engine.h"

namespace mfx {

// active_mask (state.py:62-67)
__device__ __forceinline__ bool det_active(int v, int n, int s, int t, const long long *ex,
                                           const int *h) {
  return v != s && v != t && ex[v] > 0 && h[v] < n;
}

template <typename CapT>
__global__ void det_round_kernel(const int *__restrict__ off, const int *__restrict__ adj,
                                 const int *__restrict__ rev, CapT *cf, long long *ex, int *h,
                                 int *work, int n, int s, int t, int kc, int topology,
                                 Ctrl *ctrl) {
  if (blockIdx.x | threadIdx.x) return;
  // _push_rounds (solver.py:216-222): stop once no vertex is active
  int nw = 0;
  for (int v = 0; v < n; ++v)
    if (det_active(v, n, s, t, ex, h)) work[nw++] = v;
  ctrl->active = nw;
  if (nw == 0) return;
  if (topology) {  // active_worklist, topology mode (solver.py:167-175)
    nw = 0;
    for (int v = 0; v < n; ++v)
      if (v != s && v != t) work[nw++] = v;
  }
  unsigned long long pushes = 0, relabels = 0, repairs = 0;
  // _push_relabel_chunk over the whole worklist (kernels.py:19-67)
  for (int w = 0; w < nw; ++w) {
    const int u = work[w];
    for (int cnt = 0; cnt < kc; ++cnt) {
      const long long e = ex[u];
      if (e <= 0 || h[u] >= n) break;
      int best = -1, bh = n + 1;
      for (int i = off[u]; i < off[u + 1]; ++i)
        if (cf[i] > 0) {
          const int hv = h[adj[i]];
          if (hv < bh) {
            bh = hv;
            best = i;
          }
        }
      if (best < 0) {
        h[u] = n;
        ++relabels;
        break;
      }
      if (h[u] > bh) {
        const long long c = (long long)cf[best];
        const CapT d = (CapT)(e < c ? e : c);
        cf[best] -= d;
        cf[rev[best]] += d;
        ex[u] -= d;
        ex[adj[best]] += d;
        ++pushes;
      } else {
        h[u] = bh + 1 > n ? n : bh + 1;
        ++relabels;
      }
    }
  }
  // _remove_invalid_chunk over the same worklist (kernels.py:70-93)
  for (int w = 0; w < nw; ++w) {
    const int u = work[w];
    const int hu = h[u];
    for (int i = off[u]; i < off[u + 1]; ++i) {
      const int v = adj[i];
      if (cf[i] > 0 && hu > h[v] + 1) {
        const CapT amt = cf[i];
        cf[i] = 0;
        cf[rev[i]] += amt;
        ex[u] -= amt;
        ex[v] += amt;
        ++repairs;
      }
    }
  }
  ctrl->pushes += pushes;
  ctrl->relabels += relabels;
  ctrl->repairs += repairs;
  ctrl->rounds += 1;
  // _RunStats.check_ceiling (solver.py:196-201)
  if (ctrl->pushes + ctrl->relabels > ctrl->ceiling) ctrl->status = 3;
}

cudaError_t launch_det_round(const GraphObj &g, StateObj &st, int kc, int topology) {
  const Topology &T = *g.topo;
  int *work = T.ws.heavy;  // capacity n; the deterministic loop owns the workspace
  st.tl_ok = false;
  if (T.cap_bytes == 8)
    det_round_kernel<long long><<<1, 32, 0, T.stream>>>(T.off, T.adj, T.rev, (long long *)st.cf,
                                                        st.ex, st.h, work, T.n, st.s, st.t, kc,
                                                        topology, st.ctrl);
  else
    det_round_kernel<int><<<1, 32, 0, T.stream>>>(T.off, T.adj, T.rev, (int *)st.cf, st.ex,
                                                  st.h, work, T.n, st.s, st.t, kc, topology,
                                                  st.ctrl);
  count_launch();
  return cudaGetLastError();
}

}  // namespace mfx
