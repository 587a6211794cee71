// api.cu -- the C-ABI (include/mfx.h) over the device engine.
//
// Error text mirrors the reference exceptions word for word (graph.py:48-61,
// dynamic.py:63-88, solver.py:79-84, 196-201, 244-250, 279-281) so the Python
// shim can re-raise the same classes with the same messages.
#include <limits.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <vector>

#include "../../include/mfx.h"
#include "engine.h"

struct mfx_graph {
  mfx::GraphObj g;
};
struct mfx_state {
  mfx::StateObj s;
  mfx::Ctrl *host_ctrl = nullptr;  // pinned mirror for async result download
  long long *host_err = nullptr;   // pinned mirror of the batch error block
  ~mfx_state() {
    if (host_ctrl) cudaFreeHost(host_ctrl);
    if (host_err) cudaFreeHost(host_err);
  }
};

namespace mfx {

thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};
void count_launch(int k) { g_launches += k; }

static int fail(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t _e = (x);                                                                 \
    if (_e != cudaSuccess)                                                                \
      return fail(MFX_CUDA_ERROR, "CUDA error %s at %s:%d: %s", cudaGetErrorName(_e),     \
                  __FILE__, __LINE__, cudaGetErrorString(_e));                            \
  } while (0)

template <typename T>
static void dfree(T *&p);

static std::atomic<unsigned long long> g_cap_ids{1};
static uint64_t next_cap_id() { return g_cap_ids++; }

// every entry point that touches a topology's workspace / stream holds its lock
#define LOCK_TOPO(T) std::lock_guard<std::recursive_mutex> _topo_lock((T).mu)

template <typename T>
static void dfree(T *&p) {
  if (p) cudaFree((void *)p);
  p = nullptr;
}

Workspace::~Workspace() {
  for (int q = 0; q < 2; ++q)
    for (int b = 0; b < NBIN; ++b) dfree(F[q][b]);
  for (int b = 0; b < NBIN; ++b) dfree(R[b]);
  dfree(bases);
  dfree(heavy);
  dfree(mark);
  dfree(bmark);
  dfree(reg);
  dfree(stamp);
  dfree(vbin);
  dfree(rdirty);
  dfree(trace);
  dfree(slot_first);
  dfree(d_batch);
  dfree(d_slot);
  dfree(d_uv);
  dfree(d_err);
  dfree(d_red);
}

Topology::~Topology() {
  cudaSetDevice(device);
  dfree(off);
  dfree(adj);
  dfree(rev);
  dfree(orig);
  ws.~Workspace();
  new (&ws) Workspace();
  for (auto &e : ev)
    if (e) cudaEventDestroy(e);
  if (stream) cudaStreamDestroy(stream);
}

GraphObj::~GraphObj() {
  if (topo) cudaSetDevice(topo->device);
  dfree(cap0);
  dfree(pc);
}

StateObj::~StateObj() {
  if (topo) cudaSetDevice(topo->device);
  dfree(cf);
  dfree(ex);
  dfree(h);
  dfree(ctrl);
  dfree(tl[0]);
  dfree(tl[1]);
}

cudaError_t ensure_workspace(Topology &t) {
  Workspace &w = t.ws;
  if (w.mark) return cudaSuccess;
  size_t n = (size_t)(t.n > 0 ? t.n : 1);
  w.n = t.n;
  {  // work lists: the asynchronous push phase logs every (re-)queued vertex
    size_t rc = 4 * n + 4096;
    w.rcap = rc > (size_t)INT_MAX ? INT_MAX : (int)rc;
  }
  cudaError_t e;
  for (int q = 0; q < 2; ++q)
    for (int b = 0; b < NBIN; ++b)
      if ((e = cudaMalloc(&w.F[q][b], sizeof(int) * n))) return e;
  for (int b = 0; b < NBIN; ++b) {
    if ((e = cudaMalloc(&w.R[b], sizeof(int) * (size_t)w.rcap))) return e;
    // async push consumers wait for slots != -1: lists start (and are reset to) empty
    if ((e = cudaMemsetAsync(w.R[b], 0xFF, sizeof(int) * (size_t)w.rcap, t.stream))) return e;
  }
  if ((e = cudaMalloc(&w.rdirty, sizeof(int) * NBIN))) return e;
  if ((e = cudaMemsetAsync(w.rdirty, 0, sizeof(int) * NBIN, t.stream))) return e;
  if ((e = cudaMalloc(&w.bases, sizeof(int) * n))) return e;
  if ((e = cudaMalloc(&w.heavy, sizeof(int) * n))) return e;
  if ((e = cudaMalloc(&w.stamp, sizeof(unsigned) * 4))) return e;
  if ((e = cudaMemsetAsync(w.stamp, 0, sizeof(unsigned) * 4, t.stream))) return e;
  if ((e = cudaMalloc(&w.slot_first, sizeof(int) * (size_t)(t.S > 0 ? t.S : 1)))) return e;
  if ((e = cudaMemsetAsync(w.slot_first, 0x7f, sizeof(int) * (size_t)(t.S > 0 ? t.S : 1),
                           t.stream)))
    return e;
  if ((e = cudaMalloc(&w.d_err, sizeof(long long) * 8))) return e;
  if ((e = cudaMalloc(&w.d_red, sizeof(unsigned long long) * 64))) return e;
  if (const char *tc = getenv("MFX_TRACE_CAP")) {
    w.trace_cap = atoi(tc);
    if (w.trace_cap > 0 && (e = cudaMalloc(&w.trace, sizeof(unsigned long long) * w.trace_cap)))
      return e;
  }
  if ((e = cudaMalloc(&w.vbin, n))) return e;
  if ((e = launch_vbin(t, w.vbin))) return e;
  if ((e = cudaMalloc(&w.reg, n))) return e;
  if ((e = cudaMalloc(&w.bmark, sizeof(int) * n))) return e;
  if ((e = cudaMemsetAsync(w.bmark, 0, sizeof(int) * n, t.stream))) return e;
  if ((e = cudaMalloc(&w.mark, sizeof(unsigned) * n))) return e;
  return cudaMemsetAsync(w.mark, 0, sizeof(unsigned) * n, t.stream);
}

// Variant choice: graphs with most slots in long rows (R-MAT: 91 % in rows of
// >= 32 slots) gain from 4x the resident warps; grids and roads (short rows,
// long BFS) lose to the spills of the 64-register build.  $MFX_VARIANT = 256 |
// 512 overrides.
static int choose_variant(Topology &t) {
  if (t.variant >= 0) return t.variant;
  int v = 0;
  if (const char *e = getenv("MFX_VARIANT")) {
    v = atoi(e) == 512 ? 1 : 0;
  } else {
    int pm = 0;
    if (long_row_permille(t, &pm) == cudaSuccess && pm >= 500) v = 1;
  }
  t.variant = v;
  return v;
}

cudaError_t launch_solve(const GraphObj &g, StateObj &st, const SolveConfig &cfg, int *launches) {
  if (choose_variant(*g.topo)) {
    // long-row graphs: one push-or-relabel step per visit of a long row
    // (each step rescans the row; R-MAT 20 dynamic 7.6 -> 5.4 ms)
    SolveConfig c = cfg;
    if (c.coop_kc == 0) c.coop_kc = 1;
    if (c.wave_time < 0) c.wave_time = 0;  // (cheap BFS, productive waves: R-MAT static +25 %)
    // long rows are handed to the next epoch from the CTA ring anyway, so the
    // ring adds work without saving barriers (C1 static 2.1 -> 1.8 ms strict)
    if (c.bfs_local < 0) c.bfs_local = 0;
    return v512::launch_solve(g, st, c, launches);
  }
  // short-row graphs: a push phase is cut off once it has run 1.25x the last
  // global relabel's time (C2: 9.0 -> 8.0 ms/batch, static 30 -> 26.5 ms);
  // 0.75x in dynamic solves, whose late rounds bounce a few units of excess
  // (C2 7.2 -> 6.8 ms/batch; static keeps 1.25x: 0.75x costs it 3 %)
  SolveConfig c = cfg;
  if (c.wave_time < 0) c.wave_time = c.dyn_bases && c.what == WHAT_SOLVE && c.strand > 0 ? 6 : 10;
  if (c.bfs_local < 0) c.bfs_local = 128;
  return v256::launch_solve(g, st, c, launches);
}

cudaError_t launch_pp_setup(const GraphObj &g, StateObj &st, bool crossing, const long long *gate) {
  if (choose_variant(*g.topo)) return v512::launch_pp_setup(g, st, crossing, gate);
  return v256::launch_pp_setup(g, st, crossing, gate);
}

cudaError_t ensure_batch_capacity(Topology &t, int64_t k) {
  Workspace &w = t.ws;
  if (k <= w.kcap && w.d_batch) return cudaSuccess;
  int64_t cap = k > 1024 ? k : 1024;
  dfree(w.d_batch);
  dfree(w.d_slot);
  dfree(w.d_uv);
  cudaError_t e;
  if ((e = cudaMalloc(&w.d_batch, sizeof(int64_t) * 3 * (size_t)cap))) return e;
  if ((e = cudaMalloc(&w.d_slot, sizeof(int) * (size_t)cap))) return e;
  if ((e = cudaMalloc(&w.d_uv, sizeof(int) * 2 * (size_t)cap))) return e;
  w.kcap = cap;
  return cudaSuccess;
}

}  // namespace mfx

using namespace mfx;

// SolverParams(deterministic=True): each round = the device global relabel
// (static: bases {t}, nothing forbidden; dynamic: {t} U deficient, s
// forbidden) followed by the serial round kernel of det.cu; then the usual
// finalize for flow and cut.  Host-stepped: one sync per round.
static int det_rounds(const GraphObj &g, mfx_state *st, SolveConfig cfg, bool dynamic,
                      int *launches) {
  cfg.strand = 0;
  Topology &T = *g.topo;
  StateObj &s = st->s;
  cfg.dyn_bases = dynamic ? 1 : 0;
  cfg.forbidden = dynamic ? s.s : -1;
  cfg.what = WHAT_BFS;
  const double tmo = cfg.timeout_s;
  cudaEvent_t start = T.ev[1];
  for (int round = 0;; ++round) {
    cfg.reset_counters = round == 0;
    CK(launch_solve(g, s, cfg, launches));
    CK(launch_det_round(g, s, cfg.kc, cfg.topology));
    if (launches) *launches += 1;
    CK(cudaMemcpyAsync(st->host_ctrl, s.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, T.stream));
    CK(cudaStreamSynchronize(T.stream));
    const Ctrl &c = *st->host_ctrl;
    if (c.status == 3 || c.status == 6 || c.active == 0) break;
    float ms = 0;
    CK(cudaEventRecord(T.ev[2], T.stream));
    CK(cudaEventSynchronize(T.ev[2]));
    cudaEventElapsedTime(&ms, start, T.ev[2]);
    if (ms > tmo * 1e3) {
      st->host_ctrl->status = 6;
      CK(cudaMemcpyAsync(&s.ctrl->status, &st->host_ctrl->status, sizeof(int),
                         cudaMemcpyHostToDevice, T.stream));
      break;
    }
  }
  if (st->host_ctrl->status == 3 || st->host_ctrl->status == 6) {
    int status = st->host_ctrl->status;  // (the finalize launch would clear it)
    CK(cudaMemcpyAsync(&s.ctrl->status, &status, sizeof(int), cudaMemcpyHostToDevice, T.stream));
    return MFX_OK;
  }
  cfg.what = WHAT_FINAL;
  cfg.reset_counters = false;
  CK(launch_solve(g, s, cfg, launches));
  return MFX_OK;
}

// A state whose residuals were last consistent with other capacity contents
// (set_cap0, or a batch applied through another state / graph copy): the
// reference recomputes excess from max(0, cap0 - cf) on every solve_dynamic
// (dynamic.py:114-116) and reads cf[rev] directly.  Here the BFS reads the
// reverse residual as pc - cf, so the pair sums must still hold: if they do,
// the excess is rebuilt in full before the next use; if not, the state no
// longer describes a flow on this graph and the call is rejected.
static int sync_caps(const GraphObj &g, StateObj &st) {
  if (st.cap_id == g.cap_id) return MFX_OK;
  Topology &T = *g.topo;
  CK(ensure_workspace(T));
  unsigned long long out[2];
  CK(launch_pair_check(g, st, T.ws.d_red));
  CK(cudaMemcpyAsync(out, T.ws.d_red, sizeof(out), cudaMemcpyDeviceToHost, T.stream));
  CK(cudaStreamSynchronize(T.stream));
  if (out[0])
    return fail(MFX_SOLVER_ERROR,
                "state residuals do not match the graph's capacities (%llu slot pair(s) "
                "violate residual-sum conservation, first slot %llu); the capacities changed "
                "after this state was solved -- start from init_residuals",
                out[0], out[1]);
  st.excess_consistent = false;
  st.terminated_known = false;
  st.cap_id = g.cap_id;
  return MFX_OK;
}


// ---------------------------------------------------------------------------
static int make_topology(int device, std::shared_ptr<Topology> &topo) {
  int count = 0;
  CK(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count)
    return fail(MFX_VALUE_ERROR, "device %d out of range [0, %d)", device, count);
  CK(cudaSetDevice(device));
  topo = std::make_shared<Topology>();
  topo->device = device;
  CK(cudaStreamCreateWithFlags(&topo->stream, cudaStreamNonBlocking));
  for (auto &e : topo->ev) CK(cudaEventCreate(&e));
  CK(cudaDeviceGetAttribute(&topo->num_sms, cudaDevAttrMultiProcessorCount, device));
  return MFX_OK;
}

// Choose the residual width and materialise cap0 / pair sums from int64 cap0.
static int finish_graph(mfx_graph *G, int64_t *d_cap0_64, int force_wide) {
  Topology &T = *G->g.topo;
  unsigned long long *d_mx = nullptr, mx = 0;
  CK(cudaMalloc(&d_mx, sizeof(unsigned long long)));
  CK(pair_max_int64(T, d_cap0_64, d_mx));
  CK(cudaMemcpyAsync(&mx, d_mx, sizeof(mx), cudaMemcpyDeviceToHost, T.stream));
  CK(cudaStreamSynchronize(T.stream));
  cudaFree(d_mx);
  T.cap_bytes = (!force_wide && mx < (1ull << 31)) ? 4 : 8;
  size_t S = (size_t)(T.S > 0 ? T.S : 1);
  CK(cudaMalloc(&G->g.cap0, S * T.cap_bytes));
  CK(cudaMalloc(&G->g.pc, S * T.cap_bytes));
  CK(launch_convert_cap(d_cap0_64, G->g.cap0, T.cap_bytes, T.S, T.stream));
  CK(launch_refresh_pc(G->g));
  G->g.cap_id = next_cap_id();
  CK(cudaStreamSynchronize(T.stream));
  CK(ensure_workspace(T));
  CK(cudaStreamSynchronize(T.stream));
  return MFX_OK;
}

static int build_common(int64_t n, int64_t m, const int64_t *d_us, const int64_t *d_vs,
                        const int64_t *d_caps, const int64_t *h_us, const int64_t *h_vs,
                        const int64_t *h_caps, int device, int force_wide, mfx_graph **out) {
  *out = nullptr;
  if (n <= 0) return fail(MFX_GRAPH_ERROR, "vertex count must be positive, got %lld", (long long)n);
  std::shared_ptr<Topology> topo;
  int rc = make_topology(device, topo);
  if (rc) return rc;
  int64_t err[2];
  int64_t *d_cap0 = nullptr;
  CK(build_bicsr_device(n, m, d_us, d_vs, d_caps, *topo, &d_cap0, err, nullptr));
  if (err[0]) {
    if (d_cap0) cudaFree(d_cap0);
    long long i = err[1];
    auto val = [&](const int64_t *h, const int64_t *d) -> long long {
      if (h) return h[i];
      long long v = 0;
      cudaMemcpy(&v, d + i, sizeof(v), cudaMemcpyDeviceToHost);
      return v;
    };
    switch (err[0]) {
      case 1: return fail(MFX_GRAPH_ERROR, "vertex count must be positive, got %lld", (long long)n);
      case 2:
        return fail(MFX_GRAPH_ERROR, "edge %lld: source vertex %lld out of range [0, %lld)", i,
                    val(h_us, d_us), (long long)n);
      case 3:
        return fail(MFX_GRAPH_ERROR, "edge %lld: target vertex %lld out of range [0, %lld)", i,
                    val(h_vs, d_vs), (long long)n);
      case 4:
        return fail(MFX_GRAPH_ERROR, "edge %lld: negative capacity %lld", i, val(h_caps, d_caps));
      default:
        return fail(MFX_VALUE_ERROR, "graph exceeds the int32 slot layout of one device");
    }
  }
  mfx_graph *G = new mfx_graph();
  G->g.topo = topo;
  rc = finish_graph(G, d_cap0, force_wide);
  cudaFree(d_cap0);
  if (rc) {
    delete G;
    return rc;
  }
  *out = G;
  return MFX_OK;
}

struct Staged {
  void *p = nullptr;
  ~Staged() {
    if (p) cudaFree(p);
  }
};

extern "C" {

int mfx_version(void) { return 1; }
const char *mfx_last_error(void) { return g_last_error.c_str(); }
int mfx_device_count(int *count) {
  CK(cudaGetDeviceCount(count));
  return MFX_OK;
}
int64_t mfx_launch_count(void) { return g_launches.load(); }

int mfx_graph_build(int64_t n, int64_t m, const int64_t *us, const int64_t *vs,
                    const int64_t *caps, int device, int force_wide, mfx_graph **out) {
  if (n <= 0) return fail(MFX_GRAPH_ERROR, "vertex count must be positive, got %lld", (long long)n);
  CK(cudaSetDevice(device));
  Staged buf;
  size_t M = (size_t)(m > 0 ? m : 1);
  CK(cudaMalloc(&buf.p, 3 * M * sizeof(int64_t)));
  int64_t *d = (int64_t *)buf.p;
  if (m > 0) {
    CK(cudaMemcpy(d, us, m * sizeof(int64_t), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d + M, vs, m * sizeof(int64_t), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d + 2 * M, caps, m * sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  return build_common(n, m, d, d + M, d + 2 * M, us, vs, caps, device, force_wide, out);
}

int mfx_graph_build_device(int64_t n, int64_t m, const int64_t *d_us, const int64_t *d_vs,
                           const int64_t *d_caps, int device, int force_wide, mfx_graph **out) {
  return build_common(n, m, d_us, d_vs, d_caps, nullptr, nullptr, nullptr, device, force_wide, out);
}

int mfx_graph_from_bicsr(int64_t n, int64_t S, const int64_t *offsets, const int64_t *adj,
                         const int64_t *rev, const int64_t *cap0, const uint8_t *is_original,
                         int device, int force_wide, mfx_graph **out) {
  *out = nullptr;
  if (n <= 0) return fail(MFX_GRAPH_ERROR, "vertex count must be positive, got %lld", (long long)n);
  if (S >= INT_MAX) return fail(MFX_VALUE_ERROR, "graph exceeds the int32 slot layout of one device");
  std::shared_ptr<Topology> topo;
  int rc = make_topology(device, topo);
  if (rc) return rc;
  size_t SS = (size_t)(S > 0 ? S : 1);
  Staged b64, borig;
  CK(cudaMalloc(&b64.p, sizeof(int64_t) * ((size_t)n + 1 + 3 * SS)));
  CK(cudaMalloc(&borig.p, SS));
  int64_t *d_off = (int64_t *)b64.p, *d_adj = d_off + n + 1, *d_rev = d_adj + SS,
          *d_cap = d_rev + SS;
  CK(cudaMemcpy(d_off, offsets, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
  if (S > 0) {
    CK(cudaMemcpy(d_adj, adj, sizeof(int64_t) * S, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_rev, rev, sizeof(int64_t) * S, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_cap, cap0, sizeof(int64_t) * S, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(borig.p, is_original, S, cudaMemcpyHostToDevice));
  }
  CK(topology_from_bicsr(n, S, d_off, d_adj, d_rev, (const uint8_t *)borig.p, *topo));
  long long mo = 0;
  for (int64_t i = 0; i < S; ++i) mo += is_original[i] != 0;
  topo->m_original = (int)mo;
  mfx_graph *G = new mfx_graph();
  G->g.topo = topo;
  rc = finish_graph(G, d_cap, force_wide);
  if (rc) {
    delete G;
    return rc;
  }
  *out = G;
  return MFX_OK;
}

int mfx_graph_info_get(const mfx_graph *g, mfx_graph_info *info) {
  const Topology &T = *g->g.topo;
  info->n = T.n;
  info->S = T.S;
  info->m_original = T.m_original;
  info->self_loops_dropped = T.diag[0];
  info->parallel_edges_merged = T.diag[1];
  info->reverse_stubs_added = T.diag[2];
  info->cap_bytes = T.cap_bytes;
  info->device = T.device;
  return MFX_OK;
}

static int widen_download_i32(const int *d, int64_t *h, size_t cnt, cudaStream_t s) {
  if (!h || cnt == 0) return MFX_OK;
  std::vector<int> tmp(cnt);
  CK(cudaMemcpyAsync(tmp.data(), d, sizeof(int) * cnt, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (size_t i = 0; i < cnt; ++i) h[i] = tmp[i];
  return MFX_OK;
}

static int download_cap(const void *d, int cap_bytes, int64_t *h, size_t cnt, cudaStream_t s) {
  if (!h || cnt == 0) return MFX_OK;
  if (cap_bytes == 8) {
    CK(cudaMemcpyAsync(h, d, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return MFX_OK;
  }
  return widen_download_i32((const int *)d, h, cnt, s);
}

int mfx_graph_download(const mfx_graph *g, int64_t *offsets, int64_t *adj, int64_t *src,
                       int64_t *rev, int64_t *cap0, uint8_t *is_original) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  int rc;
  if ((rc = widen_download_i32(T.off, offsets, (size_t)T.n + 1, T.stream))) return rc;
  if ((rc = widen_download_i32(T.adj, adj, (size_t)T.S, T.stream))) return rc;
  if ((rc = widen_download_i32(T.rev, rev, (size_t)T.S, T.stream))) return rc;
  if ((rc = download_cap(g->g.cap0, T.cap_bytes, cap0, (size_t)T.S, T.stream))) return rc;
  if (is_original && T.S > 0) {
    CK(cudaMemcpyAsync(is_original, T.orig, (size_t)T.S, cudaMemcpyDeviceToHost, T.stream));
    CK(cudaStreamSynchronize(T.stream));
  }
  if (src && T.S > 0) {
    Staged b;
    CK(cudaMalloc(&b.p, sizeof(int64_t) * (size_t)T.S));
    CK(download_src(T, (int64_t *)b.p));
    CK(cudaMemcpyAsync(src, b.p, sizeof(int64_t) * (size_t)T.S, cudaMemcpyDeviceToHost, T.stream));
    CK(cudaStreamSynchronize(T.stream));
  }
  return MFX_OK;
}

int mfx_graph_copy(const mfx_graph *g, mfx_graph **out) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  mfx_graph *G = new mfx_graph();
  G->g.topo = g->g.topo;
  G->g.cap_id = g->g.cap_id;  // same contents
  size_t bytes = (size_t)(T.S > 0 ? T.S : 1) * T.cap_bytes;
  cudaError_t e = cudaMalloc(&G->g.cap0, bytes);
  if (!e) e = cudaMalloc(&G->g.pc, bytes);
  if (!e) e = cudaMemcpyAsync(G->g.cap0, g->g.cap0, bytes, cudaMemcpyDeviceToDevice, T.stream);
  if (!e) e = cudaMemcpyAsync(G->g.pc, g->g.pc, bytes, cudaMemcpyDeviceToDevice, T.stream);
  if (!e) e = cudaStreamSynchronize(T.stream);
  if (e) {
    delete G;
    CK(e);
  }
  *out = G;
  return MFX_OK;
}

int mfx_graph_set_cap0(mfx_graph *g, const int64_t *cap0) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  if (T.S == 0) return MFX_OK;
  CK(ensure_workspace(T));
  Staged b;
  CK(cudaMalloc(&b.p, sizeof(int64_t) * (size_t)T.S));
  CK(cudaMemcpy(b.p, cap0, sizeof(int64_t) * (size_t)T.S, cudaMemcpyHostToDevice));
  // negative capacities, and (int32 storage) pair sums that reach 2^31
  unsigned long long bad[2];
  CK(launch_cap_check(T, (const int64_t *)b.p, T.ws.d_red));
  CK(cudaMemcpyAsync(bad, T.ws.d_red, sizeof(bad), cudaMemcpyDeviceToHost, T.stream));
  CK(cudaStreamSynchronize(T.stream));
  if (bad[0] != ~0ull)
    return fail(MFX_GRAPH_ERROR, "edge %llu has negative capacity %lld", bad[0],
                (long long)cap0[bad[0]]);
  if (bad[1] != ~0ull)
    return fail(MFX_VALUE_ERROR,
                "capacity %lld on slot %llu: pair sum overflows the int32 residual storage; "
                "rebuild the graph with wide capacities",
                (long long)cap0[bad[1]], bad[1]);
  CK(launch_convert_cap((const int64_t *)b.p, g->g.cap0, T.cap_bytes, T.S, T.stream));
  CK(launch_refresh_pc(g->g));
  CK(cudaStreamSynchronize(T.stream));
  g->g.cap_id = next_cap_id();  // states solved against the old capacities are now stale
  return MFX_OK;
}

int mfx_edge_indices(const mfx_graph *g, int64_t k, const int64_t *us, const int64_t *vs,
                     int64_t *out) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  if (k <= 0) return MFX_OK;
  CK(ensure_batch_capacity(T, k));
  int64_t *d = T.ws.d_batch;
  CK(cudaMemcpyAsync(d, us, sizeof(int64_t) * k, cudaMemcpyHostToDevice, T.stream));
  CK(cudaMemcpyAsync(d + k, vs, sizeof(int64_t) * k, cudaMemcpyHostToDevice, T.stream));
  CK(launch_edge_indices(g->g, k, d, d + k, d + 2 * k));
  CK(cudaMemcpyAsync(out, d + 2 * k, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, T.stream));
  CK(cudaStreamSynchronize(T.stream));
  return MFX_OK;
}

void mfx_graph_free(mfx_graph *g) { delete g; }

// ---- state -------------------------------------------------------------------
int mfx_state_create(const mfx_graph *g, int64_t source, int64_t sink, mfx_state **out) {
  *out = nullptr;
  const Topology &T = *g->g.topo;
  if (source < 0 || source >= T.n)
    return fail(MFX_VALUE_ERROR, "source %lld out of range [0, %d)", (long long)source, T.n);
  if (sink < 0 || sink >= T.n)
    return fail(MFX_VALUE_ERROR, "sink %lld out of range [0, %d)", (long long)sink, T.n);
  CK(cudaSetDevice(T.device));
  mfx_state *S = new mfx_state();
  StateObj &st = S->s;
  st.topo = g->g.topo;
  st.s = (int)source;
  st.t = (int)sink;
  st.cap_id = g->g.cap_id;
  size_t SS = (size_t)(T.S > 0 ? T.S : 1);
  cudaError_t e = cudaMalloc(&st.cf, SS * T.cap_bytes);
  if (!e) e = cudaMalloc(&st.ex, sizeof(long long) * (size_t)T.n);
  if (!e) e = cudaMalloc(&st.h, sizeof(int) * (size_t)T.n);
  if (!e) e = cudaMalloc(&st.ctrl, sizeof(Ctrl));
  if (!e) e = cudaMemsetAsync(st.ctrl, 0, sizeof(Ctrl), T.stream);
  if (!e) e = cudaHostAlloc(&S->host_ctrl, sizeof(Ctrl), cudaHostAllocDefault);
  if (!e) e = cudaHostAlloc(&S->host_err, sizeof(long long) * 8, cudaHostAllocDefault);
  if (!e) e = launch_init_state(g->g, st);
  if (!e) e = cudaStreamSynchronize(T.stream);
  if (e) {
    delete S;
    CK(e);
  }
  *out = S;
  return MFX_OK;
}

int mfx_state_copy(const mfx_state *st, mfx_state **out) {
  Topology &T = *st->s.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  mfx_state *S = new mfx_state();
  StateObj &d = S->s;
  d.topo = st->s.topo;
  d.s = st->s.s;
  d.t = st->s.t;
  d.excess_consistent = st->s.excess_consistent;
  d.terminated_known = st->s.terminated_known;
  d.cap_id = st->s.cap_id;
  size_t cfb = (size_t)(T.S > 0 ? T.S : 1) * T.cap_bytes;
  cudaError_t e = cudaMalloc(&d.cf, cfb);
  if (!e) e = cudaMalloc(&d.ex, sizeof(long long) * (size_t)T.n);
  if (!e) e = cudaMalloc(&d.h, sizeof(int) * (size_t)T.n);
  if (!e) e = cudaMalloc(&d.ctrl, sizeof(Ctrl));
  if (!e) e = cudaHostAlloc(&S->host_ctrl, sizeof(Ctrl), cudaHostAllocDefault);
  if (!e) e = cudaHostAlloc(&S->host_err, sizeof(long long) * 8, cudaHostAllocDefault);
  if (!e) e = cudaMemcpyAsync(d.cf, st->s.cf, cfb, cudaMemcpyDeviceToDevice, T.stream);
  if (!e) e = cudaMemcpyAsync(d.ex, st->s.ex, sizeof(long long) * T.n, cudaMemcpyDeviceToDevice, T.stream);
  if (!e) e = cudaMemcpyAsync(d.h, st->s.h, sizeof(int) * T.n, cudaMemcpyDeviceToDevice, T.stream);
  if (!e) e = cudaMemcpyAsync(d.ctrl, st->s.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToDevice, T.stream);
  // the reached-set lists travel with the control block (a snapshot resumes
  // sparse relabels at once, and its first solve allocates nothing)
  for (int q = 0; q < 2 && !e && st->s.tl[q]; ++q) {
    e = cudaMalloc(&d.tl[q], sizeof(int) * (size_t)T.n);
    if (!e) e = cudaMemcpyAsync(d.tl[q], st->s.tl[q], sizeof(int) * (size_t)T.n,
                                cudaMemcpyDeviceToDevice, T.stream);
  }
  if (!e) d.tl_ok = st->s.tl_ok && d.tl[1] != nullptr;
  if (!e) e = cudaStreamSynchronize(T.stream);
  if (e) {
    delete S;
    CK(e);
  }
  *out = S;
  return MFX_OK;
}

int mfx_state_assign(mfx_state *dst, const mfx_state *src) {
  if (dst->s.topo != src->s.topo)
    return fail(MFX_VALUE_ERROR, "states belong to different graph topologies");
  Topology &T = *src->s.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  size_t cfb = (size_t)(T.S > 0 ? T.S : 1) * T.cap_bytes;
  CK(cudaMemcpyAsync(dst->s.cf, src->s.cf, cfb, cudaMemcpyDeviceToDevice, T.stream));
  CK(cudaMemcpyAsync(dst->s.ex, src->s.ex, sizeof(long long) * T.n, cudaMemcpyDeviceToDevice, T.stream));
  CK(cudaMemcpyAsync(dst->s.h, src->s.h, sizeof(int) * T.n, cudaMemcpyDeviceToDevice, T.stream));
  CK(cudaStreamSynchronize(T.stream));
  dst->s.s = src->s.s;
  dst->s.t = src->s.t;
  dst->s.excess_consistent = src->s.excess_consistent;
  dst->s.terminated_known = src->s.terminated_known;
  dst->s.cap_id = src->s.cap_id;
  dst->s.tl_ok = false;
  return MFX_OK;
}

int mfx_state_upload(mfx_state *st, const int64_t *cf, const int64_t *excess,
                     const int64_t *height) {
  Topology &T = *st->s.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  if (cf && T.S > 0) {
    if (T.cap_bytes == 8) {
      CK(cudaMemcpy(st->s.cf, cf, sizeof(int64_t) * T.S, cudaMemcpyHostToDevice));
    } else {
      std::vector<int> tmp((size_t)T.S);
      for (int64_t i = 0; i < T.S; ++i) {
        if (cf[i] < INT_MIN || cf[i] > INT_MAX)
          return fail(MFX_VALUE_ERROR, "residual %lld does not fit the int32 residual storage",
                      (long long)cf[i]);
        tmp[i] = (int)cf[i];
      }
      CK(cudaMemcpy(st->s.cf, tmp.data(), sizeof(int) * T.S, cudaMemcpyHostToDevice));
    }
  }
  if (excess) CK(cudaMemcpy(st->s.ex, excess, sizeof(int64_t) * T.n, cudaMemcpyHostToDevice));
  if (height) {
    std::vector<int> tmp((size_t)T.n);
    for (int v = 0; v < T.n; ++v) tmp[v] = (int)height[v];
    CK(cudaMemcpy(st->s.h, tmp.data(), sizeof(int) * T.n, cudaMemcpyHostToDevice));
  }
  st->s.excess_consistent = false;
  st->s.terminated_known = false;
  st->s.tl_ok = false;
  st->s.cap_id = 0;  // arbitrary residuals: pair sums are checked at the next use
  return MFX_OK;
}

int mfx_state_download(const mfx_state *st, int64_t *cf, int64_t *excess, int64_t *height) {
  Topology &T = *st->s.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  int rc;
  if ((rc = download_cap(st->s.cf, T.cap_bytes, cf, (size_t)T.S, T.stream))) return rc;
  if (excess) {
    CK(cudaMemcpyAsync(excess, st->s.ex, sizeof(int64_t) * T.n, cudaMemcpyDeviceToHost, T.stream));
    CK(cudaStreamSynchronize(T.stream));
  }
  if ((rc = widen_download_i32(st->s.h, height, (size_t)T.n, T.stream))) return rc;
  return MFX_OK;
}

void mfx_state_free(mfx_state *st) { delete st; }

int mfx_saturate_source(mfx_state *st, const mfx_graph *g) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  CK(launch_saturate(g->g, st->s));
  CK(cudaStreamSynchronize(T.stream));
  st->s.terminated_known = false;
  return MFX_OK;
}

int mfx_mask(const mfx_state *st, int which, uint8_t *out) {
  Topology &T = *st->s.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  Staged b;
  CK(cudaMalloc(&b.p, (size_t)T.n));
  CK(launch_mask(st->s, which, (uint8_t *)b.p));
  CK(cudaMemcpyAsync(out, b.p, (size_t)T.n, cudaMemcpyDeviceToHost, T.stream));
  CK(cudaStreamSynchronize(T.stream));
  return MFX_OK;
}

// ---- solver ------------------------------------------------------------------
static unsigned long long operation_ceiling(long long n, long long m) {
  // n^2 + n*E + 4 n^2 (n + E) (solver.py:37-44), saturated to 64 bits
  long double c = (long double)n * n + (long double)n * m + 4.0L * n * n * (long double)(n + m);
  if (c >= 1.8e19L) return ~0ull;
  unsigned __int128 x = (unsigned __int128)n * n + (unsigned __int128)n * m +
                        (unsigned __int128)4 * n * n * (unsigned __int128)(n + m);
  return (unsigned long long)x;
}

static int resolve_config(const Topology &T, const mfx_params *p, SolveConfig &cfg) {
  mfx_params d{};
  if (!p) p = &d;
  if (p->mode != 0 && p->mode != 1)
    return fail(MFX_VALUE_ERROR, "mode must be one of ('data', 'topology'), got %d", p->mode);
  if (p->kernel_cycles < 0)
    return fail(MFX_VALUE_ERROR, "kernel_cycles must be >= 1 (or 0 for the default)");
  long long kc = p->kernel_cycles;
  if (kc == 0) kc = T.n > 0 ? (T.m_original + (long long)T.n - 1) / T.n : 1;
  if (kc < 1) kc = 1;
  if (kc > INT_MAX) kc = INT_MAX;
  cfg.kc = (int)kc;
  cfg.topology = p->mode;
  cfg.max_waves = p->max_waves;
  cfg.async = p->schedule == 1;
  if (const char *sch = getenv("MFX_SCHEDULE")) cfg.async = sch[0] == 'a';
  if (p->async_budget > 0) cfg.async_budget = p->async_budget;
  cfg.flags = p->flags;
  if (const char *fl = getenv("MFX_FLAGS")) cfg.flags = atoi(fl);
  if (p->bfs_local != 0) cfg.bfs_local = p->bfs_local < 0 ? 0 : p->bfs_local;
  if (const char *bl = getenv("MFX_BFS_LOCAL")) cfg.bfs_local = atoi(bl) < 0 ? 0 : atoi(bl);
  if (p->bfs_local_max > 0) cfg.bfs_local_max = p->bfs_local_max;
  if (const char *bm = getenv("MFX_BFS_LOCAL_MAX")) cfg.bfs_local_max = atoi(bm);
  if (const char *lc = getenv("MFX_LQ_CAP")) cfg.lq_cap = atoi(lc);
  if (const char *ti = getenv("MFX_TAIL_ITEMS")) cfg.tail_items = atoi(ti);
  if (const char *tc = getenv("MFX_TAIL_CAP")) cfg.tail_cap = atoi(tc);
  if (const char *ck = getenv("MFX_COOP_KC")) cfg.coop_kc = atoi(ck);
  if (const char *wm = getenv("MFX_WALK_MAX")) cfg.walk_max = atoi(wm);  // (< 0: off)
  if (const char *wd = getenv("MFX_WALK_DEPTH")) cfg.walk_depth = atoi(wd);
  if (const char *mc = getenv("MFX_MAX_CTAS")) cfg.max_ctas = atoi(mc);
  if (const char *tl = getenv("MFX_TAIL_LOCAL")) cfg.tail_local = atoi(tl);
  if (const char *wt = getenv("MFX_WAVE_TIME")) cfg.wave_time = atoi(wt);
  if (const char *rs = getenv("MFX_RING_SLEEP")) cfg.ring_sleep = atoi(rs);
  cfg.strand = -1;  // auto: on in dynamic solves
  if (const char *sr = getenv("MFX_STRAND")) cfg.strand = atoi(sr);
  if (const char *ee = getenv("MFX_EARLY")) cfg.early = atoi(ee);
  if (const char *tr = getenv("MFX_TRACK")) cfg.track = atoi(tr);
  if (const char *sp = getenv("MFX_SPARSE")) cfg.sparse = atoi(sp);
  if (const char *rp = getenv("MFX_RAMP")) cfg.ramp = atoi(rp) > 0 ? atoi(rp) : 4;
  if (p->wave_mult > 0 || p->wave_add > 0) {
    cfg.wave_mult = p->wave_mult;
    cfg.wave_add = p->wave_add;
  }
  double tmo = 600.0;
  if (const char *env = getenv("MFX_TIMEOUT_S")) tmo = atof(env) > 0 ? atof(env) : tmo;
  cfg.timeout_s = p->timeout_s > 0 ? p->timeout_s : tmo;
  cfg.blocks_per_sm = p->blocks_per_sm;
  cfg.deterministic = p->deterministic != 0;
  cfg.ceiling = operation_ceiling(T.n, T.m_original);
  if (const char *ce = getenv("MFX_CEILING")) cfg.ceiling = strtoull(ce, nullptr, 10);  // tests
  return MFX_OK;
}

static void fill_result(const mfx_state *st, mfx_result *r) {
  const Ctrl &c = *st->host_ctrl;
  r->flow = c.flow;
  r->cut = c.cut;
  r->rounds = (int64_t)c.rounds;
  r->pushes = (int64_t)c.pushes;
  r->relabels = (int64_t)c.relabels;
  r->repairs = (int64_t)c.repairs;
  r->bfs_levels = (int64_t)c.levels;
  r->waves = (int64_t)c.waves;
  r->bytes_alg = (int64_t)c.bytes;
  r->ns_bfs = (double)c.phase_ns[PH_BFS];
  r->ns_push = (double)c.phase_ns[PH_PUSH];
  r->ns_repair = (double)c.phase_ns[PH_REPAIR];
  r->status = c.status;
  r->async_items = (int64_t)c.async_items;
  r->bfs_epochs = (int64_t)c.epochs;
}

static int solve_status(mfx_state *st, mfx_result *r) {
  const Ctrl &c = *st->host_ctrl;
  // the reached-set list is valid iff the launch's last relabel kept it and
  // nothing aborted (an aborted relabel leaves its list partial)
  st->s.tl_ok = c.status == 0 && c.tl_ok != 0;
  if (c.status == 6)
    return fail(MFX_TIMEOUT, "device watchdog expired after %lld rounds", (long long)c.rounds);
  if (c.status == 3)
    return fail(MFX_SOLVER_ERROR,
                "push/relabel count %llu exceeded the termination ceiling %llu; solver state is "
                "likely corrupt",
                c.pushes + c.relabels, c.ceiling);
  if (r->flow != r->cut)
    return fail(MFX_SOLVER_ERROR, "flow %lld does not match cut capacity %lld", (long long)r->flow,
                (long long)r->cut);
  return MFX_OK;
}

static float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int mfx_global_relabel(mfx_state *st, const mfx_graph *g, int dynamic_bases, int64_t *reached) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  int rc0 = sync_caps(g->g, st->s);
  if (rc0) return rc0;
  SolveConfig cfg;
  cfg.what = WHAT_BFS;
  if (const char *fl = getenv("MFX_FLAGS")) cfg.flags = atoi(fl);  // (tests: forced retry)
  cfg.dyn_bases = dynamic_bases ? 1 : 0;
  cfg.forbidden = dynamic_bases ? st->s.s : -1;
  CK(launch_solve(g->g, st->s, cfg, nullptr));
  CK(cudaMemcpyAsync(st->host_ctrl, st->s.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, T.stream));
  CK(cudaStreamSynchronize(T.stream));
  if (reached) *reached = st->host_ctrl->reached;
  st->s.terminated_known = false;
  return MFX_OK;
}

int mfx_solve_static(const mfx_graph *g, mfx_state *st, const mfx_params *p, mfx_result *r) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  memset(r, 0, sizeof(*r));
  if (st->s.s == st->s.t) return fail(MFX_VALUE_ERROR, "source and sink must differ");
  if (st->s.topo != g->g.topo) return fail(MFX_VALUE_ERROR, "state belongs to another graph");
  SolveConfig cfg;
  int rc = resolve_config(T, p, cfg);
  if (rc) return rc;
  CK(cudaSetDevice(T.device));
  cfg.what = WHAT_SOLVE;
  cfg.dyn_bases = 1;
  cfg.forbidden = st->s.s;
  int launches = 0;
  CK(cudaEventRecord(T.ev[0], T.stream));
  CK(launch_init_state(g->g, st->s));
  CK(launch_saturate(g->g, st->s));
  st->s.cap_id = g->g.cap_id;
  st->s.excess_consistent = true;
  launches += 1;
  CK(cudaEventRecord(T.ev[1], T.stream));
  if (cfg.deterministic) {
    if ((rc = det_rounds(g->g, st, cfg, false, &launches))) return rc;
  } else {
    CK(launch_solve(g->g, st->s, cfg, &launches));
  }
  CK(cudaEventRecord(T.ev[2], T.stream));
  CK(cudaMemcpyAsync(st->host_ctrl, st->s.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, T.stream));
  CK(cudaEventRecord(T.ev[3], T.stream));
  CK(cudaEventSynchronize(T.ev[3]));
  CK(cudaGetLastError());
  fill_result(st, r);
  r->ms_update = ev_ms(T.ev[0], T.ev[1]);
  r->ms_solve = ev_ms(T.ev[1], T.ev[2]);
  r->ms_total = ev_ms(T.ev[0], T.ev[3]);
  r->launches = launches;
  st->s.terminated_known = r->status == 0;
  return solve_status(st, r);
}

static int batch_error(const long long *err, int64_t k, const int64_t *h_us, const int64_t *h_vs,
                       const int64_t *h_caps, const int64_t *d_us, const int64_t *d_vs,
                       const int64_t *d_caps) {
  auto get = [&](const int64_t *h, const int64_t *d, long long j) -> long long {
    if (h) return h[j];
    long long v = 0;
    cudaMemcpy(&v, d + j, sizeof(v), cudaMemcpyDeviceToHost);
    return v;
  };
  (void)k;
  if (err[0] != LLONG_MAX) {
    long long j = err[0];
    return fail(MFX_BATCH_ERROR, "update %lld (%lld->%lld): negative capacity %lld", j,
                get(h_us, d_us, j), get(h_vs, d_vs, j), get(h_caps, d_caps, j));
  }
  if (err[1] != LLONG_MAX) {
    long long j = err[1];
    return fail(MFX_BATCH_ERROR,
                "update %lld targets edge %lld->%lld which is not an edge of the original graph",
                j, get(h_us, d_us, j), get(h_vs, d_vs, j));
  }
  if (err[3] != LLONG_MAX) {
    long long j = err[3];
    return fail(MFX_BATCH_ERROR, "duplicate update for edge %lld->%lld", get(h_us, d_us, j),
                get(h_vs, d_vs, j));
  }
  if (err[4] != LLONG_MAX) {
    long long j = err[4];
    return fail(MFX_VALUE_ERROR,
                "update %lld (%lld->%lld): capacity %lld overflows the int32 residual storage; "
                "rebuild the graph with wide capacities",
                j, get(h_us, d_us, j), get(h_vs, d_vs, j), get(h_caps, d_caps, j));
  }
  return MFX_OK;
}

static int require_terminated(mfx_state *st, const char *what) {
  if (st->s.terminated_known) return MFX_OK;
  Topology &T = *st->s.topo;
  CK(ensure_workspace(T));
  unsigned long long cnt = 0;
  CK(launch_count_active(st->s, T.ws.d_red));
  CK(cudaMemcpyAsync(&cnt, T.ws.d_red, sizeof(cnt), cudaMemcpyDeviceToHost, T.stream));
  CK(cudaStreamSynchronize(T.stream));
  if (cnt) return fail(MFX_SOLVER_ERROR, "%s requires a terminated solver state", what);
  return MFX_OK;
}

static int solve_dynamic_common(mfx_graph *g, mfx_state *st, int64_t k, const int64_t *h_us,
                                const int64_t *h_vs, const int64_t *h_caps, const int64_t *d_us,
                                const int64_t *d_vs, const int64_t *d_caps, const mfx_params *p,
                                mfx_result *r) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  memset(r, 0, sizeof(*r));
  if (st->s.topo != g->g.topo) return fail(MFX_VALUE_ERROR, "state belongs to another graph");
  SolveConfig cfg;
  int rc = resolve_config(T, p, cfg);
  if (rc) return rc;
  CK(cudaSetDevice(T.device));
  if ((rc = sync_caps(g->g, st->s))) return rc;
  if ((rc = require_terminated(st, "solve_dynamic"))) return rc;
  CK(ensure_batch_capacity(T, k));
  int launches = 0;
  CK(cudaEventRecord(T.ev[0], T.stream));
  if (h_us && k > 0) {  // host batch: stage it (part of the timed end-to-end call)
    int64_t *d = T.ws.d_batch;
    CK(cudaMemcpyAsync(d, h_us, sizeof(int64_t) * k, cudaMemcpyHostToDevice, T.stream));
    CK(cudaMemcpyAsync(d + k, h_vs, sizeof(int64_t) * k, cudaMemcpyHostToDevice, T.stream));
    CK(cudaMemcpyAsync(d + 2 * k, h_caps, sizeof(int64_t) * k, cudaMemcpyHostToDevice, T.stream));
    d_us = d;
    d_vs = d + k;
    d_caps = d + 2 * k;
  }
  if (!st->s.excess_consistent) {  // uploaded state: full recompute_excess first
    CK(launch_recompute_excess(g->g, st->s));
    ++launches;
  }
  CK(launch_batch(g->g, &st->s, k, d_us, d_vs, d_caps, true, true, &launches));
  CK(launch_saturate(g->g, st->s, T.ws.d_err));
  ++launches;
  CK(cudaEventRecord(T.ev[1], T.stream));
  cfg.what = WHAT_SOLVE;
  cfg.dyn_bases = 1;
  cfg.forbidden = st->s.s;
  cfg.gate = T.ws.d_err;
  cfg.batch_k = k;
  // the excess walk ($MFX_WALK_MAX / $MFX_WALK_DEPTH) is off by default since
  // the early-exit relabel and the stranded-excess rule: C4 16.5 (off) vs
  // 19.3 ms/batch (4096 / 1024)
  if (cfg.walk_max > 0 && cfg.walk_depth == 0) cfg.walk_depth = 1024;
  if (cfg.strand < 0) cfg.strand = 1;
  if (cfg.deterministic) {
    // (a failed batch leaves the state untouched: skip the rounds)
    CK(cudaMemcpyAsync(st->host_err, T.ws.d_err, sizeof(long long) * 8, cudaMemcpyDeviceToHost,
                       T.stream));
    CK(cudaStreamSynchronize(T.stream));
    if ((rc = batch_error(st->host_err, k, h_us, h_vs, h_caps, d_us, d_vs, d_caps))) return rc;
    if ((rc = det_rounds(g->g, st, cfg, true, &launches))) return rc;
  } else {
    CK(launch_solve(g->g, st->s, cfg, &launches));
  }
  CK(cudaEventRecord(T.ev[2], T.stream));
  CK(cudaMemcpyAsync(st->host_ctrl, st->s.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, T.stream));
  CK(cudaMemcpyAsync(st->host_err, T.ws.d_err, sizeof(long long) * 8, cudaMemcpyDeviceToHost,
                     T.stream));
  CK(cudaEventRecord(T.ev[3], T.stream));
  CK(cudaEventSynchronize(T.ev[3]));
  CK(cudaGetLastError());
  if ((rc = batch_error(st->host_err, k, h_us, h_vs, h_caps, d_us, d_vs, d_caps))) {
    st->s.tl_ok = false;  // (the kernel skipped: conservative, the next relabel seeds in full)
    return rc;
  }
  if (k > 0) g->g.cap_id = next_cap_id();
  st->s.cap_id = g->g.cap_id;
  fill_result(st, r);
  r->updates = k;
  r->ms_update = ev_ms(T.ev[0], T.ev[1]);
  r->ms_solve = ev_ms(T.ev[1], T.ev[2]);
  r->ms_total = ev_ms(T.ev[0], T.ev[3]);
  r->launches = launches;
  st->s.excess_consistent = true;
  st->s.terminated_known = r->status == 0;
  return solve_status(st, r);
}

int mfx_solve_dynamic(mfx_graph *g, mfx_state *st, int64_t k, const int64_t *us, const int64_t *vs,
                      const int64_t *new_caps, const mfx_params *p, mfx_result *r) {
  return solve_dynamic_common(g, st, k, us, vs, new_caps, nullptr, nullptr, nullptr, p, r);
}

int mfx_solve_dynamic_device(mfx_graph *g, mfx_state *st, int64_t k, const int64_t *d_us,
                             const int64_t *d_vs, const int64_t *d_caps, const mfx_params *p,
                             mfx_result *r) {
  return solve_dynamic_common(g, st, k, nullptr, nullptr, nullptr, d_us, d_vs, d_caps, p, r);
}

// solve_dynamic_pushpull (dynamic.py:292-377): regions from the prior cut,
// batch pre-phase, A->B saturation, the two region-restricted pipelines as
// one device round loop, then ordinary dynamic rounds for what crosses.
static int pushpull_common(mfx_graph *g, mfx_state *st, int64_t k, const int64_t *us,
                           const int64_t *vs, const int64_t *new_caps, const mfx_params *p,
                           mfx_result *r, bool final_pass) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  memset(r, 0, sizeof(*r));
  if (st->s.topo != g->g.topo) return fail(MFX_VALUE_ERROR, "state belongs to another graph");
  SolveConfig cfg;
  int rc = resolve_config(T, p, cfg);
  if (rc) return rc;
  // every pipeline and the final pass check against 2x the ceiling
  // (dynamic.py:322); the device counters accumulate over all of them
  cfg.ceiling = cfg.ceiling > (~0ull >> 1) ? ~0ull : 2 * cfg.ceiling;
  CK(cudaSetDevice(T.device));
  if ((rc = sync_caps(g->g, st->s))) return rc;
  if ((rc = require_terminated(st, "solve_dynamic_pushpull"))) return rc;
  {  // the prior heights must carry a cut certificate: s in A, t in B
    int hs = 0, ht = 0;
    CK(cudaMemcpy(&hs, st->s.h + st->s.s, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&ht, st->s.h + st->s.t, sizeof(int), cudaMemcpyDeviceToHost));
    if (hs != T.n || ht == T.n)
      return fail(MFX_SOLVER_ERROR,
                  "prior state carries no usable cut certificate; run a full solve first");
  }
  CK(ensure_batch_capacity(T, k));
  int launches = 0;
  CK(cudaEventRecord(T.ev[0], T.stream));
  const int64_t *d_us = nullptr, *d_vs = nullptr, *d_caps = nullptr;
  if (k > 0) {
    int64_t *d = T.ws.d_batch;
    CK(cudaMemcpyAsync(d, us, sizeof(int64_t) * k, cudaMemcpyHostToDevice, T.stream));
    CK(cudaMemcpyAsync(d + k, vs, sizeof(int64_t) * k, cudaMemcpyHostToDevice, T.stream));
    CK(cudaMemcpyAsync(d + 2 * k, new_caps, sizeof(int64_t) * k, cudaMemcpyHostToDevice, T.stream));
    d_us = d;
    d_vs = d + k;
    d_caps = d + 2 * k;
  }
  CK(launch_pp_setup(g->g, st->s, false, nullptr));  // regions before the batch
  ++launches;
  if (!st->s.excess_consistent) {
    CK(launch_recompute_excess(g->g, st->s));
    ++launches;
  }
  CK(launch_batch(g->g, &st->s, k, d_us, d_vs, d_caps, true, true, &launches));
  CK(launch_saturate(g->g, st->s, T.ws.d_err));
  CK(launch_pp_setup(g->g, st->s, true, T.ws.d_err));  // _saturate_crossing
  launches += 2;
  CK(cudaEventRecord(T.ev[1], T.stream));
  cfg.what = WHAT_SOLVE;
  cfg.gate = T.ws.d_err;
  cfg.pushpull = true;
  // the region-restricted relabels start from wide base sets (every overflowing
  // A-side vertex); the CTA rings still pay there (C2: 126 -> 10 epochs/batch)
  const int blm = cfg.bfs_local_max;
  if (!(p && p->bfs_local_max > 0) && !getenv("MFX_BFS_LOCAL_MAX")) cfg.bfs_local_max = 1 << 20;
  CK(launch_solve(g->g, st->s, cfg, &launches));
  cfg.bfs_local_max = blm;
  if (final_pass) {
    cfg.pushpull = false;  // final pass: overflow on the B side meets deficits on the A side
    cfg.reset_counters = false;
    cfg.dyn_bases = 1;
    cfg.forbidden = st->s.s;
    if (cfg.strand < 0) cfg.strand = 1;  // (the dynamic solve's stop / demand-covered rules)
    CK(launch_solve(g->g, st->s, cfg, &launches));
  }
  CK(cudaEventRecord(T.ev[2], T.stream));
  CK(cudaMemcpyAsync(st->host_ctrl, st->s.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, T.stream));
  CK(cudaMemcpyAsync(st->host_err, T.ws.d_err, sizeof(long long) * 8, cudaMemcpyDeviceToHost,
                     T.stream));
  CK(cudaEventRecord(T.ev[3], T.stream));
  CK(cudaEventSynchronize(T.ev[3]));
  CK(cudaGetLastError());
  if ((rc = batch_error(st->host_err, k, us, vs, new_caps, d_us, d_vs, d_caps))) return rc;
  if (k > 0) g->g.cap_id = next_cap_id();
  st->s.cap_id = g->g.cap_id;
  fill_result(st, r);
  r->updates = k;
  r->ms_update = ev_ms(T.ev[0], T.ev[1]);
  r->ms_solve = ev_ms(T.ev[1], T.ev[2]);
  r->ms_total = ev_ms(T.ev[0], T.ev[3]);
  r->launches = launches;
  st->s.excess_consistent = true;
  if (!final_pass) {  // the host steps the final rounds (mfx_step)
    st->s.terminated_known = false;
    if (st->host_ctrl->status == 6) return fail(MFX_TIMEOUT, "device watchdog expired");
    if (st->host_ctrl->status == 3)
      return fail(MFX_SOLVER_ERROR, "push/relabel count %llu exceeded the termination ceiling %llu",
                  st->host_ctrl->pushes + st->host_ctrl->relabels, st->host_ctrl->ceiling);
    return MFX_OK;
  }
  st->s.terminated_known = r->status == 0;
  return solve_status(st, r);
}

int mfx_solve_dynamic_pushpull(mfx_graph *g, mfx_state *st, int64_t k, const int64_t *us,
                               const int64_t *vs, const int64_t *new_caps, const mfx_params *p,
                               mfx_result *r) {
  return pushpull_common(g, st, k, us, vs, new_caps, p, r, true);
}

int mfx_pushpull_regions(mfx_graph *g, mfx_state *st, int64_t k, const int64_t *us,
                         const int64_t *vs, const int64_t *new_caps, const mfx_params *p,
                         mfx_result *r) {
  return pushpull_common(g, st, k, us, vs, new_caps, p, r, false);
}

int mfx_apply_updates(mfx_graph *g, mfx_state *st, int64_t k, const int64_t *us,
                      const int64_t *vs, const int64_t *new_caps) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  if (st) {
    int rc0 = sync_caps(g->g, st->s);
    if (rc0) return rc0;
  }
  CK(ensure_batch_capacity(T, k));
  int64_t *d = T.ws.d_batch;
  if (k > 0) {
    CK(cudaMemcpyAsync(d, us, sizeof(int64_t) * k, cudaMemcpyHostToDevice, T.stream));
    CK(cudaMemcpyAsync(d + k, vs, sizeof(int64_t) * k, cudaMemcpyHostToDevice, T.stream));
    CK(cudaMemcpyAsync(d + 2 * k, new_caps, sizeof(int64_t) * k, cudaMemcpyHostToDevice, T.stream));
  }
  CK(launch_batch(g->g, st ? &st->s : nullptr, k, d, d + k, d + 2 * k, true, false, nullptr));
  long long err[8];
  CK(cudaMemcpyAsync(err, T.ws.d_err, sizeof(err), cudaMemcpyDeviceToHost, T.stream));
  CK(cudaStreamSynchronize(T.stream));
  int rc = batch_error(err, k, us, vs, new_caps, nullptr, nullptr, nullptr);
  if (rc) return rc;
  if (k > 0) g->g.cap_id = next_cap_id();
  if (st) st->s.cap_id = g->g.cap_id;
  if (st && k > 0) {
    // apply_updates alone leaves excess stale until recompute_excess (dynamic.py:114-116)
    st->s.excess_consistent = false;
    st->s.terminated_known = false;
  }
  return MFX_OK;
}

int mfx_dynamic_prephase(mfx_graph *g, mfx_state *st, int64_t k, const int64_t *us,
                         const int64_t *vs, const int64_t *new_caps) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  int rc;
  if ((rc = sync_caps(g->g, st->s))) return rc;
  if ((rc = require_terminated(st, "solve_dynamic"))) return rc;
  CK(ensure_batch_capacity(T, k));
  int64_t *d = T.ws.d_batch;
  if (k > 0) {
    CK(cudaMemcpyAsync(d, us, sizeof(int64_t) * k, cudaMemcpyHostToDevice, T.stream));
    CK(cudaMemcpyAsync(d + k, vs, sizeof(int64_t) * k, cudaMemcpyHostToDevice, T.stream));
    CK(cudaMemcpyAsync(d + 2 * k, new_caps, sizeof(int64_t) * k, cudaMemcpyHostToDevice, T.stream));
  }
  if (!st->s.excess_consistent) CK(launch_recompute_excess(g->g, st->s));
  CK(launch_batch(g->g, &st->s, k, d, d + k, d + 2 * k, true, true, nullptr));
  CK(launch_saturate(g->g, st->s, T.ws.d_err));
  long long err[8];
  CK(cudaMemcpyAsync(err, T.ws.d_err, sizeof(err), cudaMemcpyDeviceToHost, T.stream));
  CK(cudaStreamSynchronize(T.stream));
  if ((rc = batch_error(err, k, us, vs, new_caps, nullptr, nullptr, nullptr))) return rc;
  if (k > 0) g->g.cap_id = next_cap_id();
  st->s.cap_id = g->g.cap_id;
  st->s.excess_consistent = true;
  st->s.terminated_known = false;
  return MFX_OK;
}

int mfx_recompute_excess(mfx_state *st, const mfx_graph *g) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  int rc0 = sync_caps(g->g, st->s);
  if (rc0) return rc0;
  CK(launch_recompute_excess(g->g, st->s));
  CK(cudaStreamSynchronize(T.stream));
  st->s.excess_consistent = true;
  return MFX_OK;
}

int mfx_step(const mfx_graph *g, mfx_state *st, const mfx_params *p, int step, int dynamic_bases,
             int64_t *active, mfx_result *r) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  SolveConfig cfg;
  int rc = resolve_config(T, p, cfg);
  if (rc) return rc;
  CK(cudaSetDevice(T.device));
  if ((rc = sync_caps(g->g, st->s))) return rc;
  // static rounds: bases {t}, nothing forbidden (solver.py:155-164); dynamic:
  // bases {t} U deficient, s forbidden (dynamic.py:119-133)
  cfg.dyn_bases = dynamic_bases ? 1 : 0;
  cfg.forbidden = dynamic_bases ? st->s.s : -1;
  cfg.reset_counters = (step & 0x10) != 0;  // first step of an instrumented solve
  step &= 0xF;
  if (step == 0) cfg.what = WHAT_BFS;
  else if (step == 1) cfg.what = WHAT_ROUND;
  else cfg.what = WHAT_FINAL;
  int launches = 0;
  if (cfg.deterministic && cfg.what == WHAT_ROUND) {
    CK(launch_det_round(g->g, st->s, cfg.kc, cfg.topology));
    ++launches;
  } else {
    CK(launch_solve(g->g, st->s, cfg, &launches));
  }
  CK(cudaMemcpyAsync(st->host_ctrl, st->s.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, T.stream));
  CK(cudaStreamSynchronize(T.stream));
  if (r) {
    memset(r, 0, sizeof(*r));
    fill_result(st, r);
    r->launches = launches;
  }
  if (active) *active = st->host_ctrl->active;
  st->s.terminated_known = false;
  if (st->host_ctrl->status == 6) return fail(MFX_TIMEOUT, "device watchdog expired");
  if (st->host_ctrl->status == 3)
    return fail(MFX_SOLVER_ERROR,
                "push/relabel count %llu exceeded the termination ceiling %llu; solver state is "
                "likely corrupt",
                st->host_ctrl->pushes + st->host_ctrl->relabels, st->host_ctrl->ceiling);
  if (step == 2) st->s.terminated_known = true;
  return MFX_OK;
}

int mfx_certificate(const mfx_state *st, const mfx_graph *g, int64_t *cut, uint8_t *a_mask) {
  mfx_verify_report rep;
  int rc;
  if (cut) {
    if ((rc = mfx_verify(st, g, &rep))) return rc;
    *cut = rep.cut_capacity;
  }
  if (a_mask) return mfx_mask(st, 2, a_mask);
  return MFX_OK;
}

int mfx_verify(const mfx_state *st, const mfx_graph *g, mfx_verify_report *rep) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  Staged b;
  CK(cudaMalloc(&b.p, sizeof(long long) * 16));
  CK(launch_verify(g->g, st->s, (long long *)b.p));
  long long v[16];
  CK(cudaMemcpyAsync(v, b.p, sizeof(v), cudaMemcpyDeviceToHost, T.stream));
  CK(cudaStreamSynchronize(T.stream));
  rep->negative_cf = v[0];
  rep->pair_violations = v[1];
  rep->excess_mismatch = v[2];
  rep->excess_sum = v[3];
  rep->active_vertices = v[4];
  rep->unsaturated_ab = v[5];
  rep->loaded_ba = v[6];
  rep->cut_capacity = v[7];
  rep->flow_at_bases = v[8];
  rep->source_in_b = v[9];
  rep->sink_in_a = v[10];
  rep->first_bad_slot = v[11] == LLONG_MAX ? -1 : v[11];
  return MFX_OK;
}

int mfx_bench_barrier(const mfx_graph *g, mfx_state *st, int iters, int blocks_per_sm,
                      double *ns_per_barrier) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  SolveConfig cfg;
  cfg.what = WHAT_BARRIER;
  cfg.kc = iters;
  cfg.blocks_per_sm = blocks_per_sm;
  CK(launch_solve(g->g, st->s, cfg, nullptr));  // warm-up
  CK(cudaEventRecord(T.ev[0], T.stream));
  CK(launch_solve(g->g, st->s, cfg, nullptr));
  CK(cudaEventRecord(T.ev[1], T.stream));
  CK(cudaEventSynchronize(T.ev[1]));
  *ns_per_barrier = 1e6 * ev_ms(T.ev[0], T.ev[1]) / (iters > 0 ? iters : 1);
  return MFX_OK;
}

// Dependent-load latency (the latency roofline's unit): one thread chases
// indices through a `words`-entry permutation that jumps ~ a page per step
// (odd multiplier mod 2^k), so every load misses the caches.
__global__ void chase_init_kernel(unsigned *p, unsigned long long words) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < words;
       i += (unsigned long long)gridDim.x * blockDim.x)
    p[i] = (unsigned)((i * 40503ull + 12345ull) & (words - 1));
}
__global__ void chase_kernel(const unsigned *p, int steps, unsigned *sink, unsigned long long *ns) {
  unsigned j = 0;
  const unsigned long long t0 = globaltimer();
  for (int s = 0; s < steps; ++s) j = __ldcg(p + j);
  const unsigned long long t1 = globaltimer();
  *sink = j;
  *ns = t1 - t0;
}

int mfx_bench_chase(const mfx_graph *g, int64_t bytes, int steps, double *ns_per_load) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  unsigned long long words = 1;
  while (words * 2 * sizeof(unsigned) <= (unsigned long long)bytes) words *= 2;
  unsigned *p = nullptr;
  unsigned long long *d = nullptr;
  CK(cudaMalloc(&p, words * sizeof(unsigned) + 64));
  d = (unsigned long long *)(p + words);
  chase_init_kernel<<<T.num_sms * 8, 256, 0, T.stream>>>(p, words);
  chase_kernel<<<1, 1, 0, T.stream>>>(p, 64, (unsigned *)(d + 1), d);  // (warm the TLB path)
  chase_kernel<<<1, 1, 0, T.stream>>>(p, steps, (unsigned *)(d + 1), d);
  unsigned long long ns = 0;
  cudaError_t e = cudaMemcpyAsync(&ns, d, sizeof(ns), cudaMemcpyDeviceToHost, T.stream);
  if (!e) e = cudaStreamSynchronize(T.stream);
  cudaFree(p);
  CK(e);
  *ns_per_load = (double)ns / (steps > 0 ? steps : 1);
  return MFX_OK;
}

int mfx_trace_fetch(const mfx_state *st, const mfx_graph *g, uint64_t *out, int64_t cap,
                    int64_t *count) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  *count = 0;
  if (!T.ws.trace) return MFX_OK;
  long long tn = 0;
  CK(cudaMemcpy(&tn, &st->s.ctrl->trace_n, sizeof(tn), cudaMemcpyDeviceToHost));
  if (tn > cap) tn = cap;
  if (tn > T.ws.trace_cap) tn = T.ws.trace_cap;
  if (tn > 0) CK(cudaMemcpy(out, T.ws.trace, sizeof(uint64_t) * tn, cudaMemcpyDeviceToHost));
  *count = tn;
  return MFX_OK;
}

int mfx_sample_batch(mfx_graph *g, int64_t source, int64_t sink, int64_t k_dec, int64_t k_inc,
                     uint64_t seed, double bias, int64_t *us, int64_t *vs, int64_t *caps,
                     int64_t *got) {
  Topology &T = *g->g.topo;
  LOCK_TOPO(T);
  if (source < 0 || source >= T.n || sink < 0 || sink >= T.n)
    return fail(MFX_VALUE_ERROR, "source / sink out of range [0, %d)", T.n);
  if (k_dec < 0 || k_inc < 0) return fail(MFX_VALUE_ERROR, "negative update counts");
  CK(cudaSetDevice(T.device));
  long long n_got = 0;
  CK(sample_batch(g->g, (int)source, (int)sink, k_dec, k_inc, seed, bias, (long long *)us,
                  (long long *)vs, (long long *)caps, &n_got));
  *got = n_got;
  return MFX_OK;
}

int mfx_reached_list(const mfx_state *st, int32_t *out, int64_t cap, int64_t *count) {
  Topology &T = *st->s.topo;
  LOCK_TOPO(T);
  CK(cudaSetDevice(T.device));
  *count = -1;
  if (!st->s.tl_ok) return MFX_OK;
  Ctrl c;
  CK(cudaMemcpy(&c, st->s.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
  long long cnt = c.snap[C_REACHED];
  if (cnt > cap) return fail(MFX_VALUE_ERROR, "reached list of %lld entries exceeds cap %lld", cnt,
                             (long long)cap);
  if (cnt > 0)
    CK(cudaMemcpy(out, st->s.tl[c.tl_cur & 1], sizeof(int) * cnt, cudaMemcpyDeviceToHost));
  *count = cnt;
  return MFX_OK;
}

int mfx_transfer_bytes(int64_t k, int64_t *h2d, int64_t *d2h) {
  *h2d = 3 * (int64_t)sizeof(int64_t) * k;                       // batch us, vs, new caps
  *d2h = (int64_t)sizeof(Ctrl) + 8 * (int64_t)sizeof(long long);  // result block + error block
  return MFX_OK;
}

int mfx_host_alloc(size_t bytes, void **ptr) {
  CK(cudaHostAlloc(ptr, bytes ? bytes : 16, cudaHostAllocDefault));
  return MFX_OK;
}
int mfx_host_free(void *ptr) {
  CK(cudaFreeHost(ptr));
  return MFX_OK;
}
void *mfx_graph_stream(const mfx_graph *g) { return (void *)g->g.topo->stream; }

}  // extern "C"
