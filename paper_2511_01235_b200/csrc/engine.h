// engine.h -- host-side objects and internal launch entry points of libmfx.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <mutex>
#include <string>

#include "mfx_internal.cuh"

namespace mfx {

constexpr int kFirstNone = 0x7f7f7f7f;  // byte-fill sentinel of Workspace::slot_first

// Workspace for the persistent solve kernel, sized by (n, S); shared by every
// state that lives on the same topology (calls are serialised per process).
struct Workspace {
  int n = 0;
  int rcap = 0;
  int *F[2][NBIN] = {};  // BFS frontiers (double buffered), capacity n per bin
  int *R[NBIN] = {};     // round list (push waves + repair scope), capacity rcap per bin
  int *bases = nullptr;  // last global relabel's base set, capacity n
  int *heavy = nullptr;  // heavy rows scratch, capacity n
  unsigned *mark = nullptr;  // wave stamps, n
  int *bmark = nullptr;      // BFS epoch stamps (next-frontier dedupe), n
  uint8_t *reg = nullptr;    // push-pull regions (1 = prior cut's A side), n
  unsigned *stamp = nullptr; // current wave stamp (1 word)
  uint8_t *vbin = nullptr;   // degree class per vertex, n
  int *rdirty = nullptr;     // NBIN: used extent of each R list (reset to -1 before reuse)
  unsigned long long *trace = nullptr;  // diagnostics ($MFX_TRACE_CAP entries)
  int trace_cap = 0;
  int *slot_first = nullptr; // batch duplicate detection, S (kept at kFirstNone)
  // batch staging
  int64_t kcap = 0;
  int64_t *d_batch = nullptr;  // 3*kcap int64 (us, vs, caps)
  int *d_slot = nullptr;       // kcap resolved slots
  int *d_uv = nullptr;         // 2*kcap decomposed (u, v)
  long long *d_err = nullptr;  // batch error block (8 x int64)
  unsigned long long *d_red = nullptr;  // reduction scratch (64 x u64)
  ~Workspace();
};

struct Topology {
  int device = 0;
  int n = 0;
  int S = 0;
  int m_original = 0;
  int64_t diag[3] = {0, 0, 0};
  int cap_bytes = 4;
  int *off = nullptr, *adj = nullptr, *rev = nullptr;
  uint8_t *orig = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {};
  int num_sms = 0;
  int variant = -1;  // solve-kernel build: 0 = v256, 1 = v512 (-1: not chosen yet)
  Workspace ws;
  // every C-ABI call on this topology (graph copies and their states share the
  // workspace, the stream and the events) holds this lock
  std::recursive_mutex mu;
  ~Topology();
};

struct GraphObj {
  std::shared_ptr<Topology> topo;
  void *cap0 = nullptr;  // CapT[S]
  void *pc = nullptr;    // CapT[S]
  // identity of the current capacity contents: a fresh id on every cap0
  // write (builds, set_cap0, applied batches); copies inherit it
  uint64_t cap_id = 0;
  ~GraphObj();
};

struct StateObj {
  std::shared_ptr<Topology> topo;
  int s = 0, t = 0;
  void *cf = nullptr;        // CapT[S]
  long long *ex = nullptr;   // int64[n]
  int *h = nullptr;          // int32[n]
  Ctrl *ctrl = nullptr;      // control block
  bool excess_consistent = true;  // excess == sum_row(cf - cap0) known to hold
  // Reached-set lists (int32[n] each, allocated by the first tracked solve):
  // a tracked solve appends every vertex its relabels reach, so
  // tl[ctrl->tl_cur][0, ctrl->reached) is exactly {h < n}.  tl_ok: that holds
  // now (cleared by anything else that writes h).
  int *tl[2] = {nullptr, nullptr};
  bool tl_ok = false;
  bool terminated_known = false;  // last op was a completed solve
  uint64_t cap_id = 0;            // capacities cf / excess were last consistent with
  ~StateObj();
};

// ---- solve kernel front-end (solve.cu) ------------------------------------
enum What { WHAT_SOLVE = 0, WHAT_BFS = 1, WHAT_ROUND = 2, WHAT_FINAL = 3, WHAT_BARRIER = 4 };

struct SolveConfig {
  int what = WHAT_SOLVE;
  int dyn_bases = 1;   // bases {t} U deficient (else {t})
  int forbidden = -1;  // vertex never discovered (s in dynamic mode)
  int kc = 1;
  int max_waves = 0;
  int wave_mult = 2;  // auto wave budget per round: wave_mult * BFS levels / 4 + wave_add
  int wave_add = 4;
  int async = 0;          // asynchronous push phase (work queue) instead of waves
  int async_budget = 16;  // items per initially active vertex before a global relabel
  int flags = 0;          // mfx_params.flags (bit 0: BFS without h pre-load)
  int bfs_local_max = 64; // ... while the frontier holds <= this many items per CTA
  int lq_cap = kLQ;       // CTA-local queue capacity per sub-level
  int tail_items = 0;     // push: extra waves past the budget while a wave holds <= tail_items
  int tail_cap = 0;       //   ... up to tail_cap waves per round
  int coop_kc = 0;        // steps per visit of a long row (0: kc); each step rescans the row
  int walk_max = 0;       // excess walk when a global relabel finds <= walk_max active vertices
  int walk_depth = 0;     // ... and the BFS is at least walk_depth levels deep
  int max_ctas = 0;       // cap on the persistent grid (0: every SM at full occupancy)
  int tail_local = 256;   // push waves of <= tail_local short-row items run in CTA 0 alone
  int ring_sleep = 64;    // ns an idle warp sleeps between polls of its CTA's BFS ring
  int wave_time = -1;     // > 0: a push phase ends once it has run wave_time/8 x the last BFS's
                          //   time; 0 off; < 0 auto (10 on short-row graphs, off on long-row)
  int bfs_local = -1;     // CTA-local BFS levels per grid barrier (0 = level-synchronous);
                          //   < 0 auto: 128 on short-row graphs, 0 on long-row graphs
  int topology = 0;
  double timeout_s = 600.0;
  int blocks_per_sm = 0;
  unsigned long long ceiling = ~0ull;
  bool reset_counters = true;
  const long long *gate = nullptr;  // batch error block: skip the solve if the batch failed
  bool pushpull = false;  // O2 pipelines (region-restricted push / pull rounds)
  bool deterministic = false;  // serial round kernel (det.cu), reference deterministic mode
  int strand = 0;  // push phase ends once the sink is cut off and every deficit is filled
  int early = 1;   // solve relabels stop once every excess holder is labelled (0 off)
  int track = 1;   // WHAT_SOLVE launches keep the reached-set list (StateObj::tl; 0 off)
  int ramp = 4;    // first ring epoch's labels when the demand-covered exit is in reach
  int sparse = 1;  // relabels reset / seed from that list when it is small (0 off)
  long long batch_k = 0;  // dynamic solves: updates of the batch (their endpoints seed too)
};

// Dispatch to the solve-kernel build chosen for the graph (Topology::variant).
cudaError_t launch_solve(const GraphObj &g, StateObj &st, const SolveConfig &cfg, int *launches);
// push-pull set-up: crossing = false -> regions from the terminated heights;
// true -> push every A->B residual across the prior cut (gated by a batch)
cudaError_t launch_pp_setup(const GraphObj &g, StateObj &st, bool crossing, const long long *gate);
namespace v256 {
cudaError_t launch_solve(const GraphObj &g, StateObj &st, const SolveConfig &cfg, int *launches);
cudaError_t launch_pp_setup(const GraphObj &g, StateObj &st, bool crossing, const long long *gate);
}  // namespace v256
namespace v512 {
cudaError_t launch_solve(const GraphObj &g, StateObj &st, const SolveConfig &cfg, int *launches);
cudaError_t launch_pp_setup(const GraphObj &g, StateObj &st, bool crossing, const long long *gate);
}  // namespace v512
// fraction (in 1/1000) of the slots that sit in rows longer than kBin0Max
cudaError_t long_row_permille(const Topology &t, int *permille);
cudaError_t ensure_workspace(Topology &t);
cudaError_t ensure_batch_capacity(Topology &t, int64_t k);

// ---- state / batch kernels (state.cu) -------------------------------------
cudaError_t launch_init_state(const GraphObj &g, StateObj &st);
cudaError_t launch_vbin(const Topology &t, uint8_t *vbin);
// device batch sampler (state.cu; gen.py fast_batch semantics, host outputs)
cudaError_t sample_batch(const GraphObj &g, int s, int t, long long k_dec, long long k_inc,
                         unsigned long long seed, double bias, long long *us, long long *vs,
                         long long *caps, long long *got);
// gate: optional batch error block; the kernel is a no-op if the batch failed
cudaError_t launch_saturate(const GraphObj &g, StateObj &st, const long long *gate = nullptr);
cudaError_t launch_refresh_pc(const GraphObj &g);
cudaError_t launch_mask(const StateObj &st, int which, uint8_t *d_out);
cudaError_t launch_recompute_excess(const GraphObj &g, StateObj &st);
cudaError_t launch_count_active(const StateObj &st, unsigned long long *d_out);
// one deterministic round after a global relabel: worklist, serial push, serial repair (det.cu)
cudaError_t launch_det_round(const GraphObj &g, StateObj &st, int kc, int topology);
cudaError_t launch_pair_check(const GraphObj &g, const StateObj &st, unsigned long long *d_out);
cudaError_t launch_cap_check(const Topology &T, const int64_t *d_cap, unsigned long long *d_out);
// Batch: validate into ws.d_err (no mutation), then apply only if no error.
// update_excess: move excess at repaired endpoints (fused solve_dynamic path);
// false mirrors apply_updates alone, which leaves excess to recompute_excess.
cudaError_t launch_batch(GraphObj &g, StateObj *st, int64_t k, const int64_t *d_us,
                         const int64_t *d_vs, const int64_t *d_caps, bool apply,
                         bool update_excess, int *launches);
cudaError_t launch_edge_indices(const GraphObj &g, int64_t k, const int64_t *d_us,
                                const int64_t *d_vs, int64_t *d_out);
cudaError_t launch_verify(const GraphObj &g, const StateObj &st, long long *d_rep);
cudaError_t launch_convert_cap(const int64_t *src, void *dst, int cap_bytes, int64_t cnt,
                               cudaStream_t s);
cudaError_t launch_widen_cap(const void *src, int64_t *dst, int cap_bytes, int64_t cnt,
                             cudaStream_t s);
cudaError_t pair_max_int64(const Topology &topo, const int64_t *d_cap0, unsigned long long *d_out);

// ---- builder (build.cu) ---------------------------------------------------
// Builds the topology and int64 cap0 on the device from device edge arrays.
// Returns 0 or an error: kind in err[0] (1 n<=0, 2 src range, 3 dst range,
// 4 negative cap), offending edge index in err[1].
cudaError_t build_bicsr_device(int64_t n, int64_t m, const int64_t *d_us, const int64_t *d_vs,
                               const int64_t *d_caps, Topology &topo, int64_t **d_cap0_out,
                               int64_t err[2], int *launches);
cudaError_t topology_from_bicsr(int64_t n, int64_t S, const int64_t *d_off, const int64_t *d_adj,
                                const int64_t *d_rev, const uint8_t *d_orig, Topology &topo);
cudaError_t download_src(const Topology &topo, int64_t *d_src);

extern thread_local std::string g_last_error;
void count_launch(int k = 1);

}  // namespace mfx
