// solve.cu -- the persistent cooperative push-relabel solve kernel.
//
// One launch runs the whole round loop of the reference _push_rounds
// (solver.py:204-241) on the device:
//
//   loop:  global relabel (frontier BFS from the bases, kernels.py:168-215)
//          -> active set compacted during discovery (state.py:62-67)
//          -> exit when empty (solver.py:221-222: device-side convergence)
//          -> push phase: waves of bounded push/relabel (kernels.py:19-67)
//             over the live active list; a vertex that becomes active during
//             a wave joins the next wave (excess moves several
//             hops per global relabel instead of one)
//          -> repair of steep edges (kernels.py:70-93) over every vertex
//             processed in the round
//   finalize: flow = sum of excess over the bases (dynamic.py:141-143),
//             cut = sum cap0 over A->B slots, A = {h == n} (solver.py:178-184)
//
// Work is binned by degree (vbin): thread / warp / CTA per vertex, and
// grid-wide expansion for huge rows (s and t of the grid config have ~2.1 M
// slots).  Every loop that appends to a work list is warp-uniform, so the
// appends of a warp are staged in shared memory and published 32 at a time
// with one atomic (the per-list counters are the hottest addresses of the
// whole solve).  Phases are separated by a software grid barrier whose last
// arriving CTA snapshots the append counters and checks the watchdog and the
// operation ceiling, so every loop decision is taken on identical values.
#include <limits.h>
#include <stdio.h>
#include <stdlib.h>

#include "engine.h"

#ifndef MFX_SOLVE_NS
#define MFX_SOLVE_NS v256
#endif

namespace mfx {
// Compiled twice (Makefile): v256 = 256-thread CTAs, 2 per SM, no register
// cap (latency-bound grids and roads); v512 = 512-thread CTAs, 2 per SM,
// 64 registers (4x the resident warps, for graphs whose slots sit mostly in
// long rows, e.g. R-MAT).  api.cu picks per graph (Topology::variant).
namespace MFX_SOLVE_NS {

constexpr unsigned FULL = 0xffffffffu;

// length of the reached-set list at the start of the current BFS epoch
// (tracked launches; 0 during the seeding pass)
__shared__ int s_tl_base;
// which reached-set list holds the last relabel's reach (Ctrl::tl_cur; each
// CTA's copy, flipped by its thread 0 at the end of every tracked relabel)
__shared__ int s_tl_cur;
// the running relabel appends to its list (its predecessor reached < n/16,
// so it is expected to reach few vertices too); the last relabel's list is
// valid (launch: the host's StateObj::tl_ok; then: that relabel tracked)
__shared__ int s_tl_trk, s_tl_ok;
// this round's repair stamp (Workspace::bmark): a vertex listed by several
// waves of the round is repaired once
__shared__ unsigned s_rep_stamp;
// deficits this CTA filled during its current run of tail waves (CTA 0 alone
// pushes then: the stop test reads this instead of Ctrl::fills in L2)
__shared__ unsigned s_fills;

template <typename CapT>
struct SolveArgs {
  int n;
  int s, t;
  int forbidden;
  int dyn_bases;
  int kc;
  int max_waves;  // > 0: fixed waves per round; 0: wave_mult * BFS levels + wave_add
  int wave_mult;
  int wave_add;
  int async;         // asynchronous push phase (data mode only)
  int async_budget;  // items per initially active vertex before the next global relabel
  int *rdirty;       // NBIN used extents of the R lists (device, shared by states)
  int bfs_local;     // labels a CTA's BFS ring may run ahead per grid barrier (0 = level-synchronous)
  int flags;         // bit 0: BFS relaxes with the atomic alone (no pre-load of h[v])
  int bfs_local_max; // the ring only when the frontier <= this many items per CTA
  int lq_cap;        // CTA ring capacity is 2 x lq_cap (<= 2 kLQ; the rest spills)
  int tail_items;    // push: after the wave budget, continue while a wave holds <= this many
  int tail_cap;      //   ... up to this many waves in the round
  int coop_kc;       // push/relabel steps per visit of a cooperative (long) row
  int walk_max;      // excess walk after a global relabel with <= this many active vertices
  int walk_depth;    // ... at least this many BFS levels deep
  int tail_local;    // push waves of <= this many items run in CTA 0 alone (0: off)
  int wave_time;     // push phase time budget, eighths of the last BFS's time (0: off)
  int strand;        // end a push phase once the sink is cut off and every deficit is filled
  int early;         // solve relabels stop once every excess holder is labelled
  int ring_sleep;    // ns an idle warp sleeps between polls of the BFS ring
  int track;         // keep the reached-set list: every relabel appends what it reaches
  int ramp;          // first ring epoch's labels when the demand-covered exit is in reach
  int sparse;        // the first relabel may seed from the list (StateObj::tl_ok)
  int *tl[2];        // the two reached-set lists (n each)
  const int *buv;    // the batch's (u, v) endpoints (2 * bk), first relabel after a batch
  long long bk;
  const uint8_t *__restrict__ reg;  // push-pull: 1 = prior cut's A side (pull), 0 = B side
  int *bmark;        // per-vertex epoch stamp: next-frontier dedupe
  int topology;
  int what;
  int rcap;
  const int *__restrict__ off;
  const int *__restrict__ adj;
  const int *__restrict__ rev;
  const uint8_t *__restrict__ vbin;  // degree class of every vertex (bin_of(deg))
  const CapT *__restrict__ cap0;
  const CapT *__restrict__ pc;
  CapT *cf;
  long long *ex;
  int *h;
  int *F0[NBIN];
  int *F1[NBIN];
  int *R[NBIN];
  int *bases;
  int *heavy;
  unsigned *mark;
  unsigned *stamp;  // persistent wave stamp shared by all states of the topology
  Ctrl *ctrl;
  const long long *gate;  // batch error block (dynamic solves), may be null
  unsigned long long *trace;  // optional phase trace (diagnostics), may be null
  int trace_cap;
};

// algorithmic bytes per event, CapT-dependent
template <typename CapT>
struct Bytes {
  static constexpr int kVertex = 20;                          // off(2x4) + h 4 + ex 8
  static constexpr int kSlot = 8 + (int)sizeof(CapT);         // adj + cf + h[v]
  static constexpr int kBfsSlot = 8 + 2 * (int)sizeof(CapT);  // adj + cf + pc + h[v]
  static constexpr int kPush = 2 * (int)sizeof(CapT) + 16 + 4;
  static constexpr int kDisc = 8;
};

struct Local {
  unsigned long long pushes = 0, relabels = 0, repairs = 0, bytes = 0;
};

// per-warp staging queues in shared memory: q0 = next frontier (bin 0),
// q1 = next push wave / active list (bin 0)
#ifndef MFX_WQ
#define MFX_WQ 64
#endif
constexpr int kWQ = MFX_WQ;         // per-warp staging capacity (per queue)
constexpr int kFlush = kWQ - 32;    // publish once this many items are staged
struct WarpQ {
  int cnt[3];
  int item[3][kWQ];  // q0 next frontier, q1 round list, q2 reached-set list (track)
};

// ---------------------------------------------------------------------------
// grid barrier with a leader action
// ---------------------------------------------------------------------------
struct Sync {
  unsigned gen;
  int *s_snap;  // smem copy of ctrl->snap after the last barrier
  int *s_abort;
  unsigned long long deadline, ceiling;  // read once at kernel start
  int strand;                            // SolveArgs::strand
  unsigned long long t_last;             // block 0: phase timing
  unsigned long long t_tail;             // block 0: last tail-wave timestamp (trace)
  unsigned long long ph[PH_N];
  unsigned long long *trace;  // block 0: (phase << 60 | items << 32 | dt_ns) per barrier
  int trace_cap, trace_n;
};

__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned *p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Arrival is an acq_rel RMW on the counter (releases this CTA's writes, which
// bar.sync made visible to thread 0; the last arriver acquires everyone's);
// the release store of the generation publishes the leader's snapshot.
// No full fences on the critical path.
__device__ __noinline__ void grid_sync(Ctrl *c, Sync &sy, unsigned snap_mask, unsigned acc_mask,
                                       unsigned clear_mask, int phase) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile Ctrl *vc = c;
    unsigned prev = atom_add_acq_rel(&c->bar_count, 1u);
    if (prev == gridDim.x - 1) {
      const unsigned rd = snap_mask | acc_mask;
      int lv[C_NCTR], sv[C_NCTR];
#pragma unroll
      for (int i = 0; i < C_NCTR; ++i) {  // all loads in flight together
        lv[i] = (rd >> i & 1) ? vc->live[i] : 0;
        sv[i] = ((acc_mask & ~clear_mask & ~snap_mask) >> i & 1) ? vc->snap[i] : 0;
      }
      unsigned long long p = vc->pushes, r = vc->relabels;
      int ab = vc->abort;
      // stranded-excess rule inputs, loaded with the rest (off the chain
      // when the rule is off: the leader's loads are the barrier's latency)
      const bool st_on = sy.strand && phase == PH_PUSH;
      const unsigned long long fills = st_on ? vc->fills : 0ull;
      const int talive = st_on ? vc->snap[C_TALIVE] : 1;
      const int dbases = st_on ? vc->snap[C_DBASES] : 0;
#pragma unroll
      for (int i = 0; i < C_NCTR; ++i) {
        if (rd >> i & 1) {
          vc->snap[i] = i == C_DEPTH ? (lv[i] > sv[i] ? lv[i] : sv[i]) : lv[i] + sv[i];
          vc->live[i] = 0;
        } else if (clear_mask >> i & 1) {
          vc->snap[i] = 0;
        }
      }
      // demand-covered rule (BFS barriers that accumulate the relabel's
      // counters): with the sink cut off, the deficits are the only bases
      // that can absorb excess; once the labelled holders carry at least
      // their total, the relabel may stop.  Allowed only while the total
      // deficit keeps shrinking between such stops, so the rounds progress.
      if (phase == PH_BFS && ((acc_mask | clear_mask) >> C_EHOLD & 1)) {
        const bool fresh = (clear_mask >> C_EHOLD & 1) != 0;  // the seeding barrier
        const long long d = (fresh ? 0 : vc->x_snap[0]) + vc->x_live[0];
        const long long x = (fresh ? 0 : vc->x_snap[1]) + vc->x_live[1];
        vc->x_snap[0] = d;
        vc->x_snap[1] = x;
        vc->x_live[0] = vc->x_live[1] = 0;
        const bool fire = sy.strand && vc->snap[C_TALIVE] == 0 && d > 0 && x >= d &&
                          d < vc->efill_d;
        if (fire) vc->efill_d = d;
        vc->snap[C_EFILL] = fire;
      }  // (other BFS barriers -- sparse reset, exit listing -- keep it)
      const unsigned long long now = globaltimer();
      const unsigned long long wdl = vc->wave_deadline;
      vc->snap[C_STOP] = phase == PH_PUSH && ((wdl != 0 && now > wdl) ||
                                              (talive == 0 && fills >= (unsigned)dbases));
      if (!ab) {
        if (now > sy.deadline) {
          vc->abort = 1;
          vc->status = 6;
        } else if (p + r > sy.ceiling) {
          vc->abort = 1;
          vc->status = 3;
        }
      }
      vc->bar_count = 0;
      st_release_u32(&c->bar_gen, sy.gen + 1);
    } else {
      unsigned spins = 0;
      while (ld_acquire_u32(&c->bar_gen) == sy.gen) {
        __nanosleep(20);
        if ((++spins & 0xFFFFu) == 0) {
          // escape hatch: a CTA is stuck far past the watchdog; give up so the
          // launch terminates instead of hanging the device.
          if (globaltimer() > sy.deadline + 30ull * 1000000000ull) {
            vc->abort = 1;
            vc->status = 6;
            break;
          }
        }
      }
    }
    sy.gen += 1;
    int snapv[C_NCTR];
#pragma unroll
    for (int i = 0; i < C_NCTR; ++i) snapv[i] = vc->snap[i];
    int ab = vc->abort;
#pragma unroll
    for (int i = 0; i < C_NCTR; ++i) sy.s_snap[i] = snapv[i];
    *sy.s_abort = ab;
    if (blockIdx.x == 0) {
      unsigned long long now = globaltimer();
      unsigned long long dt = now - sy.t_last;
      sy.ph[phase] += dt;
      sy.t_last = now;
      if (sy.trace && sy.trace_n < sy.trace_cap) {
        unsigned items = 0;  // work published for the next phase
        for (int i = 0; i < 8; ++i) items += (unsigned)snapv[i];
        sy.trace[sy.trace_n++] = ((unsigned long long)phase << 60) |
                                 ((unsigned long long)(items & 0xFFFFFFFu) << 32) |
                                 (dt & 0xFFFFFFFFull);
      }
    }
  }
  __syncthreads();
}

// block-wide sum, result valid in thread 0
template <typename T>
__device__ __forceinline__ T block_sum(T v, T *scratch) {
  v = warp_sum(v);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[w] = v;
  __syncthreads();
  T r = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kWarps; ++i) r += scratch[i];
  return r;
}

__device__ void flush_counters(Ctrl *c, Local &lc, unsigned long long *scr) {
  unsigned long long p = block_sum(lc.pushes, scr);
  if (threadIdx.x == 0 && p) atomicAdd(&c->pushes, p);
  unsigned long long r = block_sum(lc.relabels, scr);
  if (threadIdx.x == 0 && r) atomicAdd(&c->relabels, r);
  unsigned long long q = block_sum(lc.repairs, scr);
  if (threadIdx.x == 0 && q) atomicAdd(&c->repairs, q);
  unsigned long long b = block_sum(lc.bytes, scr);
  if (threadIdx.x == 0 && b) atomicAdd(&c->bytes, b);
  lc = Local();
}

// inclusive warp scan (full warp)
__device__ __forceinline__ long long warp_incl_scan(long long v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long w = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += w;
  }
  return v;
}

// PP = the push-pull pipelines of O2 (dynamic.py:178-377): the prior cut's
// A side (reg 1) pulls deficits from its supply, the B side (reg 0) pushes
// overflow to the sink and its deficits, every scan stays inside the vertex's
// own region, and the two pipelines run as one device round loop.
template <typename CapT, bool PP = false>
struct Kern {
  const SolveArgs<CapT> &a;
  Sync &sy;
  Local &lc;
  WarpQ *q;  // this warp's staging queues
  int gtid, gthreads, gwarp, gwarps, lane, wib;
  int swarp;  // warp index with CTAs fastest: thin lists spread over every SM
  int *rctr;  // next-wave list counters: the global live ones, or CTA 0's own in tail mode
  int act_cnt;  // active discoveries counted by this lane in the current level
  // the list the running relabel appends to / the last relabel's
  __device__ __forceinline__ int *tl_new() const { return s_tl_cur ? a.tl[0] : a.tl[1]; }
  __device__ __forceinline__ const int *tl_old() const { return s_tl_cur ? a.tl[1] : a.tl[0]; }
  long long *s_sink;  // per-CTA sum of excess pushed into the sink this round
  long long sink_acc; // this thread's share, not yet added to s_sink

  // Excess arriving at v.  The sink receives pushes from up to every pixel of
  // the grid config in the same wave; a global atomic on ex[t] per push
  // serialises at one L2 slice and even a shared-memory atomic per push
  // serialises a CTA, so each thread sums the sink's share in a register and
  // sink_flush publishes it once per round (nothing reads ex[t] before the
  // round ends: t never pushes and the global relabel takes it as a base by
  // identity).  Returns the previous excess of v (for the sink: a positive
  // dummy, it never activates).
  __device__ __forceinline__ long long add_excess(int v, long long d) {
    if (v == a.t) {
      sink_acc += d;
      return 1;
    }
    return atomic_add(a.ex + v, d);
  }
  __device__ __forceinline__ void sink_flush() {  // whole CTA, before a grid barrier
    const long long w = warp_sum(sink_acc);
    sink_acc = 0;
    if (lane == 0 && w) atomicAdd((unsigned long long *)s_sink, (unsigned long long)w);
    __syncthreads();
    if (threadIdx.x == 0) {  // (only thread 0 touches s_sink here)
      const long long x = *s_sink;
      if (x) {
        atomic_add(a.ex + a.t, x);
        *s_sink = 0;
      }
    }
  }

  __device__ Kern(const SolveArgs<CapT> &a_, Sync &sy_, Local &lc_, WarpQ *wq, long long *sink)
      : a(a_), sy(sy_), lc(lc_), s_sink(sink) {
    gtid = blockIdx.x * blockDim.x + threadIdx.x;
    gthreads = gridDim.x * blockDim.x;
    sink_acc = 0;
    lane = threadIdx.x & 31;
    wib = threadIdx.x >> 5;
    gwarp = gtid >> 5;
    gwarps = gthreads >> 5;
    swarp = wib * (int)gridDim.x + (int)blockIdx.x;
    rctr = a.ctrl->live + C_RNEXT;
    q = wq + wib;
    act_cnt = 0;
    hexc = 0;
  }

  __device__ __forceinline__ int vbin(int v) const { return __ldg(a.vbin + v); }
  // a push took a deficient base's excess to >= 0 (stranded-excess rule)
  __device__ __forceinline__ void fill_once() const {
    atomicAdd(&a.ctrl->fills, 1ull);
    atomicAdd(&s_fills, 1u);
  }
  __device__ __forceinline__ int region(int v) const { return PP ? (int)__ldg(a.reg + v) : 0; }

  // ---- warp-synchronous list appends (every lane of the warp must call) ----
  __device__ __forceinline__ void stage(int qi, bool pred, int v, int *counter, int *buf, int base,
                                        int cap) {
    unsigned b = __ballot_sync(FULL, pred);
    if (b == 0) return;
    int c = q->cnt[qi];
    if (pred) q->item[qi][c + __popc(b & lanemask_lt())] = v;
    c += __popc(b);
    __syncwarp();
    if (c >= kFlush) {  // publish everything staged with one atomic
      int g = 0;
      if (lane == 0) g = atomicAdd(counter, c);
      g = __shfl_sync(FULL, g, 0);
      for (int k = lane; k < c; k += 32) {
        int p = base + g + k;
        if (p < cap) buf[p] = q->item[qi][k];
        else a.ctrl->overflow = 1;
      }
      c = 0;
    }
    __syncwarp();
    if (lane == 0) q->cnt[qi] = c;
    __syncwarp();
  }

  __device__ __forceinline__ void stage_flush(int qi, int *counter, int *buf, int base, int cap) {
    int c = q->cnt[qi];
    if (c == 0) return;
    int g = 0;
    if (lane == 0) g = atomicAdd(counter, c);
    g = __shfl_sync(FULL, g, 0);
    for (int k = lane; k < c; k += 32) {
      int p = base + g + k;
      if (p < cap) buf[p] = q->item[qi][k];
      else a.ctrl->overflow = 1;
    }
    __syncwarp();
    if (lane == 0) q->cnt[qi] = 0;
    __syncwarp();
  }

  __device__ __forceinline__ void direct(bool pred, int v, int *counter, int *buf, int base, int cap) {
    unsigned b = __ballot_sync(FULL, pred);
    if (b == 0) return;
    int leader = __ffs(b) - 1;
    int g = 0;
    if (lane == leader) g = atomicAdd(counter, __popc(b));
    g = __shfl_sync(FULL, g, leader);
    if (pred) {
      int p = base + g + __popc(b & lanemask_lt());
      if (p < cap) buf[p] = v;
      else a.ctrl->overflow = 1;
    }
  }

  // bin 0 through the staging queue, bins 1..3 (rare) directly
  __device__ __forceinline__ void append_binned(int qi, bool pred, int v, int bin, int *counters,
                                                int *const *bufs, const int *bases, int cap) {
    stage(qi, pred && bin == 0, v, counters, bufs[0], bases[0], cap);
    if (__any_sync(FULL, pred && bin != 0)) {
#pragma unroll
      for (int b = 1; b < NBIN; ++b)
        direct(pred && bin == b, v, counters + b, bufs[b], bases[b], cap);
    }
  }

  // =========================================================================
  // global relabel (kernels.py:168-215)
  // =========================================================================
  // Frontier BFS over reverse residual slots with label-correcting relaxation
  // (atomicMin on h): between two grid barriers ("epoch") a CTA may expand
  // its own discoveries, up to `local_levels` labels past the epoch's start
  // depth, from a shared-memory work ring drained asynchronously by its warps
  // (ring_drain: no barrier between BFS levels).  Ring overflow and the
  // discoveries past the label cap go to the global next frontier
  // (deduplicated per epoch by an epoch stamp).  Every lowering of h[v]
  // schedules an expansion of v that re-reads h[v], so the fixpoint is the
  // exact BFS distance (bit-exact with the reference's FIFO BFS, tested);
  // local_levels = 0 is the strict level-synchronous BFS.
  //
  // A discovery costs one atomic: the item carries a "first visit" flag
  // (bit 31) and the expansion of that item, which loads off/h anyway, also
  // loads ex and appends an active vertex to the round list (state.py:62-67)
  // binned by the degree it just read.  Rows longer than kBin0Max met by a
  // thread-per-item pass are handed to the CTA's warps (shared list) or, past
  // kBin1Max, to the next epoch's CTA / grid-wide lists.
  static constexpr int kFirstBit = (int)0x80000000;
  static constexpr int kIdMask = 0x7fffffff;
  static constexpr int kHQ = 256;  // CTA heavy-row list
  static constexpr int kRing = 2 * kLQ;  // (power of two)
  static constexpr int kEmpty = -1;      // (not an item: ids are < 2^31 - 1)
  enum { RQ_TAIL = 0, RQ_HEAD = 1, RQ_RD = 2, RQ_DONE = 3 };
  unsigned ep_next;  // ownership stamp of the coming asynchronous push phase
  unsigned bst;      // this epoch's stamp for next-frontier dedupe
  int disc_cnt;      // first discoveries (+ bases) by this lane
  int xc;            // trace mode: vertices this lane expanded in the epoch
  int max_lab;       // largest label this lane set
  long long hexc;    // excess of the active vertices this lane listed (demand-covered exit)
  bool loc_ok;       // discoveries may go to the CTA-local queue
  bool nocheck;      // relax with the atomic alone (no h[v] pre-load)
  int *ring;         // CTA-local work ring (shared memory, kRing slots, kEmpty = free)
  unsigned *rq;      // its counters: RQ_TAIL reserved, RQ_HEAD claimed, RQ_RD released, RQ_DONE
  int ring_cap;      // slots the ring may hold at once (<= kRing)
  int lcap;          // largest label a discovery may carry into the ring this epoch
  int *hq;           // CTA heavy-row list (shared memory, kHQ)
  int *hq_cnt;
  bool hq_ok;        // long rows may go to the CTA's heavy-row list
  const int *rb_;    // round-list bases of this epoch (shared)
  int *const *Fn_;   // next-frontier lists of this epoch

  __device__ __forceinline__ bool relax(int v, int nl, bool &first) {
    int old = atomicMin(a.h + v, nl);
    first = old == a.n;
    return nl < old;
  }

  // k ring slots, or -1 when the ring lacks room (slots are free once
  // released, RQ_RD, which follows the claim order).  One lane.
  __device__ __forceinline__ int ring_reserve(int k) {
    volatile unsigned *vq = rq;
    for (;;) {
      unsigned t = vq[RQ_TAIL], r = vq[RQ_RD];
      if ((int)(t + k - r) > ring_cap) return -1;
      if (atomicCAS(rq + RQ_TAIL, t, t + k) == t) return (int)t;
    }
  }

  // CTA-local BFS over the ring, asynchronous: each warp claims up to 32
  // queued items, expands them (its discoveries join the ring) and marks
  // them done; no barrier between BFS levels, the atomicMin relaxation makes
  // the order immaterial (label-correcting).  Ends when every reserved item
  // is done (done is read before tail; an expansion reserves its discoveries
  // before its item counts as done).  Whole CTA.
  __device__ void ring_drain() {
    volatile unsigned *vq = rq;
    volatile int *vr = ring;
    for (;;) {
      unsigned h = 0;
      int c = 0;
      bool fin = false;
      if (lane == 0) {
        for (;;) {
          h = vq[RQ_HEAD];
          unsigned t = vq[RQ_TAIL];
          if (h == t) break;
          c = (int)(t - h) < 32 ? (int)(t - h) : 32;
          if (atomicCAS(rq + RQ_HEAD, h, h + c) == h) break;
          c = 0;
        }
        if (c == 0) {
          unsigned d = vq[RQ_DONE];
          __threadfence_block();
          fin = d == vq[RQ_TAIL];
        }
      }
      c = __shfl_sync(FULL, c, 0);
      if (c == 0) {
        if (__shfl_sync(FULL, (int)fin, 0)) break;
        if (a.ring_sleep > 0) __nanosleep(a.ring_sleep);
        continue;
      }
      h = __shfl_sync(FULL, h, 0);
      int item = 0;
      if (lane < c) {  // a reserved slot is written right after its reservation
        const int q = (int)((h + lane) & (kRing - 1));
        while ((item = vr[q]) == kEmpty) {
        }
        vr[q] = kEmpty;
      }
      __syncwarp();
      if (lane == 0) {  // release in claim order
        while (vq[RQ_RD] != h) {
        }
        __threadfence_block();
        vq[RQ_RD] = h + c;
      }
      expand_item(lane < c, item);
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        atomicAdd(rq + RQ_DONE, (unsigned)c);
      }
    }
  }

  // Label of v lowered (low) to nl; first = v was unreached.  Warp-synchronous.
  __device__ __forceinline__ void discovered(bool low, bool first, int v, int nl) {
    if (low) {
      max_lab = nl > max_lab ? nl : max_lab;
      if (first) {
        ++disc_cnt;
        lc.bytes += Bytes<CapT>::kDisc;
      }
    }
    const int item = v | (first ? kFirstBit : 0);
    bool glob = low;
    if (loc_ok) {  // expanded by this CTA within the epoch (ring), label permitting
      const bool want = low && nl <= lcap;
      unsigned m = __ballot_sync(FULL, want);
      if (m) {
        int leader = __ffs(m) - 1, pos0 = 0;
        if (lane == leader) pos0 = ring_reserve(__popc(m));
        pos0 = __shfl_sync(FULL, pos0, leader);
        if (want && pos0 >= 0) {  // (no room: the global next frontier)
          ring[(pos0 + __popc(m & lanemask_lt())) & (kRing - 1)] = item;
          glob = false;
        }
      }
    }
    // once per epoch in the global list: a first discovery cannot be listed
    // yet; a re-lowered vertex may be (rows handed to the next epoch make
    // even the level-synchronous mode label-correcting)
    if (glob && !first) glob = atomicMax(a.bmark + v, bst) < bst;
    else if (glob) a.bmark[v] = bst;
    stage(0, glob, item, a.ctrl->live + C_FNEXT, Fn_[0], 0, a.n);
  }

  // Report the relaxations of a row chunk: bit k of `low` set = vv[k] was
  // lowered to nl (bit k of `fst`: first visit).  Each lane walks its set
  // bits in order; the warp loops as often as its busiest lane has bits, so
  // discovered() (ballots, ring reservation, staging) is inlined once and
  // runs once per actual discovery instead of once per slot of the row (a
  // thread-per-row pass unrolled over 8 slots otherwise inlines it 8 times:
  // ~5 K instructions of the kernel's hot code).  Warp-synchronous.
  template <int K>
  __device__ __forceinline__ void report(unsigned low, unsigned fst, const int (&vv)[K], int nl) {
    while (__any_sync(FULL, low != 0)) {
      const int k = low ? __ffs(low) - 1 : 0;
      int v = vv[0];
#pragma unroll
      for (int q = 1; q < K; ++q) v = k == q ? vv[q] : v;  // (register select, no local array)
      const bool l = low != 0;
      discovered(l, l && (fst >> k & 1), v, nl);
      low &= low - 1;
    }
  }

  // K slots i, i + stride, ... (< hi) per lane of a long row: every load of
  // the K slots is issued before any result is consumed, so a row scan is
  // not a chain of one-slot round trips.  Warp-uniform trip count.
  template <int K>
  __device__ __forceinline__ void discover_slots(int i, int stride, int hi, int nl, int ru) {
    int vv[K];
    CapT rr[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = i + k * stride;
      const bool valid = j < hi;
      vv[k] = valid ? __ldg(a.adj + j) : -1;
      CapT f = valid ? (CapT)ldcg((const CapT *)(a.cf + j)) : (CapT)0;
      rr[k] = !valid ? (CapT)0 : (PP && ru == 1) ? f : __ldg(a.pc + j) - f;
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (vv[k] == a.forbidden || (PP && vv[k] >= 0 && region(vv[k]) != ru)) rr[k] = 0;
    int hv[K];
    if (!nocheck) {
#pragma unroll
      for (int k = 0; k < K; ++k) hv[k] = rr[k] > 0 ? ldcg(a.h + vv[k]) : -1;
    }
    bool low[K], fst[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      fst[k] = false;
      low[k] = rr[k] > 0 && (nocheck || hv[k] > nl) && relax(vv[k], nl, fst[k]);
    }
#pragma unroll
    {
      unsigned lm = 0, fm = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        lm |= (unsigned)low[k] << k;
        fm |= (unsigned)fst[k] << k;
      }
      report<K>(lm, fm, vv, nl);
    }
  }

  // Thread per item: the row (<= kBin0Max slots) is expanded with every load
  // issued before any result is consumed; first visits join the round list
  // when active; longer rows are handed on.  Warp-synchronous.
  __device__ __forceinline__ void expand_item(bool valid, int item) {
    const int u = item & kIdMask;
    const bool first = valid && item < 0;
    xc += valid;
    int lo = 0, d = 0, hu = a.n;
    long long eu = 0;
    if (valid) {
      lo = __ldg(a.off + u);
      d = __ldg(a.off + u + 1) - lo;
      hu = ldcg(a.h + u);
      if (first) eu = ldcg(a.ex + u);
      lc.bytes += Bytes<CapT>::kVertex;
    }
    const int ru = valid ? region(u) : 0;
    const bool act = first && u != a.s && u != a.t && (ru == 1 ? eu < 0 : eu > 0);
    act_cnt += act;
    if (!PP && act) hexc += eu;
    // reached-set list: a vertex joins at its first expansion (exactly once
    // per relabel: one first-visit item per discovery); an early exit lists
    // the first-visit items it leaves unexpanded (exit_list).  The append
    // counter is C_REACHED itself.  (Appending at the discovery instead put
    // one more inlined append per slot into the hot loop: C2 +8 %.)
    if (s_tl_trk) stage(2, first, u, a.ctrl->live + C_REACHED, tl_new(), s_tl_base, a.n);
    // queued for the push phase: owned (async) / listed for wave 0 (walk dedupe)
    if (act && (a.async || a.walk_max > 0)) a.mark[u] = ep_next;
    append_binned(1, act && !a.topology, u, bin_of(d), a.ctrl->live + C_RNEXT, a.R, rb_, a.rcap);
    const bool heavy = valid && d > kBin0Max;
    if (__any_sync(FULL, heavy)) {
      // (only items of the grid-wide pass: those are spread evenly over the
      // CTAs; a CTA's own ring hands long rows to the whole grid)
      bool mid = hq_ok && heavy && d <= kBin1Max, to_cta = false;
      unsigned m = __ballot_sync(FULL, mid);
      if (m) {  // warp-per-row rows: this CTA's warps, after this pass
        int leader = __ffs(m) - 1, pos0 = 0;
        if (lane == leader) pos0 = atomicAdd(hq_cnt, __popc(m));
        pos0 = __shfl_sync(FULL, pos0, leader);
        int p = pos0 + __popc(m & lanemask_lt());
        if (mid && p < kHQ) {
          hq[p] = u;
          to_cta = true;
        }
      }
      int hb = heavy && !to_cta ? bin_of(d) : 0;
#pragma unroll
      for (int b = 1; b < NBIN; ++b)  // next epoch's warp / CTA / grid lists
        direct(heavy && !to_cta && hb == b, u, a.ctrl->live + C_FNEXT + b, Fn_[b], 0, a.n);
    }
    if (heavy) d = 0;
    lc.bytes += (unsigned long long)d * Bytes<CapT>::kBfsSlot;
    const int nl = hu + 1;
    int vv[kBin0Max], hv[kBin0Max];
    CapT rr[kBin0Max];
#pragma unroll
    for (int k = 0; k < kBin0Max; ++k) {  // heads + reverse residuals of the row
      vv[k] = k < d ? __ldg(a.adj + lo + k) : -1;
      rr[k] = k < d ? __ldg(a.pc + lo + k) - (CapT)ldcg((const CapT *)(a.cf + lo + k)) : (CapT)0;
    }
    if (PP) {  // pull side: forward residuals; either side: own region only
#pragma unroll
      for (int k = 0; k < kBin0Max; ++k) {
        if (k < d && ru == 1) rr[k] = (CapT)ldcg((const CapT *)(a.cf + lo + k));
        if (k < d && region(vv[k]) != ru) rr[k] = 0;
      }
    }
    bool low[kBin0Max], fst[kBin0Max];
    if (nocheck) {
#pragma unroll
      for (int k = 0; k < kBin0Max; ++k) {
        fst[k] = false;
        low[k] = rr[k] > 0 && vv[k] != a.forbidden && relax(vv[k], nl, fst[k]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < kBin0Max; ++k)  // head heights across residual slots only
        hv[k] = (rr[k] > 0 && vv[k] != a.forbidden) ? ldcg(a.h + vv[k]) : -1;
#pragma unroll
      for (int k = 0; k < kBin0Max; ++k) {
        fst[k] = false;
        low[k] = hv[k] > nl && relax(vv[k], nl, fst[k]);
      }
    }
#pragma unroll
    {
      unsigned lm = 0, fm = 0;
#pragma unroll
      for (int k = 0; k < kBin0Max; ++k) {
        lm |= (unsigned)low[k] << k;
        fm |= (unsigned)fst[k] << k;
      }
      report<kBin0Max>(lm, fm, vv, nl);
    }
  }

  // Warp per row over the CTA's heavy-row list (whole CTA calls).
  __device__ void drain_heavy() {
    __syncthreads();
    int c = *hq_cnt;
    __syncthreads();
    if (c == 0) return;
    if (c > kHQ) c = kHQ;
    for (int j = wib; j < c; j += kWarps) {
      int u = hq[j];
      int lo = __ldg(a.off + u), hi = __ldg(a.off + u + 1);
      int nl = ldcg(a.h + u) + 1;
      if (lane == 0) lc.bytes += (unsigned long long)(hi - lo) * Bytes<CapT>::kBfsSlot;
      for (int i0 = lo; i0 < hi; i0 += 4 * 32) discover_slots<4>(i0 + lane, 32, hi, nl, region(u));  // (4 gathers in flight)
    }
    __syncthreads();
    if (threadIdx.x == 0) *hq_cnt = 0;
  }

  __device__ void level_flush(int *const *Fn, const int *rbase) {
    stage_flush(0, a.ctrl->live + C_FNEXT, Fn[0], 0, a.n);
    stage_flush(1, a.ctrl->live + C_RNEXT, a.R[0], rbase[0], a.rcap);
    int c = warp_sum(act_cnt);
    if (lane == 0 && c) atomicAdd(a.ctrl->live + C_ACTIVE, c);
    act_cnt = 0;
    if (!PP) {
      const long long x = warp_sum(hexc);
      if (lane == 0 && x) atomicAdd((unsigned long long *)&a.ctrl->x_live[1], (unsigned long long)x);
      hexc = 0;
    }
    if (s_tl_trk) {
      stage_flush(2, a.ctrl->live + C_REACHED, tl_new(), s_tl_base, a.n);
    } else {
      c = warp_sum(disc_cnt);
      if (lane == 0 && c) atomicAdd(a.ctrl->live + C_REACHED, c);
    }
    disc_cnt = 0;
    int m = max_lab;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      int w = __shfl_xor_sync(FULL, m, o);
      m = w > m ? w : m;
    }
    if (lane == 0 && m) atomicMax(a.ctrl->live + C_DEPTH, m);
  }

  // Early exit of a tracked relabel: the first-visit items of the frontier
  // it leaves unexpanded (bin 0 of epoch E's list) join the reached-set
  // list, whose length the barrier then publishes.  Whole grid.
  __device__ void exit_list(int E, int cnt0) {
    if (!s_tl_trk) return;
    __syncthreads();
    if (threadIdx.x == 0) s_tl_base = sy.s_snap[C_REACHED];
    __syncthreads();
    const int *Fc0 = (E & 1) ? a.F1[0] : a.F0[0];
    for (int j0 = gwarp * 32; j0 < cnt0; j0 += gwarps * 32) {
      const int j = j0 + lane;
      const int item = j < cnt0 ? ldcg(Fc0 + j) : 0;
      stage(2, item < 0, item & kIdMask, a.ctrl->live + C_REACHED, tl_new(), s_tl_base, a.n);
    }
    stage_flush(2, a.ctrl->live + C_REACHED, tl_new(), s_tl_base, a.n);
    grid_sync(a.ctrl, sy, 0, 1u << C_REACHED, 0, PH_BFS);
  }

  // Trace mode: per-epoch expansion counts (sum and max over CTAs), recorded
  // by CTA 0 after the epoch's barrier as a phase-6 trace entry.  Whole CTA.
  __device__ void epoch_stats(int E, bool before) {
    __shared__ unsigned s_xc;
    Ctrl *c = a.ctrl;
    if (before) {
      if (threadIdx.x == 0) s_xc = 0;
      __syncthreads();
      int w = warp_sum(xc);
      if (lane == 0 && w) atomicAdd(&s_xc, (unsigned)w);
      __syncthreads();
      if (threadIdx.x == 0) {
        atomicAdd(c->dbg_sum + (E & 1), s_xc);
        atomicMax(c->dbg_max + (E & 1), s_xc);
      }
    } else if (blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned sum = __ldcg(c->dbg_sum + (E & 1)), mx = __ldcg(c->dbg_max + (E & 1));
      c->dbg_sum[E & 1] = 0;
      c->dbg_max[E & 1] = 0;
      if (sy.trace && sy.trace_n < sy.trace_cap)
        sy.trace[sy.trace_n++] = (6ull << 60) | ((unsigned long long)(mx & 0xFFFFFFFu) << 32) | sum;
    }
  }

  // Returns the BFS depth (levels incl. level 0 = max label + 1); the active
  // set is left in R (wave 0).  ep: ownership stamp the following
  // asynchronous push phase will use; bstamp: persistent epoch stamp.
  // filt: holders count for the early exit only if the previous relabel of
  // this solve reached them (h < n): a vertex it left unreached has no
  // residual path to a base, pushes only move excess between reached
  // vertices (creating arcs among them) and the bases only shrink, so it
  // stays unreachable for the rest of the solve.  (A local relabel to n
  // means no residual out-arc, which nothing adds back: no push or repair
  // can target a vertex at height n.)  Not after a batch: its updates and
  // the source re-saturation change arbitrary arcs.
  //
  // Reached-set lists (StateObj::tl): a relabel whose predecessor reached
  // fewer than n/16 vertices appends everything it reaches (bases + first
  // discoveries) to a list, so {h < n} is exactly that list's entries.  The
  // next relabel then resets and searches bases over the list (plus the
  // batch endpoints, where a negative repair can create a deficit, on the
  // first relabel after a batch) instead of all n vertices: C4's sink side
  // is a corner, so a relabel there costs its reach, not a 24 M-vertex pass.
  __device__ int bfs(unsigned ep, unsigned &bstamp, int local_levels, bool early, bool filt,
                     bool first_after_batch) {
    const int n = a.n;
    int holders = 0;  // vertices (not s, t) with positive excess
    int dbases = 0;   // deficient bases (bases other than the sink)
    long long dsum = 0;  // their total deficit
    __shared__ int zero[NBIN];
    __shared__ int rb[NBIN];
    __shared__ int s_ring[kRing];
    __shared__ unsigned s_rq[4];
    __shared__ int s_hq[kHQ];
    __shared__ int s_hqc;
    // A frontier list that overflowed (label-correcting duplicates beyond
    // the per-epoch dedupe: not observed, but not excluded either) would
    // leave the labels incomplete, so the relabel is then redone in strict
    // level-synchronous mode, which lists every vertex at most once.
    int E_all = 0;  // epochs over the attempts
    if (gtid == 0) a.ctrl->bfs_t0 = globaltimer();  // (push-phase time budget)
    const int reached_old = sy.s_snap[C_REACHED];  // (the last relabel's; uniform)
    const bool trk = a.track && !PP && !a.topology && (long long)reached_old * 16 < (long long)n;
    const bool sparse0 = trk && a.sparse && s_tl_ok;
    __syncthreads();  // (everyone has read s_tl_ok)
    if (threadIdx.x == 0) s_tl_trk = trk;
    for (int attempt = 0;; ++attempt) {
    const bool sparse = sparse0 && attempt == 0;  // (the strict retry seeds in full)
    if (threadIdx.x == 0) s_tl_base = 0;
    ep_next = ep;
    disc_cnt = 0;
    max_lab = 0;
    hexc = 0;
    holders = 0;
    dbases = 0;
    dsum = 0;
    loc_ok = false;
    nocheck = (a.flags & 1) != 0;
    ring = s_ring;
    rq = s_rq;
    ring_cap = 2 * a.lq_cap < kRing ? 2 * a.lq_cap : kRing;
    lcap = 0;
    for (int q = threadIdx.x; q < kRing; q += blockDim.x) s_ring[q] = kEmpty;
    hq = s_hq;
    hq_cnt = &s_hqc;
    hq_ok = true;
    rb_ = zero;
    Fn_ = a.F0;
    if (threadIdx.x < NBIN) zero[threadIdx.x] = 0;
    if (threadIdx.x < 4) s_rq[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_hqc = 0;
    __syncthreads();
    // empty the R lists (async consumers wait on -1 slots) and the async counters
    if (!a.topology) {  // (topology mode seeds R below and never runs asynchronously)
      for (int b = 0; b < NBIN; ++b) {
        int used = ldcg(a.rdirty + b);
        if (used > a.rcap) used = a.rcap;
        for (int j = gtid; j < used; j += gthreads) a.R[b][j] = -1;
      }
    }
    if (gtid == 0) {
      for (int b = 0; b < NBIN; ++b) {
        a.ctrl->aq_head[b] = 0;
        a.ctrl->aq_done[b] = 0;
      }
      a.ctrl->aq_stop = 0;
      a.ctrl->overflow = 0;  // dropped items are re-found by this global relabel
    }
    // reset + seed bases (kernels.py:184-193); topology mode seeds wave 0.
    // A lane takes 8 consecutive vertices: 4 x 16-byte excess loads in
    // flight together and 2 x 16-byte height stores (the pass is a latency
    // chain otherwise); the rare bases are appended only when the warp has one.
    constexpr int V = 8;
    if (sparse) {
      // 1) reset the last relabel's reach (holders among it: the filt rule)
      const int *Lo = tl_old();
      for (int j = gtid; j < reached_old; j += gthreads) {
        const int v = ldcg(Lo + j);
        if (filt)
          holders += v != a.s && v != a.t && ldcg(a.h + v) < n && ldcg(a.ex + v) > 0;
        a.h[v] = n;
      }
      if (!filt && gtid == 0) holders = 1 << 29;  // (all holders unknown: EHOLD rule off)
      lc.bytes += (unsigned long long)((reached_old + gthreads - 1 - gtid) / gthreads) * 8ull;
      grid_sync(a.ctrl, sy, 0, 0, 0, PH_BFS);  // every reset lands before a base is claimed
      // 2) bases: deficits can only sit in the old reach (they were bases of
      // the last relabel) or at a batch endpoint (negative repair); t always
      const long long nb_ll = (long long)reached_old + (first_after_batch ? 2 * a.bk : 0) + 1;
      const int nb = nb_ll > (long long)INT_MAX ? INT_MAX : (int)nb_ll;
      for (int j0 = gwarp * 32; j0 < nb; j0 += gwarps * 32) {
        const int j = j0 + lane;
        int v = -1;
        if (j < reached_old) v = ldcg(Lo + j);
        else if (j < nb - 1) v = ldcg(a.buv + (j - reached_old));
        else if (j == nb - 1) v = a.t;
        bool base = false;
        long long e = 0;
        if (v >= 0 && v != a.forbidden) {
          e = ldcg(a.ex + v);
          base = v == a.t || (a.dyn_bases && v != a.s && e < 0);
          if (base) base = atomicCAS(a.h + v, n, 0) == n;  // once per vertex
        }
        dbases += base && v != a.t;
        if (base && v != a.t) dsum -= e;
        const int b = base ? vbin(v) : 0;
        append_binned(0, base, v, b, a.ctrl->live + C_FNEXT, a.F0, zero, n);
        direct(base, v, a.ctrl->live + C_BASES, a.bases, 0, n);
        stage(2, base, v, a.ctrl->live + C_REACHED, tl_new(), 0, n);
      }
      lc.bytes += (unsigned long long)((nb + gthreads - 1 - gtid) / gthreads) * 16ull;
    }
    for (int v0 = gwarp * 32 * V; !sparse && v0 < n; v0 += gwarps * 32 * V) {
      const int vb = v0 + lane * V;
      const bool full = vb + V <= n;
      long long ev[V];
      if (full) {
#pragma unroll
        for (int r = 0; r < V; r += 2) {
          const longlong2 e2 = __ldcg(reinterpret_cast<const longlong2 *>(a.ex + vb + r));
          ev[r] = e2.x;
          ev[r + 1] = e2.y;
        }
      } else {
#pragma unroll
        for (int r = 0; r < V; ++r) ev[r] = vb + r < n ? ldcg(a.ex + vb + r) : 0;
      }
      unsigned bm = 0;  // bases among this lane's vertices
      unsigned cand = 0xFFu;  // relabel candidates (filt: reached by the previous relabel)
      if (filt) {
        if (full) {
          const int4 h0 = __ldcg(reinterpret_cast<const int4 *>(a.h + vb));
          const int4 h1 = __ldcg(reinterpret_cast<const int4 *>(a.h + vb) + 1);
          cand = (unsigned)(h0.x < n) | (unsigned)(h0.y < n) << 1 | (unsigned)(h0.z < n) << 2 |
                 (unsigned)(h0.w < n) << 3 | (unsigned)(h1.x < n) << 4 | (unsigned)(h1.y < n) << 5 |
                 (unsigned)(h1.z < n) << 6 | (unsigned)(h1.w < n) << 7;
        } else {
          cand = 0;
#pragma unroll
          for (int r = 0; r < V; ++r) cand |= (unsigned)(vb + r < n && ldcg(a.h + vb + r) < n) << r;
        }
      }
      int hv[V];
#pragma unroll
      for (int r = 0; r < V; ++r) {
        const int v = vb + r;
        const bool valid = v < n;
        bool base;
        if (PP) {  // push side: sink + deficits; pull side: source + overflow
          const int rg = valid ? region(v) : 0;
          base = valid && (rg == 0 ? (v == a.t || (v != a.s && ev[r] < 0))
                                   : (v == a.s || (v != a.t && ev[r] > 0)));
          // the side's actives (push side: overflow, pull side: deficits)
          holders += valid && v != a.s && v != a.t && (rg == 0 ? ev[r] > 0 : ev[r] < 0);
        } else {
          base = valid && (v == a.t || (a.dyn_bases && v != a.s && ev[r] < 0));
          holders += valid && v != a.s && v != a.t && ev[r] > 0 && (cand >> r & 1);
        }
        if (v == a.forbidden) base = false;
        hv[r] = base ? 0 : n;
        bm |= (unsigned)base << r;
        dbases += base && v != a.t;
        if (!PP && base && v != a.t) dsum -= ev[r];
      }
      if (full) {
        reinterpret_cast<int4 *>(a.h + vb)[0] = make_int4(hv[0], hv[1], hv[2], hv[3]);
        reinterpret_cast<int4 *>(a.h + vb)[1] = make_int4(hv[4], hv[5], hv[6], hv[7]);
      } else {
#pragma unroll
        for (int r = 0; r < V; ++r)
          if (vb + r < n) a.h[vb + r] = hv[r];
      }
      disc_cnt += __popc(bm);
      if (__any_sync(FULL, bm != 0)) {
#pragma unroll
        for (int r = 0; r < V; ++r) {
          const bool base = bm >> r & 1;
          const int v = vb + r;
          int b = base ? vbin(v) : 0;
          append_binned(0, base, v, b, a.ctrl->live + C_FNEXT, a.F0, zero, n);
          direct(base, v, a.ctrl->live + C_BASES, a.bases, 0, n);
          if (trk) stage(2, base, v, a.ctrl->live + C_REACHED, tl_new(), 0, n);
        }
      }
      if (a.topology) {
#pragma unroll
        for (int r = 0; r < V; ++r) {
          const int v = vb + r;
          bool topo = v < n && v != a.s && v != a.t;
          int tb = topo ? vbin(v) : 0;
          append_binned(1, topo, v, tb, a.ctrl->live + C_RNEXT, a.R, zero, a.rcap);
        }
      }
    }
    level_flush(a.F0, zero);
    holders = warp_sum(holders);
    if (lane == 0 && holders) atomicAdd(a.ctrl->live + C_EHOLD, holders);
    // is the sink still reachable at all?  residual slots into t (the
    // reverse residual of t's row, pc - cf); with none, only deficits can
    // absorb excess this round (push-phase stop rule, Ctrl::fills)
    if (!PP) {
      // (only "none" vs "some" matters: a thread stops at its first hit, so
      // the 2.1 M-slot sink row of C2 costs one pass of loads, not 28; and
      // only the dynamic rules read it)
      int talive = 0;
      if (a.strand) {
        const int t0 = __ldg(a.off + a.t), t1 = __ldg(a.off + a.t + 1);
        for (int i = t0 + gtid; i < t1 && talive == 0; i += gthreads)
          talive = __ldg(a.adj + i) != a.forbidden &&
                   __ldg(a.pc + i) - (CapT)ldcg((const CapT *)(a.cf + i)) > 0;
      }
      talive = warp_sum(talive);
      dbases = warp_sum(dbases);
      if (lane == 0 && talive) atomicAdd(a.ctrl->live + C_TALIVE, talive);
      if (lane == 0 && dbases) atomicAdd(a.ctrl->live + C_DBASES, dbases);
      dsum = warp_sum(dsum);
      if (lane == 0 && dsum)
        atomicAdd((unsigned long long *)&a.ctrl->x_live[0], (unsigned long long)dsum);
      if (gtid == 0 && !a.strand) atomicAdd(a.ctrl->live + C_DBASES, 1 << 30);  // rule off
      if (gtid == 0) a.ctrl->fills = 0;
    }
    if (!sparse) lc.bytes += (unsigned long long)((n + gthreads - 1 - gtid) / gthreads) * 12ull;
    const unsigned fmask = 0xFu << C_FNEXT, rmask = 0xFu << C_RNEXT;
    const unsigned amask = (1u << C_ACTIVE) | (1u << C_REACHED) | (1u << C_DEPTH) |
                           (1u << C_EHOLD) | (1u << C_TALIVE) | (1u << C_DBASES);
    if (a.trace) {  // trace: CTA 0's seeding pass done (phase-4 entry)
      __syncthreads();
      if (blockIdx.x == 0 && threadIdx.x == 0 && sy.trace_n < sy.trace_cap)
        sy.trace[sy.trace_n++] = (4ull << 60) | ((globaltimer() - sy.t_last) & 0xFFFFFFFFull);
    }
    grid_sync(a.ctrl, sy, fmask | (1u << C_BASES), rmask | amask, rmask | amask, PH_BFS);
    int E = 0;
    // With the demand-covered exit in reach (sink cut off, deficits to
    // fill) the ring epochs start short and double, so the barrier that can
    // stop the relabel comes a few labels after the holders near the
    // deficits are found, not after a full 128-label epoch (uniform: snap)
    int ramp = early && a.strand && sy.s_snap[C_TALIVE] == 0 && sy.s_snap[C_DBASES] > 0 ? a.ramp : 0;
    for (;;) {
      int cnt[NBIN];
      int tot = 0;
      for (int b = 0; b < NBIN; ++b) {
        cnt[b] = sy.s_snap[C_FNEXT + b];
        if (cnt[b] > n) cnt[b] = n;
        tot += cnt[b];
      }
      if (tot == 0 || *sy.s_abort) break;
      // the sink alone, cut off (no residual slot into it) and no deficit:
      // nothing can be discovered -- C4's closing relabel after its
      // deficits are filled skips the epoch that would confirm that
      if (!PP && E == 0 && a.strand && sy.s_snap[C_TALIVE] == 0 && sy.s_snap[C_DBASES] == 0) break;
      // Early exit (solve rounds only): every vertex holding excess has been
      // expanded, so the round's active list is complete; vertices beyond
      // keep h = n, which no push can cross, and the solve's last global
      // relabel (no holder left) always runs to the end, so the certificate
      // still comes from exact distances.
      // (push-pull relabels never certify -- the ordinary final pass does --
      // so with no active vertex on either side they stop at once)
      if (early && (sy.s_snap[C_EHOLD] > 0 || PP) && sy.s_snap[C_ACTIVE] >= sy.s_snap[C_EHOLD]) {
        exit_list(E, cnt[0]);
        break;
      }
      // Demand-covered exit (dynamic solves, sink cut off): the holders
      // labelled so far carry at least the total deficit, so this round's
      // pushes can fill every deficit without the far holders (C4: a batch's
      // new deficit is a few hops from the excess its decrease created,
      // while excess stranded near the source lies ~10^4 levels away).  The
      // barrier leader allows it only while the total deficit shrinks.
      if (early && sy.s_snap[C_EFILL]) {
        exit_list(E, cnt[0]);
        break;
      }
      if (threadIdx.x < NBIN) rb[threadIdx.x] = sy.s_snap[C_RNEXT + threadIdx.x];
      if (threadIdx.x == 0) s_tl_base = sy.s_snap[C_REACHED];
      __syncthreads();
      rb_ = rb;
      bst = ++bstamp;
      xc = 0;
      // the CTA ring only while the frontier is thin (latency-bound levels);
      // wide levels stay grid-wide so no CTA serialises a share of them
      // (R-MAT hubs)
      loc_ok = local_levels > 0 && tot <= a.bfs_local_max * (int)gridDim.x;
      lcap = sy.s_snap[C_DEPTH] + (ramp && ramp < local_levels ? ramp : local_levels);
      ramp *= 2;  // (labels so far <= C_DEPTH)
      // flags bit 1: thin (latency-bound) epochs relax by atomic alone
      nocheck = (a.flags & 1) != 0 || ((a.flags & 2) != 0 && loc_ok);
      int *const *Fc = (E & 1) ? a.F1 : a.F0;
      Fn_ = (E & 1) ? a.F0 : a.F1;
      // bin 0: thread per item (warp-uniform trip count).  Wide frontiers in
      // chunks of 32 dealt over the CTAs first (swarp).
      if (loc_ok) {
        // thin frontier: dealt one item at a time over the CTAs, so every
        // CTA's ring starts from an even share of it
        const int tid_dealt = (lane * kWarps + wib) * (int)gridDim.x + (int)blockIdx.x;
        for (int j0 = 0; j0 < cnt[0]; j0 += gthreads) {
          int j = j0 + tid_dealt;
          bool valid = j < cnt[0];
          expand_item(valid, valid ? ldcg(Fc[0] + j) : 0);
        }
      } else {
        for (int j0 = swarp * 32; j0 < cnt[0]; j0 += gwarps * 32) {
          int j = j0 + lane;
          bool valid = j < cnt[0];
          expand_item(valid, valid ? ldcg(Fc[0] + j) : 0);
        }
      }
      // bin 1: warp per row
      for (int j = swarp; j < cnt[1]; j += gwarps) {
        int u = ldcg(Fc[1] + j);
        int lo = __ldg(a.off + u), hi = __ldg(a.off + u + 1);
        int nl = ldcg(a.h + u) + 1;
        xc += lane == 0;
        if (lane == 0)
          lc.bytes += Bytes<CapT>::kVertex + (unsigned long long)(hi - lo) * Bytes<CapT>::kBfsSlot;
        for (int i0 = lo; i0 < hi; i0 += 4 * 32) discover_slots<4>(i0 + lane, 32, hi, nl, region(u));  // (4 gathers in flight)
      }
      // bin 2: CTA per row
      for (int j = blockIdx.x; j < cnt[2]; j += gridDim.x) {
        int u = ldcg(Fc[2] + j);
        int lo = __ldg(a.off + u), hi = __ldg(a.off + u + 1);
        int nl = ldcg(a.h + u) + 1;
        if (threadIdx.x == 0)
          lc.bytes += Bytes<CapT>::kVertex + (unsigned long long)(hi - lo) * Bytes<CapT>::kBfsSlot;
        for (int i0 = lo; i0 < hi; i0 += 4 * blockDim.x)
          discover_slots<4>(i0 + threadIdx.x, blockDim.x, hi, nl, region(u));
      }
      // bin 3: whole grid per row
      for (int j = 0; j < cnt[3]; ++j) {
        int u = ldcg(Fc[3] + j);
        int lo = __ldg(a.off + u), hi = __ldg(a.off + u + 1);
        int nl = ldcg(a.h + u) + 1;
        if (gtid == 0)
          lc.bytes += Bytes<CapT>::kVertex + (unsigned long long)(hi - lo) * Bytes<CapT>::kBfsSlot;
        for (int i0 = lo + gwarp * 32; i0 < hi; i0 += 4 * gthreads)
          discover_slots<4>(i0 + lane, gthreads, hi, nl, region(u));
      }
      drain_heavy();
      hq_ok = false;
      // this CTA's own discoveries, asynchronously, up to label lcap
      if (loc_ok) ring_drain();
      hq_ok = true;
      loc_ok = false;
      level_flush(Fn_, rb);
      if (a.trace) epoch_stats(E, true);
      grid_sync(a.ctrl, sy, fmask, rmask | amask, 0, PH_BFS);
      if (a.trace) epoch_stats(E, false);
      ++E;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_hqc = 0;
    E_all += E;
    // (read after the last barrier: uniform; flags bit 3 forces the retry, for tests)
    const bool ovf = ldcg(&a.ctrl->overflow) != 0 || ((a.flags & 8) != 0 && attempt == 0);
    if (!ovf || local_levels == 0 || *sy.s_abort || attempt > 0) break;
    local_levels = 0;
    early = false;
    filt = false;
    __syncthreads();
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // a tracked relabel's list is the current one now
      if (trk) s_tl_cur ^= 1;
      s_tl_ok = trk;
      s_tl_trk = 0;
      if (blockIdx.x == 0) {
        a.ctrl->tl_cur = s_tl_cur;
        a.ctrl->tl_ok = trk;
      }
    }
    __syncthreads();
    const int depth = sy.s_snap[C_DEPTH] + 1;
    if (sy.trace && threadIdx.x == 0 && sy.trace_n + 1 < sy.trace_cap) {
      // trace: the relabel's exit inputs (phase-8: deficit | labelled excess;
      // phase-9: efill | sink slots | deficient bases | holders | active)
      volatile Ctrl *vc = a.ctrl;
      const unsigned long long D = (unsigned long long)vc->x_snap[0] & 0xFFFFFFFull;
      const unsigned long long X = (unsigned long long)vc->x_snap[1] & 0xFFFFFFFFull;
      sy.trace[sy.trace_n++] = (8ull << 60) | (D << 32) | X;
      sy.trace[sy.trace_n++] =
          (9ull << 60) | ((unsigned long long)(sy.s_snap[C_EFILL] & 1) << 59) |
          ((unsigned long long)(sy.s_snap[C_TALIVE] & 0x7F) << 52) |
          ((unsigned long long)(sy.s_snap[C_DBASES] & 0xFFF) << 40) |
          ((unsigned long long)(sy.s_snap[C_EHOLD] & 0xFFFFF) << 20) |
          (unsigned long long)(sy.s_snap[C_ACTIVE] & 0xFFFFF);
    }
    if (gtid == 0) {
      a.ctrl->levels += depth;
      a.ctrl->epochs += E_all;
      a.ctrl->last_levels = depth;
      a.ctrl->reached = sy.s_snap[C_REACHED];
      for (int b = 0; b < NBIN; ++b) a.rdirty[b] = sy.s_snap[C_RNEXT + b];
    }
    return depth;
  }

  // =========================================================================
  // push phase (kernels.py:19-67) with in-phase re-activation
  // =========================================================================
  // Append v (degree class b, loaded ahead by the caller) to the next wave
  // once (stamp dedupe).  Warp-synchronous.
  __device__ __forceinline__ void activate(bool pred, int v, int b, unsigned stamp,
                                           const int *nbase) {
    if (pred) pred = atomicMax(a.mark + v, stamp) < stamp;
    append_binned(1, pred, v, b, rctr, a.R, nbase, a.rcap);
  }

  // Thread per vertex (rows of <= kBin0Max slots).  The row (head, reverse
  // slot, residual, head height) is loaded once with all loads in flight,
  // then up to KC push/relabel steps run on that register snapshot: cf only
  // grows under concurrent pushes and only this thread lowers it, so
  // snapshot - own pushes is a safe lower bound; stale neighbour heights are
  // the lock-free algorithm's tolerated race.
  template <bool Async>
  __device__ void push_thread(bool valid, int u, unsigned stamp, const int *nbase) {
    const int n = a.n;
    int lo = 0, d = 0, hu = n;
    long long eu = 0;
    const int ru = (PP && valid) ? region(u) : 0;
    const bool pull = PP && ru == 1;  // pull side: deficit = -excess, reversed residuals
    if (valid) {
      lo = __ldg(a.off + u);
      d = __ldg(a.off + u + 1) - lo;
      hu = ldcg(a.h + u);
      eu = ldcg(a.ex + u);
      if (pull) eu = -eu;
      lc.bytes += Bytes<CapT>::kVertex;
      // a deficient base (height 0, not the sink) that a push listed for
      // this wave and that holds no deficit any more: filled (a later
      // refill may count it twice, which only ends the phase earlier)
      if (!PP && a.strand && !a.topology && hu == 0 && eu >= 0 && u != a.t && u != a.s)
        fill_once();
    }
    const bool live = eu > 0 && hu < n;
    if (!live) d = 0;
    int vv[kBin0Max], hh[kBin0Max], rv[kBin0Max];
    CapT cc[kBin0Max];
#pragma unroll
    for (int k = 0; k < kBin0Max; ++k) {
      vv[k] = k < d ? __ldg(a.adj + lo + k) : 0;
      rv[k] = k < d ? __ldg(a.rev + lo + k) : 0;
      cc[k] = k < d ? (CapT)ldcg((const CapT *)(a.cf + lo + k)) : (CapT)0;
    }
    if (PP) {
#pragma unroll
      for (int k = 0; k < kBin0Max; ++k) {
        if (k < d && pull) cc[k] = __ldg(a.pc + lo + k) - cc[k];  // cf(v -> u)
        if (k < d && region(vv[k]) != ru) cc[k] = 0;
      }
    }
    int bb[kBin0Max];  // degree classes of the heads, in flight with their heights
#pragma unroll
    for (int k = 0; k < kBin0Max; ++k) {
      hh[k] = cc[k] > 0 ? ldcg(a.h + vv[k]) : INT_MAX;
      bb[k] = cc[k] > 0 ? vbin(vv[k]) : 0;
    }
    lc.bytes += (unsigned long long)d * Bytes<CapT>::kSlot;
    // Each slot is pushed at most once per visit (a push either saturates it
    // or exhausts u), so the old head excess per slot fits in registers and
    // the activation tests wait for all atomics together after the loop.
    long long oldv[kBin0Max];
    unsigned clm[kBin0Max];
#pragma unroll
    for (int k = 0; k < kBin0Max; ++k) clm[k] = ~0u;
    unsigned pushed = 0;
    long long e_after = eu;  // u's excess after its last push (from the atomic)
    bool own_atomic = false;
    long long own_old = 0, own_d = 0;
    if (live) {
      for (int cnt = 0; cnt < a.kc; ++cnt) {
        if (eu <= 0 || hu >= n) break;
        int bh = INT_MAX, bk = -1;  // first minimum in slot order (kernels.py:40-48)
#pragma unroll
        for (int k = 0; k < kBin0Max; ++k)
          if (cc[k] > 0 && hh[k] < bh) {
            bh = hh[k];
            bk = k;
          }
        if (bk < 0) {  // no residual out-edge: nothing can ever leave u
          hu = n;
          a.h[u] = n;
          lc.relabels++;
          break;
        }
        if (hu > bh) {
#pragma unroll
          for (int k = 0; k < kBin0Max; ++k)
            if (k == bk) {
              long long dd = eu < (long long)cc[k] ? eu : (long long)cc[k];
              cc[k] -= (CapT)dd;
              eu -= dd;
              if (pull) {  // pull dd along (v, u) (kernels.py:96-143)
                atomic_add(a.cf + rv[k], (CapT)(-dd));
                atomic_add(a.cf + lo + k, (CapT)dd);
                oldv[k] = -atomic_add(a.ex + vv[k], -dd);
              } else {
                atomic_add(a.cf + lo + k, (CapT)(-dd));
                atomic_add(a.cf + rv[k], (CapT)dd);
                oldv[k] = add_excess(vv[k], dd);
              }
              // wave mode: the head is claimed for the next wave right away
              // (in flight with the push, not after its result)
              if (!Async && vv[k] != a.s && vv[k] != a.t) clm[k] = atomicMax(a.mark + vv[k], stamp);
              own_d += dd;
              pushed |= 1u << k;
            }
          own_atomic = true;
          lc.pushes++;
          lc.bytes += Bytes<CapT>::kPush;
        } else {
          hu = bh + 1 > n ? n : bh + 1;  // relabel from the snapshot
          a.h[u] = hu;
          lc.relabels++;
        }
      }
    }
    // u's own excess drops once by everything it pushed (one atomic, not one
    // per push: a per-push atomic whose result lands in the same register
    // made every push step wait for the previous one).  Nothing reads ex[u]
    // for a decision meanwhile: concurrent pushers into u only need "was u
    // already holding excess", which it was.
    if (own_atomic) {
      own_old = pull ? -atomic_add(a.ex + u, own_d) : atomic_add(a.ex + u, -own_d);
      e_after = own_old - own_d;
    }
    // pushes must be visible before a head is handed to another owner
    if (Async) __threadfence();
    // A pushed head joins the next wave: in wave mode whenever this push
    // claimed it (a head that already held excess, or got none net, is then
    // a no-op item; one that was claimed before is listed already); in the
    // asynchronous phase when it was not holding excess before the push.
    if (Async) {
#pragma unroll
      for (int k = 0; k < kBin0Max; ++k) {
        bool p = (pushed >> k & 1) && oldv[k] <= 0 && vv[k] != a.s && vv[k] != a.t;
        activate(p, vv[k], bb[k], stamp, nbase);
      }
    } else {  // (compacted like report(): one inlined append, run per listed head)
      unsigned lst = 0;
#pragma unroll
      for (int k = 0; k < kBin0Max; ++k) lst |= (unsigned)((pushed >> k & 1) && clm[k] < stamp) << k;
      while (__any_sync(FULL, lst != 0)) {
        const int k = lst ? __ffs(lst) - 1 : 0;
        int v = vv[0], b = bb[0];
#pragma unroll
        for (int q = 1; q < kBin0Max; ++q) {
          v = k == q ? vv[q] : v;
          b = k == q ? bb[q] : b;
        }
        append_binned(1, lst != 0, v, b, rctr, a.R, nbase, a.rcap);
        lst &= lst - 1;
      }
    }
    if (Async) {
      // Release ownership, then re-check: a pusher that found u owned did not
      // enqueue it, so whichever of us sees the other's write re-enqueues
      // (store/fence/load against add/fence/atomicMax).
      if (valid) a.mark[u] = 0;
      __threadfence();
      bool again = valid && hu < n && ldcg(a.ex + u) > 0;
      activate(again, u, 0, stamp, nbase);  // (rows here have <= kBin0Max slots)
    } else {
      activate(live && hu < n && e_after > 0, u, 0, stamp, nbase);
    }
  }

  // Cooperative push for rows of more than kBin0Max slots, by a group of G
  // threads (a warp, or the whole CTA).  One scan finds the lowest residual
  // neighbour height bh (first minimum by slot order, kernels.py:40-48);
  // the excess is then pushed across every admissible slot at height bh in
  // slot order (ordered prefix sum of the residuals), which is what
  // successive KC steps would do while bh stays the minimum, in one pass.
  template <int G, bool Async>
  __device__ void push_coop(int u, unsigned stamp, const int *nbase, long long *s_red) {
    const int n = a.n;
    const int tid = G == 32 ? lane : threadIdx.x;
    int lo = __ldg(a.off + u), hi = __ldg(a.off + u + 1);
    const int ru = region(u);
    const bool pull = PP && ru == 1;  // pull side: deficit = -excess, reversed residuals
    int hu;
    long long eu;
    if (G == 32) {
      hu = __shfl_sync(FULL, lane == 0 ? ldcg(a.h + u) : 0, 0);
      eu = __shfl_sync(FULL, lane == 0 ? ldcg(a.ex + u) : 0ll, 0);
    } else {
      __syncthreads();
      if (threadIdx.x == 0) {
        s_red[0] = ldcg(a.h + u);
        s_red[1] = ldcg(a.ex + u);
      }
      __syncthreads();
      hu = (int)s_red[0];
      eu = s_red[1];
    }
    if (pull) eu = -eu;
    bool any_push = false;
    long long last_old = 0, last_total = 0;
    for (int cnt = 0; cnt < a.coop_kc; ++cnt) {  // (each step rescans the row)
      if (eu <= 0 || hu >= n) break;
      // ---- pass 1: (height, slot) argmin over residual slots, 4-way ILP
      unsigned long long best = ~0ull;
      for (int i0 = lo + tid; i0 < hi; i0 += 4 * G) {
        CapT c4[4];
        int v4[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          int i = i0 + r * G;
          c4[r] = i < hi ? (CapT)ldcg((const CapT *)(a.cf + i)) : (CapT)0;
          v4[r] = i < hi ? __ldg(a.adj + i) : 0;
          if (PP && i < hi) {
            if (pull) c4[r] = __ldg(a.pc + i) - c4[r];
            if (region(v4[r]) != ru) c4[r] = 0;
          }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (c4[r] > 0) {
            unsigned long long key = ((unsigned long long)(unsigned)ldcg(a.h + v4[r]) << 32) |
                                     (unsigned)(i0 + r * G - lo);
            best = key < best ? key : best;
          }
        }
      }
      best = warp_min_u64(best);
      if (G > 32) {
        __syncthreads();
        if (lane == 0) s_red[wib] = (long long)best;
        __syncthreads();
        best = ~0ull;
        for (int w = 0; w < G / 32; ++w) best = (unsigned long long)s_red[w] < best ? (unsigned long long)s_red[w] : best;
      }
      if (tid == 0) lc.bytes += Bytes<CapT>::kVertex + (unsigned long long)(hi - lo) * Bytes<CapT>::kSlot;
      if (best == ~0ull) {  // no residual out-edge
        hu = n;
        if (tid == 0) {
          a.h[u] = n;
          lc.relabels++;
        }
        break;
      }
      int bh = (int)(best >> 32);
      if (hu <= bh) {  // relabel from the scan snapshot
        hu = bh + 1 > n ? n : bh + 1;
        if (tid == 0) {
          a.h[u] = hu;
          lc.relabels++;
        }
        continue;
      }
      // ---- pass 2: push along slots at height bh, ordered by slot.  In a
      // CTA row each thread takes R = 4 consecutive slots (all loads in
      // flight together), so a chunk of 4G slots costs one ordered scan of
      // the per-thread sums (hub rows: a quarter of the dependent gathers and
      // CTA barriers); warp rows are short and keep one slot per lane
      constexpr int R = G > 32 ? 4 : 1;
      int first = lo + (int)(best & 0xFFFFFFFFu);
      long long carry = 0;  // residual of admissible slots before this chunk
      for (int i0 = first - ((first - lo) % (R * G)); i0 < hi && carry < eu; i0 += R * G) {
        const int ib = i0 + R * tid;
        long long c[R];
        int v[R], vb[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = ib + r;
          c[r] = 0;
          v[r] = 0;
          vb[r] = 0;
          if (i < hi && i >= first) {
            c[r] = (long long)ldcg((const CapT *)(a.cf + i));
            if (pull) c[r] = (long long)__ldg(a.pc + i) - c[r];
            v[r] = __ldg(a.adj + i);
          }
        }
        int hv[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          hv[r] = -1;
          if (c[r] > 0) {
            vb[r] = vbin(v[r]);  // in flight with the height
            hv[r] = ldcg(a.h + v[r]);
          }
        }
        long long tsum = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (hv[r] != bh || (PP && region(v[r]) != ru)) c[r] = 0;
          tsum += c[r];
        }
        long long incl = warp_incl_scan(tsum, lane), tot;
        if (G > 32) {
          __syncthreads();
          if (lane == 31) s_red[wib] = incl;
          __syncthreads();
          long long before = 0;
          tot = 0;
          for (int w = 0; w < G / 32; ++w) {
            long long x = s_red[w];
            if (w < wib) before += x;
            tot += x;
          }
          incl += before;
        } else {
          tot = __shfl_sync(FULL, incl, 31);
        }
        long long pre = incl - tsum;  // admissible residual before this thread's slots
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = ib + r;
          long long room = eu - carry - pre;
          long long amt = room <= 0 ? 0 : (room < c[r] ? room : c[r]);
          pre += c[r];
          bool act = false;
          if (amt > 0) {
            long long old;
            if (pull) {  // pull amt along (v, u)
              atomic_add(a.cf + __ldg(a.rev + i), (CapT)(-amt));
              atomic_add(a.cf + i, (CapT)amt);
              old = -atomic_add(a.ex + v[r], -amt);
            } else {
              atomic_add(a.cf + i, (CapT)(-amt));
              atomic_add(a.cf + __ldg(a.rev + i), (CapT)amt);
              old = add_excess(v[r], amt);
              if (!PP && a.strand && old < 0 && old + amt >= 0 && v[r] != a.t)
                fill_once();
            }
            act = old <= 0 && v[r] != a.s && v[r] != a.t;
            lc.pushes++;
            lc.bytes += Bytes<CapT>::kPush;
            if (Async && act) __threadfence();  // push visible before the hand-off
          }
          activate(act, v[r], vb[r], stamp, nbase);
        }
        carry += tot;
      }
      long long moved = carry < eu ? carry : eu;
      if (tid == 0 && moved > 0) {
        last_old = pull ? -atomic_add(a.ex + u, moved) : atomic_add(a.ex + u, -moved);
        last_total = moved;
      }
      any_push = any_push || moved > 0;
      eu -= moved;
      if (G > 32) __syncthreads();
    }
    bool self = false;
    if (tid == 0) {
      if (Async) {  // release ownership, then re-check (see push_thread)
        a.mark[u] = 0;
        __threadfence();
        self = hu < n && ldcg(a.ex + u) > 0;
      } else {  // self re-activation from the fresh value returned by the last atomic
        long long e_after = any_push ? last_old - last_total : eu;
        self = hu < n && e_after > 0;
      }
    }
    if (G == 32 || wib == 0) activate(self, u, bin_of(hi - lo), stamp, nbase);
    if (G > 32) __syncthreads();
  }

  // =========================================================================
  // repair (kernels.py:70-93): saturate steep residual edges h(u) > h(v)+1
  // =========================================================================
  // slots i, i + stride, ... i + 3 stride (< hi) of u with every load in
  // flight before any is consumed (one round trip per 4 slots, not per slot)
  __device__ __forceinline__ void repair_slots4(int u, int hu, int i, int stride, int hi, int ru) {
    CapT f[4];
    int v[4], hv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = i + k * stride;
      f[k] = j < hi ? (CapT)ldcg((const CapT *)(a.cf + j)) : (CapT)0;
      if (PP && ru == 1 && j < hi) f[k] = __ldg(a.pc + j) - f[k];  // cf(v -> u)
      v[k] = j < hi ? __ldg(a.adj + j) : 0;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) hv[k] = f[k] > 0 ? ldcg(a.h + v[k]) : INT_MAX - 1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = i + k * stride;
      if (f[k] > 0 && (!PP || region(v[k]) == ru) && hu > hv[k] + 1) {
        if (PP && ru == 1) repair_pull(u, v[k], j);
        else repair_push(u, v[k], j, j);
      }
    }
  }

  // saturate slot i of u (kernels.py:87-91)
  __device__ __forceinline__ void repair_push(int u, int v, int i, int i2) {
    CapT amt = atomic_exch(a.cf + i, (CapT)0);
    if (amt > 0) {
      atomic_add(a.cf + __ldg(a.rev + i2), amt);
      atomic_add(a.ex + u, -(long long)amt);
      add_excess(v, (long long)amt);
      lc.repairs++;
      lc.bytes += Bytes<CapT>::kPush;
    }
  }
  // force-pull the full residual of (v, u) (kernels.py:146-165)
  __device__ __forceinline__ void repair_pull(int u, int v, int i) {
    CapT amt = atomic_exch(a.cf + __ldg(a.rev + i), (CapT)0);
    if (amt > 0) {
      atomic_add(a.cf + i, amt);
      atomic_add(a.ex + u, (long long)amt);
      atomic_add(a.ex + v, -(long long)amt);
      lc.repairs++;
      lc.bytes += Bytes<CapT>::kPush;
    }
  }

  // Repair scope: every vertex the round's waves listed (solver.py:233), each
  // once -- the wave lists repeat a vertex every time it is re-activated, and
  // on R-MAT the hub rows come back wave after wave (each a 10^5-slot scan).
  __device__ void repair(const int *end) {
    __shared__ int s_ok;
    const unsigned rs = s_rep_stamp;
    for (int j = gtid; j < end[0]; j += gthreads) {  // thread per row, loads batched
      int u = ldcg(a.R[0] + j);
      if (u < 0) continue;  // reserved slot never filled (queue overflow)
      if (atomicMax((unsigned *)a.bmark + u, rs) >= rs) continue;  // (repaired this round)
      int lo = __ldg(a.off + u), d = __ldg(a.off + u + 1) - lo;
      int hu = ldcg(a.h + u);
      const int ru = region(u);
      lc.bytes += Bytes<CapT>::kVertex + (unsigned long long)d * Bytes<CapT>::kSlot;
      int vv[kBin0Max], hv[kBin0Max];
      CapT cc[kBin0Max];
#pragma unroll
      for (int k = 0; k < kBin0Max; ++k) {
        vv[k] = k < d ? __ldg(a.adj + lo + k) : 0;
        cc[k] = k < d ? (CapT)ldcg((const CapT *)(a.cf + lo + k)) : (CapT)0;
      }
    if (PP) {
#pragma unroll
      for (int k = 0; k < kBin0Max; ++k) {
        if (k < d && ru == 1) cc[k] = __ldg(a.pc + lo + k) - cc[k];  // cf(v -> u)
        if (k < d && region(vv[k]) != ru) cc[k] = 0;
      }
    }
#pragma unroll
      for (int k = 0; k < kBin0Max; ++k) hv[k] = cc[k] > 0 ? ldcg(a.h + vv[k]) : INT_MAX - 1;
#pragma unroll
      for (int k = 0; k < kBin0Max; ++k) {
        if (cc[k] > 0 && hu > hv[k] + 1) {
          if (PP && ru == 1) repair_pull(u, vv[k], lo + k);
          else repair_push(u, vv[k], lo + k, lo + k);
        }
      }
    }
    for (int j = gwarp; j < end[1]; j += gwarps) {
      int u = ldcg(a.R[1] + j);
      if (u < 0) continue;
      int fresh = lane == 0 ? atomicMax((unsigned *)a.bmark + u, rs) < rs : 0;
      if (!__shfl_sync(FULL, fresh, 0)) continue;
      int lo = __ldg(a.off + u), hi = __ldg(a.off + u + 1);
      int hu = ldcg(a.h + u);
      if (lane == 0) lc.bytes += Bytes<CapT>::kVertex + (unsigned long long)(hi - lo) * Bytes<CapT>::kSlot;
      for (int i = lo + lane; i < hi; i += 4 * 32) repair_slots4(u, hu, i, 32, hi, region(u));
    }
    for (int b = 2; b < NBIN; ++b) {
      for (int j = blockIdx.x; j < end[b]; j += gridDim.x) {
        int u = ldcg(a.R[b] + j);
        if (u < 0) continue;  // (uniform across the CTA: same slot)
        __syncthreads();
        if (threadIdx.x == 0) s_ok = atomicMax((unsigned *)a.bmark + u, rs) < rs;
        __syncthreads();
        if (!s_ok) continue;
        int lo = __ldg(a.off + u), hi = __ldg(a.off + u + 1);
        int hu = ldcg(a.h + u);
        if (threadIdx.x == 0)
          lc.bytes += Bytes<CapT>::kVertex + (unsigned long long)(hi - lo) * Bytes<CapT>::kSlot;
        for (int i = lo + threadIdx.x; i < hi; i += 4 * blockDim.x)
          repair_slots4(u, hu, i, blockDim.x, hi, region(u));
      }
    }
  }

  // =========================================================================
  // excess walk (thin active sets): right after an exact global relabel,
  // carry each active vertex's excess down the BFS layers (h(v) == h(u) - 1)
  // to a base in one pass -- a waves-only round moves excess one hop per
  // grid barrier, so a few far-away active vertices would need several
  // rounds (a full global relabel each) for a ~100-hop path.  Each step
  // claims min(carry, cf) by CAS, so concurrent walkers never overdraw a
  // slot; pushes go downhill along exact labels (no relabel, the labeling
  // stays valid).  A walker stops at a base, at a long row (left to the
  // waves) or where the slots below were taken; what it leaves behind is
  // ordinary excess for the waves and the next global relabel.
  // =========================================================================
  // s0: the stamp that marks wave 0 of this round (the BFS set it on every
  // listed active vertex); a walker that stops short lists its stopping
  // vertex for wave 0 too, once.
  __device__ void walk(int cnt0, unsigned s0) {
    for (int j = gtid; j < cnt0; j += gthreads) {
      int u = ldcg(a.R[0] + j);
      if (u < 0) continue;
      int hu = ldcg(a.h + u);
      long long carry = ldcg(a.ex + u);
      int d = 0;
      bool moved = false;
      for (int step = 0; step < a.n && hu > 0 && hu < a.n && carry > 0; ++step) {
        const int lo = __ldg(a.off + u);
        d = __ldg(a.off + u + 1) - lo;
        if (d > kBin0Max) break;
        int pick = -1, v = 0;
        CapT c = 0;
        for (int k = 0; k < d && pick < 0; ++k) {
          CapT ck = (CapT)ldcg((const CapT *)(a.cf + lo + k));
          if (ck > 0) {
            int w = __ldg(a.adj + lo + k);
            if (ldcg(a.h + w) == hu - 1) {
              pick = lo + k;
              v = w;
              c = ck;
            }
          }
        }
        if (pick < 0) break;
        long long take = 0;
        for (CapT cur = c;;) {  // claim
          take = carry < (long long)cur ? carry : (long long)cur;
          if (take <= 0) break;
          CapT prev = atomic_cas(a.cf + pick, cur, (CapT)(cur - (CapT)take));
          if (prev == cur) break;
          cur = prev;
        }
        if (take <= 0) break;
        atomic_add(a.cf + __ldg(a.rev + pick), (CapT)take);
        atomic_add(a.ex + u, -take);
        const long long vold = add_excess(v, take);
        if (!PP && a.strand && vold < 0 && vold + take >= 0 && v != a.t)
          fill_once();
        lc.pushes++;
        lc.bytes += Bytes<CapT>::kVertex + (unsigned long long)d * Bytes<CapT>::kSlot +
                    Bytes<CapT>::kPush;
        carry = take;
        u = v;
        hu -= 1;
        moved = true;
      }
      if (moved && hu > 0 && hu < a.n && u != a.t && atomicMax(a.mark + u, s0) < s0) {
        const int b = bin_of(d > 0 ? d : __ldg(a.off + u + 1) - __ldg(a.off + u));
        const int p = sy.s_snap[C_RNEXT + b] + atomicAdd(a.ctrl->live + C_RNEXT + b, 1);
        if (p < a.rcap) a.R[b][p] = u;
        else a.ctrl->overflow = 1;
      }
    }
  }

  // Thin waves (<= tail_local items, no CTA-wide rows) run in CTA 0 alone,
  // wave after wave with __syncthreads between them instead of a grid
  // barrier, while the rest of the grid waits at the next barrier.  A single
  // CTA processing a wave is one schedule of it; the wave stamps keep every
  // vertex in at most one wave at a time exactly as in grid mode.  Leaves
  // the pending wave's counts in the live counters (snapshotted by the
  // barrier) and publishes base / waves / stamp for the other CTAs.
  __device__ void tail_waves(int *base, int *cnt, int &waves, unsigned &stamp, int max_waves,
                             int *nbase, long long *s_red) {
    __shared__ int s_cnt[NBIN];
    __shared__ int s_go;
    __shared__ int s_rc[NBIN];  // this CTA alone appends: list counters in shared memory
    // thread 0's stop-test inputs, read once: the push phase's deadline and
    // the fills so far (only this CTA pushes until the tail waves end)
    unsigned long long wdl = 0, fills0 = 0;
    if (threadIdx.x == 0) {
      sy.t_tail = globaltimer();
      wdl = ((volatile Ctrl *)a.ctrl)->wave_deadline;
      fills0 = ((volatile Ctrl *)a.ctrl)->fills;
      s_fills = 0;
    }
    if (threadIdx.x < NBIN) s_rc[threadIdx.x] = 0;
    rctr = s_rc;
    for (;;) {
      const unsigned next = ++stamp;
      __syncthreads();
      if (threadIdx.x < NBIN) nbase[threadIdx.x] = base[threadIdx.x] + cnt[threadIdx.x];
      __syncthreads();
      int lim[NBIN];
      for (int b = 0; b < NBIN; ++b) {
        lim[b] = base[b] + cnt[b];
        if (lim[b] > a.rcap) lim[b] = a.rcap;
      }
      for (int j0 = base[0] + wib * 32; j0 < lim[0]; j0 += kWarps * 32) {
        const int j = j0 + lane;
        const bool valid = j < lim[0];
        push_thread<false>(valid, valid ? ldcg(a.R[0] + j) : 0, next, nbase);
      }
      for (int j = base[1] + wib; j < lim[1]; j += kWarps)
        push_coop<32, false>(ldcg(a.R[1] + j), next, nbase, s_red);
      stage_flush(1, s_rc, a.R[0], nbase[0], a.rcap);
      __syncthreads();  // (also orders this CTA's list writes before the next wave reads them)
      ++waves;
      if (threadIdx.x == 0) {
        int tot = 0;
        for (int b = 0; b < NBIN; ++b) {
          s_cnt[b] = s_rc[b];
          tot += s_cnt[b];
        }
        if (sy.trace && sy.trace_n < sy.trace_cap) {  // (CTA 0 holds the trace) phase-5 entry per wave
          const unsigned long long now = globaltimer();
          sy.trace[sy.trace_n++] = (5ull << 60) | ((unsigned long long)(tot & 0xFFFFFFF) << 32) |
                                   ((now - sy.t_tail) & 0xFFFFFFFFull);
          sy.t_tail = now;
        }
        const bool go = tot > 0 && tot <= a.tail_local && s_cnt[1] <= kWarps && s_cnt[2] == 0 &&
                        s_cnt[3] == 0 &&
                        (waves < max_waves || (tot <= a.tail_items && waves < a.tail_cap)) &&
                        !(a.wave_time > 0 && wdl != 0 && globaltimer() > wdl) &&
                        !(!PP && a.strand && sy.s_snap[C_TALIVE] == 0 &&
                          fills0 + s_fills >= (unsigned)sy.s_snap[C_DBASES]);
        // consumed here: the next wave appends from zero; else the pending
        // wave's counts go to the live counters the grid barrier snapshots
        for (int b = 0; b < NBIN; ++b) {
          if (!go) a.ctrl->live[C_RNEXT + b] = s_rc[b];
          s_rc[b] = 0;
        }
        s_go = go;
      }
      __syncthreads();
      for (int b = 0; b < NBIN; ++b) {
        base[b] += cnt[b];
        cnt[b] = s_cnt[b];
      }
      if (!s_go) break;
    }
    rctr = a.ctrl->live + C_RNEXT;
    if (threadIdx.x == 0) {
      for (int b = 0; b < NBIN; ++b) a.ctrl->tail_base[b] = base[b];
      a.ctrl->tail_waves = waves;
      a.ctrl->tail_stamp = stamp;
    }
  }

  // one round's push phase + repair; wave 0 = the active list in R
  __device__ void push_round(unsigned &stamp, unsigned long long *scr, int max_waves) {
    __shared__ int nbase[NBIN];
    __shared__ long long s_red[kWarps + 2];
    int base[NBIN], cnt[NBIN];
    for (int b = 0; b < NBIN; ++b) {
      base[b] = 0;
      cnt[b] = sy.s_snap[C_RNEXT + b];
    }
    int waves = 0;
    if (gtid == 0) {  // (read by the wave barriers' leaders)
      const unsigned long long now = globaltimer();
      a.ctrl->wave_deadline =
          a.wave_time > 0 ? now + (now - a.ctrl->bfs_t0) * (unsigned long long)a.wave_time / 8 : 0;
    }
    for (;;) {
      // (only short rows: a warp-wide row in CTA 0 alone would idle the grid)
      if (a.tail_local > 0 && cnt[0] + cnt[1] <= a.tail_local && cnt[1] <= kWarps &&
          cnt[2] == 0 && cnt[3] == 0 && cnt[0] + cnt[1] > 0) {
        if (blockIdx.x == 0) tail_waves(base, cnt, waves, stamp, max_waves, nbase, s_red);
        grid_sync(a.ctrl, sy, 0xFu << C_RNEXT, 0, 0, PH_PUSH);
        int tot = 0;
        for (int b = 0; b < NBIN; ++b) {  // adopt CTA 0's wave state
          base[b] = ldcg(a.ctrl->tail_base + b);
          cnt[b] = sy.s_snap[C_RNEXT + b];
          tot += cnt[b];
        }
        waves = ldcg(&a.ctrl->tail_waves);
        stamp = (unsigned)ldcg((const int *)&a.ctrl->tail_stamp);
        if (tot == 0 || *sy.s_abort || sy.s_snap[C_STOP]) break;
        if (waves >= max_waves && (tot > a.tail_items || waves >= a.tail_cap)) break;
        continue;
      }
      unsigned next = ++stamp;
      __syncthreads();
      if (threadIdx.x < NBIN) nbase[threadIdx.x] = base[threadIdx.x] + cnt[threadIdx.x];
      __syncthreads();
      int lim[NBIN];
      for (int b = 0; b < NBIN; ++b) {
        lim[b] = base[b] + cnt[b];
        if (lim[b] > a.rcap) lim[b] = a.rcap;
      }
      for (int j0 = base[0] + gwarp * 32; j0 < lim[0]; j0 += gwarps * 32) {
        int j = j0 + lane;
        bool valid = j < lim[0];
        push_thread<false>(valid, valid ? ldcg(a.R[0] + j) : 0, next, nbase);
      }
      for (int j = base[1] + gwarp; j < lim[1]; j += gwarps)
        push_coop<32, false>(ldcg(a.R[1] + j), next, nbase, s_red);
      for (int b = 2; b < NBIN; ++b)
        for (int j = base[b] + blockIdx.x; j < lim[b]; j += gridDim.x)
          push_coop<kBlock, false>(ldcg(a.R[b] + j), next, nbase, s_red);
      stage_flush(1, a.ctrl->live + C_RNEXT, a.R[0], nbase[0], a.rcap);
      if (a.trace) {  // trace: CTA 0's own share of the wave done (phase-4 entry)
        __syncthreads();
        if (blockIdx.x == 0 && threadIdx.x == 0 && sy.trace_n < sy.trace_cap)
          sy.trace[sy.trace_n++] = (4ull << 60) | ((globaltimer() - sy.t_last) & 0xFFFFFFFFull);
      }
      // (the sink's excess and the counters are published once per round:
      // nothing reads them between waves, and the ceiling check may lag a
      // round)
      grid_sync(a.ctrl, sy, 0xFu << C_RNEXT, 0, 0, PH_PUSH);
      ++waves;
      int tot = 0;
      for (int b = 0; b < NBIN; ++b) {
        base[b] = base[b] + cnt[b];
        cnt[b] = sy.s_snap[C_RNEXT + b];
        tot += cnt[b];
      }
      // past the budget, keep going while the waves stay small (a thin wave
      // costs ~1 % of a global relabel) up to tail_cap waves
      if (tot == 0 || *sy.s_abort || sy.s_snap[C_STOP]) break;
      if (waves >= max_waves && (tot > a.tail_items || waves >= a.tail_cap)) break;
    }
    int end[NBIN];
    for (int b = 0; b < NBIN; ++b) {
      end[b] = base[b] + cnt[b];
      if (end[b] > a.rcap) end[b] = a.rcap;
    }
    repair(end);
    sink_flush();
    flush_counters(a.ctrl, lc, scr);
    if (gtid == 0) {
      a.ctrl->waves += waves;
      a.ctrl->rounds += 1;
      for (int b = 0; b < NBIN; ++b) a.rdirty[b] = end[b];
    }
    // the barrier also clears the wave counters left by the last wave
    grid_sync(a.ctrl, sy, 0xFu << C_RNEXT, 0, 0, PH_REPAIR);
  }

  // -------------------------------------------------------------------------
  // asynchronous push phase: the R lists are work queues (tail = BFS count +
  // appended, head = claimed, -1 = reserved but not yet written).  Light
  // vertices are claimed 32 at a time by a warp, bin-1 rows one per warp,
  // heavy rows one per CTA.  A vertex is owned while its mark equals the
  // phase stamp: activation is atomicMax(mark, ep) < ep, and the owner
  // releases (mark = 0) and re-checks its excess after processing, so every
  // vertex with positive excess is queued at most once at any time.  The
  // phase ends when every queued item is done (quiescence: done read before
  // tail), or after a work budget (then the next global relabel re-derives
  // the active set), with no barrier per hop.
  // -------------------------------------------------------------------------
  __device__ __forceinline__ int claim_one(int b, const int *nbase) {
    unsigned *hp = a.ctrl->aq_head + b;
    for (int tries = 0; tries < 64; ++tries) {
      unsigned h = ld_acquire_u32(hp);
      unsigned t = (unsigned)nbase[b] + (unsigned)ldcg(a.ctrl->live + C_RNEXT + b);
      if (h >= t || (int)h >= a.rcap) return -1;
      if (atomicCAS(hp, h, h + 1) == h) return (int)h;
    }
    return -1;
  }

  __device__ __forceinline__ int wait_slot(const int *list, int slot) {
    int x;
    while ((x = ldcg(list + slot)) < 0) __nanosleep(32);
    return x;
  }

  // 0 = continue, 1 = quiescent, 2 = stopped (budget), 3 = stopped elsewhere,
  // 4 = overflow, 5 = watchdog
  __device__ int async_state(const int *nbase, long long budget, unsigned *dd, unsigned *tt) {
    unsigned d = 0, t = 0;
#pragma unroll
    for (int b = 0; b < NBIN; ++b) d += ld_acquire_u32(a.ctrl->aq_done + b);
#pragma unroll
    for (int b = 0; b < NBIN; ++b) t += (unsigned)nbase[b] + (unsigned)ldcg(a.ctrl->live + C_RNEXT + b);
    *dd = d;
    *tt = t;
    if (d == t) return 1;
    volatile Ctrl *vc = a.ctrl;
    if (vc->overflow) return 4;
    // leave headroom in the queues: end the phase (global relabel) well before
    // a list could overflow (an in-flight warp publishes at most 32 + 8*32 items)
    if ((unsigned)nbase[0] + (unsigned)ldcg(a.ctrl->live + C_RNEXT) > (unsigned)(a.rcap - a.rcap / 8)) {
      vc->aq_stop = 1;
      return 2;
    }
    if (vc->aq_stop || vc->abort) return 3;
    if ((long long)d >= budget) {
      vc->aq_stop = 1;
      return 2;
    }
    if (globaltimer() > sy.deadline) {
      vc->abort = 1;
      vc->status = 6;
      return 5;
    }
    return 0;
  }

  __device__ void push_round_async(unsigned &stamp, unsigned long long *scr) {
    __shared__ int nbase[NBIN];
    __shared__ long long s_red[kWarps + 2];
    __shared__ int s_item, s_bin, s_state;
    __shared__ unsigned s_d, s_t;
    const unsigned ep = ++stamp;  // the BFS marked the queued vertices with this stamp
    long long active0 = 0;
    for (int b = 0; b < NBIN; ++b) active0 += sy.s_snap[C_RNEXT + b];
    const long long budget = (long long)a.async_budget * active0 + 4096;
    if (threadIdx.x < NBIN) nbase[threadIdx.x] = sy.s_snap[C_RNEXT + threadIdx.x];
    __syncthreads();
    int my_slot = 0;
    bool pend = false;
    for (;;) {
      // ---- heavy rows: one per CTA
      if (threadIdx.x == 0) {
        s_item = -1;
        for (int b = NBIN - 1; b >= 2 && s_item < 0; --b) {
          int x = claim_one(b, nbase);
          if (x >= 0) {
            s_item = x;
            s_bin = b;
          }
        }
      }
      __syncthreads();
      bool progress = false;
      if (s_item >= 0) {
        const int hb = s_bin;
        __shared__ int s_u;
        if (threadIdx.x == 0) s_u = wait_slot(a.R[hb], s_item);
        __syncthreads();
        push_coop<kBlock, true>(s_u, ep, nbase, s_red);
        stage_flush(1, a.ctrl->live + C_RNEXT, a.R[0], nbase[0], a.rcap);
        __syncthreads();
        if (threadIdx.x == 0) {
          __threadfence();
          atomicAdd(a.ctrl->aq_done + hb, 1u);
        }
        progress = true;
      } else {
        // ---- bin-1 rows: one per warp
        int x1 = -1;
        if (lane == 0) x1 = claim_one(1, nbase);
        x1 = __shfl_sync(FULL, x1, 0);
        if (x1 >= 0) {
          int u = 0;
          if (lane == 0) u = wait_slot(a.R[1], x1);
          u = __shfl_sync(FULL, u, 0);
          push_coop<32, true>(u, ep, nbase, s_red);
          stage_flush(1, a.ctrl->live + C_RNEXT, a.R[0], nbase[0], a.rcap);
          if (lane == 0) {
            __threadfence();
            atomicAdd(a.ctrl->aq_done + 1, 1u);
          }
          progress = true;
        }
        // ---- light vertices: a batch of 32 queue slots per warp
        if (!__any_sync(FULL, pend)) {
          unsigned c = 0;
          if (lane == 0) c = atomicAdd(a.ctrl->aq_head + 0, 32u);
          c = __shfl_sync(FULL, c, 0);
          my_slot = (int)(c + lane);
          pend = my_slot < a.rcap;
        }
        int item = pend ? ldcg(a.R[0] + my_slot) : -1;
        bool ready = item >= 0;
        unsigned rb = __ballot_sync(FULL, ready);
        if (rb) {
          push_thread<true>(ready, ready ? item : 0, ep, nbase);
          stage_flush(1, a.ctrl->live + C_RNEXT, a.R[0], nbase[0], a.rcap);
          if (lane == 0) {
            __threadfence();
            atomicAdd(a.ctrl->aq_done + 0, (unsigned)__popc(rb));
          }
          pend = pend && !ready;
          progress = true;
        }
      }
      if (!__syncthreads_or(progress)) __nanosleep(200);
      if (threadIdx.x == 0) s_state = async_state(nbase, budget, &s_d, &s_t);
      __syncthreads();
      if (s_state != 0) break;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && sy.trace && sy.trace_n < sy.trace_cap)
      sy.trace[sy.trace_n++] = (7ull << 60) | ((unsigned long long)(s_state & 0xF) << 56) |
                               ((unsigned long long)(s_d & 0xFFFFFFFu) << 28) | (s_t & 0xFFFFFFFu);
    sink_flush();
    flush_counters(a.ctrl, lc, scr);
    grid_sync(a.ctrl, sy, 0, 0, 0, PH_PUSH);
    // repair (kernels.py:70-93) over every vertex taken from the queues
    __shared__ int s_end[NBIN];
    if (threadIdx.x < NBIN) {
      int b = threadIdx.x;
      int hd = (int)ldcg((const int *)(a.ctrl->aq_head + b));
      int tl = nbase[b] + ldcg(a.ctrl->live + C_RNEXT + b);
      int e = hd < tl ? hd : tl;
      s_end[b] = e < a.rcap ? e : a.rcap;
    }
    __syncthreads();
    int end[NBIN];
    for (int b = 0; b < NBIN; ++b) end[b] = s_end[b];
    repair(end);
    sink_flush();
    flush_counters(a.ctrl, lc, scr);
    if (gtid == 0) {
      unsigned d = 0;
      for (int b = 0; b < NBIN; ++b) {
        d += ldcg((const int *)(a.ctrl->aq_done + b));
        int tl = nbase[b] + ldcg(a.ctrl->live + C_RNEXT + b);
        a.rdirty[b] = tl < a.rcap ? tl : a.rcap;
      }
      a.ctrl->async_items += d;
      a.ctrl->waves += 1;
      a.ctrl->rounds += 1;
    }
    grid_sync(a.ctrl, sy, 0xFu << C_RNEXT, 0, 0, PH_REPAIR);
  }

  // =========================================================================
  // flow (dynamic.py:141-143) and cut certificate (solver.py:178-184)
  // =========================================================================
  // slot i of a row on the walked side, head height hv: its share of the cut
  __device__ __forceinline__ long long cut_slot(bool bside, int hv, int i) const {
    if (bside) return hv == a.n ? (long long)__ldg(a.cap0 + __ldg(a.rev + i)) : 0ll;
    return hv != a.n ? (long long)__ldg(a.cap0 + i) : 0ll;
  }
  __device__ void finalize(long long *scr) {
    const int n = a.n;
    long long f = 0;
    int nb = sy.s_snap[C_BASES];
    for (int j = gtid; j < nb; j += gthreads) f += ldcg(a.ex + ldcg(a.bases + j));
    f = block_sum(f, scr);
    if (threadIdx.x == 0 && f) atomicAdd((unsigned long long *)&a.ctrl->flow, (unsigned long long)f);
    // cut = sum of cap0 over A -> B slots, A = {h == n}.  Walked from the
    // smaller side: A-side rows sum their slots into B; B-side rows (when the
    // last relabel reached fewer than n/2 vertices, e.g. C4 whose sink side
    // is a corner) sum the reverse slots of their slots out of A.  Light rows
    // inline; heavy rows (CTA each) listed from the front of `heavy`, huge
    // rows (> kBin2Max slots, e.g. the source of the grid config with ~2.1 M
    // slots; whole grid each) from the back.
    const int reached = sy.s_snap[C_REACHED];
    const bool bside = reached > 0 && 2ll * reached < (long long)n;
    // tracked launches walk the B side straight from the reached-set list
    const bool from_list = bside && s_tl_ok;
    const int *Lc = from_list ? tl_old() : nullptr;  // (flipped: the final relabel's)
    long long c = 0;
    for (int j = gtid; j < (from_list ? reached : n); j += gthreads) {
      const int u = from_list ? ldcg(Lc + j) : j;
      if (!from_list && (ldcg(a.h + u) != n) != bside) continue;
      int lo = __ldg(a.off + u), hi = __ldg(a.off + u + 1);
      if (hi - lo > 64) {
        if (hi - lo > kBin2Max) a.heavy[n - 1 - atomicAdd(a.ctrl->live + C_HUGE, 1)] = u;
        else a.heavy[atomicAdd(a.ctrl->live + C_HEAVY, 1)] = u;
        continue;
      }
      if (hi - lo <= kBin0Max) {  // short rows: every load in flight together
        int vv[kBin0Max], hv[kBin0Max];
#pragma unroll
        for (int k = 0; k < kBin0Max; ++k) vv[k] = lo + k < hi ? __ldg(a.adj + lo + k) : -1;
#pragma unroll
        for (int k = 0; k < kBin0Max; ++k) hv[k] = vv[k] >= 0 ? ldcg(a.h + vv[k]) : bside ? 0 : n;
#pragma unroll
        for (int k = 0; k < kBin0Max; ++k) c += cut_slot(bside, hv[k], lo + k);
        continue;
      }
      for (int i = lo; i < hi; ++i) c += cut_slot(bside, ldcg(a.h + __ldg(a.adj + i)), i);
    }
    grid_sync(a.ctrl, sy, (1u << C_HEAVY) | (1u << C_HUGE), 0, 0, PH_FINAL);
    int nh = sy.s_snap[C_HEAVY], ng = sy.s_snap[C_HUGE];
    for (int j = blockIdx.x; j < nh; j += gridDim.x) {
      int u = ldcg(a.heavy + j);
      int lo = __ldg(a.off + u), hi = __ldg(a.off + u + 1);
      for (int i = lo + threadIdx.x; i < hi; i += blockDim.x)
        c += cut_slot(bside, ldcg(a.h + __ldg(a.adj + i)), i);
    }
    for (int j = 0; j < ng; ++j) {
      int u = ldcg(a.heavy + n - 1 - j);
      int lo = __ldg(a.off + u), hi = __ldg(a.off + u + 1);
      for (int i = lo + gtid; i < hi; i += gthreads)
        c += cut_slot(bside, ldcg(a.h + __ldg(a.adj + i)), i);
    }
    c = block_sum(c, scr);
    if (threadIdx.x == 0 && c) atomicAdd((unsigned long long *)&a.ctrl->cut, (unsigned long long)c);
  }
};

#ifndef MFX_MIN_BLOCKS
#define MFX_MIN_BLOCKS 2
#endif

template <typename CapT, bool PP>
__global__ void __launch_bounds__(kBlock, MFX_MIN_BLOCKS)
    solve_kernel(const __grid_constant__ SolveArgs<CapT> a) {
  __shared__ int s_snap[C_NCTR];
  __shared__ int s_abort;
  __shared__ unsigned long long scr[kWarps];
  __shared__ WarpQ wq[kWarps];
  __shared__ long long s_sink;
  if (a.gate && (a.gate[0] != LLONG_MAX || a.gate[1] != LLONG_MAX || a.gate[3] != LLONG_MAX ||
                 a.gate[4] != LLONG_MAX))
    return;  // the batch was rejected: state untouched, nothing to solve
  Sync sy;
  Local lc;
  if (threadIdx.x == 0) {
    volatile Ctrl *vc = a.ctrl;
    sy.gen = vc->bar_gen;
    sy.deadline = vc->deadline_ns;
    sy.ceiling = vc->ceiling;
    sy.strand = a.strand;
    for (int i = 0; i < C_NCTR; ++i) s_snap[i] = vc->snap[i];
    s_abort = vc->abort;
    sy.t_last = globaltimer();
    for (int i = 0; i < PH_N; ++i) sy.ph[i] = 0;
    sy.trace = blockIdx.x == 0 ? a.trace : nullptr;
    sy.trace_cap = a.trace_cap;
    sy.trace_n = 0;
    s_sink = 0;
    s_tl_cur = vc->tl_cur & 1;
    s_tl_ok = a.sparse == 1;
    s_tl_trk = 0;
  }
  if ((threadIdx.x & 31) == 0)
    wq[threadIdx.x >> 5].cnt[0] = wq[threadIdx.x >> 5].cnt[1] = wq[threadIdx.x >> 5].cnt[2] = 0;
  sy.s_snap = s_snap;
  sy.s_abort = &s_abort;
  __syncthreads();
  Kern<CapT, PP> k(a, sy, lc, wq, &s_sink);
  unsigned stamp = *(volatile unsigned *)a.stamp;  // persistent wave stamp
  unsigned bstamp = ((volatile unsigned *)a.stamp)[1];  // persistent BFS epoch stamp
  if (a.what == WHAT_BARRIER) {  // barrier latency microbenchmark (kc iterations)
    for (int i = 0; i < a.kc && !s_abort; ++i) grid_sync(a.ctrl, sy, 0, 0, 0, PH_FINAL);
  } else {
    // One call site per phase routine: everything inlines into the kernel
    // and the Kern state stays in registers (a second call site of bfs or
    // push_round made nvcc outline it and spill the whole object to local
    // memory).
    const bool do_bfs = a.what == WHAT_SOLVE || a.what == WHAT_BFS;
    const bool do_push = a.what == WHAT_SOLVE || a.what == WHAT_ROUND;
    int L = (int)((volatile Ctrl *)a.ctrl)->last_levels;
    bool first_bfs = true;
    for (; do_bfs || do_push;) {
      if (do_bfs) {
        // early exit (stop once every excess holder is labelled; C4
        // dynamic 25 -> 16.5 ms/batch) in solve rounds only: the bit-exact
        // global relabel entry point, WHAT_BFS, never takes it
        // (push-pull: the region relabels stop once every active of both
        // sides is labelled -- C4's pull side is the whole 24 M-vertex A
        // side, its few deficits sit next to the excess that feeds them)
        const bool early = a.what == WHAT_SOLVE && !a.topology && (a.early || (a.flags & 4) != 0);
        L = k.bfs(stamp + 1, bstamp, a.bfs_local, early, early && !first_bfs && !PP,
                  first_bfs && a.bk > 0);
        first_bfs = false;
        int act = s_snap[C_ACTIVE];
        if (k.gtid == 0) a.ctrl->active = act;
        // with the walk enabled the BFS stamped the listed active vertices
        // with stamp + 1 (wave 0); this round's wave stamps start above it
        const bool marked = !PP && !a.async && a.walk_max > 0;
        if (marked) ++stamp;
        if (act == 0 || s_abort || !do_push) break;
        if (marked && !a.topology && act <= a.walk_max && L >= a.walk_depth) {
          k.walk(s_snap[C_RNEXT], stamp);
          k.sink_flush();
          // stopping vertices join wave 0 (accumulate the list counters)
          grid_sync(a.ctrl, sy, 0, 0xFu << C_RNEXT, 0, PH_PUSH);
        }
      }
      ++bstamp;  // (every thread: this round's repair stamp)
      if (threadIdx.x == 0) s_rep_stamp = bstamp;
      __syncthreads();
      if (a.async) k.push_round_async(stamp, scr);
      else {
        int budget = a.max_waves > 0 ? a.max_waves : a.wave_mult * L / 4 + a.wave_add;
        // after a demand-covered relabel exit the few labelled holders must
        // cross their whole distance (<= L hops) to the deficits: the usual
        // L/2 budget would stop them halfway and the next relabel could not
        // stop early (the deficit did not shrink), so it would run to the far
        // holders (C4: one 35 ms relabel per such batch)
        if (s_snap[C_EFILL] && budget < 4 * L + 8) budget = 4 * L + 8;
        k.push_round(stamp, scr, budget);
      }
      if (s_abort || !do_bfs) break;
    }
    flush_counters(a.ctrl, lc, scr);
    bool final = a.what == WHAT_FINAL || (a.what == WHAT_SOLVE && !s_abort);
    if (final && !PP) k.finalize((long long *)scr);  // (the pipelines end in ordinary rounds)
  }
  if (k.gtid == 0) {  // persistent stamps (every thread advanced identical copies)
    a.stamp[0] = stamp;
    a.stamp[1] = bstamp;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // device phase times (block 0's view)
    unsigned long long now = globaltimer();
    sy.ph[PH_FINAL] += now - sy.t_last;
    for (int i = 0; i < PH_N; ++i) a.ctrl->phase_ns[i] += sy.ph[i];
    if (sy.trace) a.ctrl->trace_n = sy.trace_n;
  }
}

// push-pull set-up (dynamic.py:178-192, 316-318): the prior cut's A side =
// {h == n} from the terminated state, and every A->B residual pushed across
template <typename CapT>
__global__ void pp_region_kernel(const int *h, int n, uint8_t *reg) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    reg[v] = h[v] == n;
}

// Slot-parallel (the source row of C2 alone holds 2.1 M slots): the tail of a
// candidate slot (residual into B) is found by binary search of the row
// offsets, and a warp whose slots share one tail adds its excess change once.
template <typename CapT>
__global__ void pp_crossing_kernel(const int *__restrict__ off, const int *__restrict__ adj,
                                   const int *__restrict__ rev, const uint8_t *__restrict__ reg,
                                   CapT *cf, long long *ex, int n, int S, const long long *gate) {
  if (gate && (gate[0] != LLONG_MAX || gate[1] != LLONG_MAX || gate[3] != LLONG_MAX ||
               gate[4] != LLONG_MAX))
    return;
  for (int i0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; i0 < S;
       i0 += gridDim.x * blockDim.x) {
    const int i = i0 + (threadIdx.x & 31);
    CapT c = 0;
    int u = -1;
    if (i < S) {
      c = cf[i];
      if (c > 0 && !reg[adj[i]]) {
        int lo = 0, hi = n;  // last row with off[row] <= i
        while (hi - lo > 1) {
          int mid = (lo + hi) >> 1;
          if (off[mid] <= i) lo = mid;
          else hi = mid;
        }
        u = reg[lo] ? lo : -1;
      }
    }
    if (u >= 0) {
      cf[i] = 0;
      atomic_add(cf + rev[i], c);
      atomic_add(ex + adj[i], (long long)c);
    }
    const unsigned any = __ballot_sync(0xffffffffu, u >= 0);
    if (!any) continue;
    const int u0 = __shfl_sync(0xffffffffu, u, __ffs(any) - 1);
    if (__all_sync(0xffffffffu, u < 0 || u == u0)) {
      long long tot = warp_sum(u >= 0 ? (long long)c : 0ll);
      if ((threadIdx.x & 31) == 0) atomic_add(ex + u0, -tot);
    } else if (u >= 0) {
      atomic_add(ex + u, -(long long)c);
    }
  }
}

template <typename CapT>
static cudaError_t launch_pp_setup_t(const GraphObj &g, StateObj &st, bool crossing,
                                     const long long *gate) {
  Topology &T = *g.topo;
  cudaError_t e = ensure_workspace(T);
  if (e) return e;
  int grid = T.num_sms * 8;
  if (!crossing) pp_region_kernel<CapT><<<grid, kBlock, 0, T.stream>>>(st.h, T.n, T.ws.reg);
  else
    pp_crossing_kernel<CapT><<<grid, kBlock, 0, T.stream>>>(T.off, T.adj, T.rev, T.ws.reg,
                                                           (CapT *)st.cf, st.ex, T.n, T.S, gate);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_pp_setup(const GraphObj &g, StateObj &st, bool crossing, const long long *gate) {
  if (g.topo->cap_bytes == 8) return launch_pp_setup_t<long long>(g, st, crossing, gate);
  return launch_pp_setup_t<int>(g, st, crossing, gate);
}

__global__ void ctrl_begin_kernel(Ctrl *c, double timeout_s, unsigned long long ceiling,
                                  int reset_counters) {
  pdl_wait();
  unsigned long long now = globaltimer();
  c->deadline_ns = now + (unsigned long long)(timeout_s * 1e9);
  c->last_ns = now;
  c->bar_count = 0;
  c->abort = 0;
  c->status = 0;
  c->overflow = 0;
  c->ceiling = ceiling;
  for (int i = 0; i < C_NCTR; ++i) c->live[i] = 0;
  c->flow = 0;
  c->cut = 0;
  c->x_live[0] = c->x_live[1] = c->x_snap[0] = c->x_snap[1] = 0;
  c->efill_d = LLONG_MAX;
  if (reset_counters) {
    for (int i = 0; i < PH_N; ++i) c->phase_ns[i] = 0;
    c->pushes = c->relabels = c->repairs = c->rounds = c->levels = c->waves = c->bytes = 0;
    c->async_items = 0;
    c->epochs = 0;
  }
}

// L2 residency for the heights: every BFS discovery test and every push
// scan reads h[] of random neighbours, so h (4n bytes; C2 17 MB, C4 96 MB)
// gets a persisting access-policy window on the engine stream, the rest of
// the traffic streams past it.
static cudaError_t set_l2_window(const Topology &T, const StateObj &st) {
  // per device (the persisting set-aside is a device-wide limit)
  static int enabled_d[64];
  static size_t max_window_d[64], max_persist_d[64], cur_persist_d[64], l2_d[64];
  static bool init_d = false;
  if (!init_d) {
    for (int i = 0; i < 64; ++i) enabled_d[i] = -1;
    init_d = true;
  }
  const int dv = T.device & 63;
  int &enabled = enabled_d[dv];
  size_t &max_window = max_window_d[dv], &max_persist = max_persist_d[dv],
         &cur_persist = cur_persist_d[dv], &l2 = l2_d[dv];
  // Default: on when the heights take at most a quarter of L2 (C1-C3, C2's
  // 17 MB: static 21.3 -> 20.6-21.2 ms, dynamic -1.5 %; neutral on R-MAT),
  // with the set-aside sized to the window.  Setting aside the device maximum
  // instead cost C2's static solve 23.6 -> 28.1 ms (15 -> 18 rounds).
  // $MFX_L2_WINDOW = 0 / 1 forces it off / on.
  const char *env = getenv("MFX_L2_WINDOW");  // (read per launch: A/B within a process)
  if (enabled < 0 && env != nullptr && atoi(env) == 0) return cudaSuccess;  // never set aside
  if (enabled < 0) {
    enabled = 1;
    int mw = 0, mp = 0, l2b = 0;
    if (cudaDeviceGetAttribute(&mw, cudaDevAttrMaxAccessPolicyWindowSize, T.device) ||
        cudaDeviceGetAttribute(&mp, cudaDevAttrMaxPersistingL2CacheSize, T.device) ||
        cudaDeviceGetAttribute(&l2b, cudaDevAttrL2CacheSize, T.device) || mw <= 0 || mp <= 0) {
      cudaGetLastError();
      enabled = 0;
    } else {
      max_window = (size_t)mw;
      max_persist = (size_t)mp;
      l2 = (size_t)l2b;
    }
  }
  const size_t hbytes = sizeof(int) * (size_t)T.n;
  const bool on = enabled > 0 && (env != nullptr ? atoi(env) != 0 : 4 * hbytes <= l2);
  cudaStreamAttrValue v = {};
  if (on) {
    size_t bytes = hbytes;
    // set aside only what the window needs (the whole carve-out starved
    // everything else: C2 static 23.6 -> 28.1 ms)
    size_t want = bytes < max_persist ? bytes : max_persist;
    if (want != cur_persist) {
      if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want)) return cudaGetLastError();
      cur_persist = want;
    }
    v.accessPolicyWindow.base_ptr = st.h;
    v.accessPolicyWindow.num_bytes = bytes < max_window ? bytes : max_window;
    v.accessPolicyWindow.hitRatio = 1.0f;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  } else if (cur_persist != 0) {  // (off: a zero-sized window clears a previous one,
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0)) return cudaGetLastError();
    cur_persist = 0;  //  and nothing stays set aside)
  }
  return cudaStreamSetAttribute(T.stream, cudaStreamAttributeAccessPolicyWindow, &v);
}

// ---------------------------------------------------------------------------
template <typename CapT>
static cudaError_t launch_solve_t(const GraphObj &g, StateObj &st, const SolveConfig &cfg,
                                  int *launches) {
  Topology &T = *g.topo;
  cudaError_t e = ensure_workspace(T);
  if (e != cudaSuccess) return e;
  Workspace &W = T.ws;
  SolveArgs<CapT> a;
  a.n = T.n;
  a.s = st.s;
  a.t = st.t;
  a.forbidden = cfg.forbidden;
  a.dyn_bases = cfg.dyn_bases;
  a.kc = cfg.kc;
  a.max_waves = cfg.max_waves;
  a.wave_mult = cfg.wave_mult;
  a.wave_add = cfg.wave_add;
  a.async = cfg.async && !cfg.topology;
  a.async_budget = cfg.async_budget;
  a.rdirty = W.rdirty;
  a.bfs_local = cfg.bfs_local;
  a.flags = cfg.flags;
  a.bfs_local_max = cfg.bfs_local_max;
  a.lq_cap = cfg.lq_cap < 1 ? 1 : cfg.lq_cap > kLQ ? kLQ : cfg.lq_cap;
  a.tail_items = cfg.tail_items;
  a.walk_max = cfg.walk_max;
  a.walk_depth = cfg.walk_depth;
  a.tail_local = cfg.tail_local;
  a.wave_time = cfg.wave_time;
  a.strand = cfg.strand > 0;
  a.early = cfg.early != 0;
  a.ring_sleep = cfg.ring_sleep;
  a.ramp = cfg.ramp;
  a.coop_kc = cfg.coop_kc > 0 ? (cfg.coop_kc < cfg.kc ? cfg.coop_kc : cfg.kc) : cfg.kc;
  a.tail_cap = cfg.tail_cap;
  a.bmark = W.bmark;
  a.topology = cfg.topology;
  a.what = cfg.what;
  a.rcap = W.rcap;
  a.off = T.off;
  a.adj = T.adj;
  a.rev = T.rev;
  a.vbin = W.vbin;
  a.cap0 = (const CapT *)g.cap0;
  a.pc = (const CapT *)g.pc;
  a.cf = (CapT *)st.cf;
  a.ex = st.ex;
  a.h = st.h;
  for (int b = 0; b < NBIN; ++b) {
    a.F0[b] = W.F[0][b];
    a.F1[b] = W.F[1][b];
    a.R[b] = W.R[b];
  }
  a.bases = W.bases;
  a.heavy = W.heavy;
  a.mark = W.mark;
  a.stamp = W.stamp;
  a.ctrl = st.ctrl;
  a.gate = cfg.gate;
  a.trace = W.trace;
  a.trace_cap = W.trace_cap;
  a.reg = cfg.pushpull ? W.reg : nullptr;
  if (cfg.pushpull) {
    a.async = 0;
    a.forbidden = -1;
  }
  // reached-set tracking (WHAT_SOLVE, ordinary rounds): the lists are
  // allocated by the first tracked launch; sparse = 1 when the list is valid
  // right now, 2 when only this launch's own relabels will make it so
  a.track = cfg.track && cfg.what == WHAT_SOLVE && !cfg.pushpull && !cfg.topology;
  if (a.track && st.tl[0] == nullptr) {
    if (cudaMalloc(&st.tl[0], sizeof(int) * (size_t)T.n) != cudaSuccess ||
        cudaMalloc(&st.tl[1], sizeof(int) * (size_t)T.n) != cudaSuccess) {
      cudaGetLastError();
      if (st.tl[0]) cudaFree(st.tl[0]);
      st.tl[0] = st.tl[1] = nullptr;
      a.track = 0;  // (no room: the relabels seed in full)
    }
  }
  a.tl[0] = st.tl[0];
  a.tl[1] = st.tl[1];
  a.sparse = a.track && cfg.sparse ? (st.tl_ok ? 1 : 2) : 0;
  if (!a.track && st.tl_ok) a.sparse = 1;  // (an untracked launch may still use the list: finalize)
  a.buv = W.d_uv;
  a.bk = cfg.dyn_bases && cfg.gate ? cfg.batch_k : 0;
  // valid again only when solve_status reads back a clean tracked finish
  st.tl_ok = false;

  if ((e = pdl_launch(ctrl_begin_kernel, 1, 1, T.stream, st.ctrl, cfg.timeout_s, cfg.ceiling,
                     cfg.reset_counters ? 1 : 0)))
    return e;

  const void *fn = cfg.pushpull ? (const void *)solve_kernel<CapT, true>
                                : (const void *)solve_kernel<CapT, false>;
  static int occ_cache[4] = {0, 0, 0, 0};
  int &occ = occ_cache[(sizeof(CapT) == 8) * 2 + (cfg.pushpull ? 1 : 0)];
  if (occ == 0) {
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kBlock, 0);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
  }
  int bps = occ;
  if (cfg.blocks_per_sm > 0 && cfg.blocks_per_sm < bps) bps = cfg.blocks_per_sm;
  int ctas = T.num_sms * bps;
  // small graphs: one CTA per SM -- a cheaper grid barrier (3.7 vs 4.5 us)
  // outweighs the halved warps when a whole level fits a few passes (C1:
  // 1.67 -> 1.50 ms, road 1024^2: 47 -> 42 ms; C2 / C3 lose, so they keep 2)
  int cap = cfg.max_ctas;
  if (cap == 0 && T.S <= (4 << 20)) cap = T.num_sms;
  // a batch whose last relabel reached few vertices (the sparse relabels of
  // C4) is a chain of thin relabel epochs and CTA-0 waves: half an SM's worth
  // of CTAs makes every grid barrier cheaper (C4 0.31 -> 0.29 ms/batch)
  if (cap == 0 && a.sparse == 1 && a.bk > 0) cap = T.num_sms / 2;
  if (cap > 0 && cap < ctas) ctas = cap;
  dim3 grid(ctas), block(kBlock);
  void *args[] = {(void *)&a};
  if ((e = set_l2_window(T, st)) != cudaSuccess) return e;
  e = cudaLaunchCooperativeKernel(fn, grid, block, args, 0, T.stream);
  if (launches) *launches += 2;
  count_launch(2);
  return e;
}

cudaError_t launch_solve(const GraphObj &g, StateObj &st, const SolveConfig &cfg, int *launches) {
  if (g.topo->cap_bytes == 8) return launch_solve_t<long long>(g, st, cfg, launches);
  return launch_solve_t<int>(g, st, cfg, launches);
}

}  // namespace MFX_SOLVE_NS
}  // namespace mfx
