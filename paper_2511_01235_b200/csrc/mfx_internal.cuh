// mfx_internal.cuh -- device data layout, control block and shared device
// helpers of the B200 max-flow engine.
//
// HBM layout (SoA, slot order identical to the reference build_bicsr: slots
// sorted by (u, v), graph.py:143-171):
//   topology (shared by graph copies, immutable):
//     off  int32[n+1]   row offsets
//     adj  int32[S]     head vertex of each slot
//     rev  int32[S]     paired reverse slot
//     orig uint8[S]     slot came from an input edge
//   capacities (private per graph copy, mutated by batches):
//     cap0 CapT[S]      capacity (0 on stubs)
//     pc   CapT[S]      pair capacity cap0[i] + cap0[rev i]; since
//                       cf[i] + cf[rev i] == pc[i] always (oracle.py:118),
//                       the BFS reads the reverse residual as pc[i] - cf[i]
//                       from u's own row instead of gathering cf[rev[i]].
//   state (per SolverState):
//     cf   CapT[S]      residual capacities
//     ex   int64[n]     signed excess
//     h    int32[n]     heights in [0, n]
// CapT is int32 when every pair sum fits (the default), else int64.
#pragma once
#include <cuda_runtime.h>

#include <utility>
#include <stdint.h>

namespace mfx {

// ---- programmatic dependent launch (the O(k) pre-phase chain) -------------
// Each small kernel of the dynamic pre-phase is launched with programmatic
// stream serialisation: it may be scheduled while its predecessor drains and
// waits on the device (griddepcontrol.wait, full completion and visibility of
// the prerequisite grid) before touching anything, so the chain pays one
// launch latency instead of one per kernel.  Every kernel launched through
// pdl_launch starts with pdl_wait().
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kern)(KArgs...), unsigned grid, unsigned block,
                              cudaStream_t st, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}


#ifndef MFX_BLOCK
#define MFX_BLOCK 256
#endif
constexpr int kBlock = MFX_BLOCK;  // threads per CTA (the solve kernel runs 2 CTAs/SM at 256)
constexpr int kWarps = kBlock / 32;
constexpr int NBIN = 4;  // 0: thread/vertex, 1: warp/vertex, 2: CTA/vertex, 3: huge
constexpr int kBin0Max = 8;
constexpr int kBin1Max = 1024;
constexpr int kBin2Max = 65536;
constexpr int kLQ = 2048;  // CTA-local BFS queue (per buffer)

__host__ __device__ inline int bin_of(int deg) {
  return deg <= kBin0Max ? 0 : deg <= kBin1Max ? 1 : deg <= kBin2Max ? 2 : 3;
}

// ---- control block (one per state, device memory) ------------------------
// live[] counters are appended to during a phase; the grid barrier's leader
// (last arriving CTA) moves them into snap[] before releasing, so every CTA
// reads identical, stable counts after the barrier.
enum CtrIdx {
  C_FNEXT = 0,   // [0..3]  next BFS frontier, per bin
  C_RNEXT = 4,   // [4..7]  next push wave (round list), per bin
  C_BASES = 8,   // bases list
  C_HEAVY = 9,   // heavy rows (finalize)
  C_ACTIVE = 10, // active vertices discovered by the global relabel
  C_HUGE = 11,   // huge rows (finalize)
  C_REACHED = 12, // vertices reached by the global relabel (bases + first discoveries)
  C_DEPTH = 13,  // largest BFS label set (max-combined, not summed)
  C_EHOLD = 14,  // vertices holding excess when the global relabel started
  C_STOP = 15,   // set by the barrier leader: this round's push-phase time budget is spent
  C_TALIVE = 16, // residual slots into the sink at the last global relabel (0: sink cut off)
  C_DBASES = 17, // deficient bases (all bases but the sink) of the last global relabel
  C_EFILL = 18,  // set by the barrier leader: the labelled excess covers every deficit (BFS may stop)
  C_NCTR = 19
};

enum Phase { PH_BFS = 0, PH_PUSH = 1, PH_REPAIR = 2, PH_FINAL = 3, PH_N = 4 };

struct Ctrl {
  unsigned int bar_count;
  unsigned int bar_gen;
  int abort;         // 1 = stop (status says why)
  int status;        // 0 ok, 3 solver error (ceiling), 6 timeout
  int live[C_NCTR];
  int snap[C_NCTR];
  unsigned long long deadline_ns;
  unsigned long long last_ns;
  unsigned long long phase_ns[PH_N];
  unsigned long long ceiling;  // pushes + relabels bound (operation_ceiling)
  // counters (flushed per round)
  unsigned long long pushes, relabels, repairs, rounds, levels, waves;
  unsigned long long bytes;
  long long flow, cut;
  long long active;   // active vertices found by the last global relabel
  long long reached;  // vertices reached by the last global relabel
  int overflow;
  int last_levels;  // BFS levels of the last global relabel
  long long trace_n;  // entries written to the diagnostics trace by the last launch
  // asynchronous push phase: per-bin queue heads / completed items, stop flag
  unsigned aq_head[NBIN];
  unsigned aq_done[NBIN];
  int aq_stop;
  int aq_pad;
  unsigned long long async_items;  // items processed by asynchronous push phases
  // deficits filled since the last global relabel (a push took a head's
  // excess from < 0 to >= 0); with the sink cut off and every deficient
  // base filled, no base is left to absorb excess: the push phase ends
  unsigned long long fills;
  // demand-covered early exit of a solve's global relabel: [0] = total
  // deficit of the deficient bases, [1] = excess of the holders labelled so
  // far; live = appended this epoch, snap = the leader's running totals
  long long x_live[2], x_snap[2];
  long long efill_d;  // total deficit at the last early exit it allowed (must shrink)
  // reached-set lists (StateObj::tl): which of the two holds the last
  // global relabel's reached set (tracked solves flip it per relabel)
  int tl_cur;
  int tl_ok;  // the last relabel of the last launch kept its list (StateObj::tl_ok)
  unsigned long long epochs;       // grid barriers spent in global relabels
  // push waves run by CTA 0 alone (thin waves): state for the other CTAs
  int tail_base[NBIN];
  int tail_waves;
  unsigned tail_stamp;
  // push-phase time budget (wave_time): start of the last global relabel,
  // and the deadline of the current push phase (0: none)
  unsigned long long bfs_t0, wave_deadline;
  // trace mode only: vertices expanded per BFS epoch (sum, max over CTAs), by epoch parity
  unsigned dbg_sum[2], dbg_max[2];
};

// ---- small device helpers -------------------------------------------------
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// L2-coherent loads for arrays mutated during a phase (cf, ex, h): L1 is not
// coherent and a persistent kernel keeps L1 lines across phases.
__device__ __forceinline__ int ldcg(const int *p) { return __ldcg(p); }
__device__ __forceinline__ long long ldcg(const long long *p) { return __ldcg(p); }

__device__ __forceinline__ int atomic_add(int *p, int v) { return atomicAdd(p, v); }
__device__ __forceinline__ long long atomic_add(long long *p, long long v) {
  return (long long)atomicAdd((unsigned long long *)p, (unsigned long long)v);
}
__device__ __forceinline__ int atomic_exch(int *p, int v) { return atomicExch(p, v); }
__device__ __forceinline__ long long atomic_exch(long long *p, long long v) {
  return (long long)atomicExch((unsigned long long *)p, (unsigned long long)v);
}

__device__ __forceinline__ int atomic_cas(int *p, int cmp, int v) { return atomicCAS(p, cmp, v); }
__device__ __forceinline__ long long atomic_cas(long long *p, long long cmp, long long v) {
  return (long long)atomicCAS((unsigned long long *)p, (unsigned long long)cmp,
                              (unsigned long long)v);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Warp-aggregated append of `v` to list `buf` at base + atomicAdd(counter):
// one atomic per warp per call.  Safe under divergence (uses __activemask).
__device__ __forceinline__ void warp_append(bool pred, int v, int *counter, int *buf, int base,
                                            int cap, int *overflow) {
  unsigned act = __activemask();
  unsigned b = __ballot_sync(act, pred);
  if (b == 0) return;
  int lane = threadIdx.x & 31;
  int leader = __ffs(b) - 1;
  int pos0 = 0;
  if (lane == leader) pos0 = atomicAdd(counter, __popc(b));
  pos0 = __shfl_sync(act, pos0, leader);
  if (pred) {
    int p = base + pos0 + __popc(b & lanemask_lt());
    if (p < cap) buf[p] = v;
    else *overflow = 1;
  }
}

// Per-bin warp-aggregated append (the bin is a function of the vertex degree).
__device__ __forceinline__ void warp_append_binned(bool pred, int v, int bin, int *counters,
                                                   int *const *bufs, const int *bases, int cap,
                                                   int *overflow) {
  unsigned act = __activemask();
  if (__ballot_sync(act, pred) == 0) return;
#pragma unroll
  for (int b = 0; b < NBIN; ++b) {
    bool p = pred && bin == b;
    unsigned m = __ballot_sync(act, p);
    if (m == 0) continue;
    int lane = threadIdx.x & 31;
    int leader = __ffs(m) - 1;
    int pos0 = 0;
    if (lane == leader) pos0 = atomicAdd(counters + b, __popc(m));
    pos0 = __shfl_sync(act, pos0, leader);
    if (p) {
      int pos = bases[b] + pos0 + __popc(m & lanemask_lt());
      if (pos < cap) bufs[b][pos] = v;
      else *overflow = 1;
    }
  }
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

}  // namespace mfx
