// part.cu -- vertex-range partitioned solver (config C5, R-MAT 26,
// ~2.1 B Bi-CSR slots: more than the int32 slot layout of one device holds).
//
// Part r owns the vertices [lo_r, hi_r) and their Bi-CSR rows (the slot range
// [off[lo_r], off[hi_r]) of the global layout, in the reference's slot order,
// graph.py:143-171), with local int32 slot indices and global head ids.  For
// every slot i, rev[i] is the index of the reverse slot inside the part that
// owns the head, found by a binary search of that part's row over peer
// memory.  Every array a peer touches (off, adj, cap0, pc, cf, ex, h, mark,
// frontiers, round lists, counters) is reached through a PeerTab of device
// pointers: same-device pointers when several parts share one GPU (tests),
// NVLink P2P pointers when the parts of one process sit on several GPUs, or
// CUDA IPC mappings when each GPU has its own process (torch.distributed).
//
// The round loop is bulk-synchronous and driven by the host, one phase per
// call (mfx_part_phase), with a cross-part barrier + tiny all-reduce between
// phases ("one exchange step per phase"):
//   global relabel  level-synchronous BFS; a discovery of a remote vertex is
//                   an atomicCAS on the owner's h plus an append to the
//                   owner's next frontier (and its round list when active)
//   push wave       bounded push/relabel (kernels.py:19-67) over the round
//                   list; on a cut slot cf[i] -= d stays local, the reverse
//                   residual and the head's excess are remote atomics
//   repair          steep residual slots (kernels.py:70-93)
//   finalize        local flow / cut partials, summed by the host
// All remote-visible updates are system-scope atomics, so concurrent parts
// (other GPUs over NVLink, other processes) combine exactly; phases are
// separated by stream synchronisation + the host barrier.
#include <limits.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/mfx.h"
#include "engine.h"

namespace mfx {

constexpr int kMaxParts = 8;
constexpr int kPartHeavy = 2048;  // rows above this are expanded / pushed by a whole CTA
constexpr int kPartHuge = 65536;  // finalize: rows above this are walked by the whole grid
constexpr int kPartBlock = 256;

// per-part device counters (int32, written by every part)
enum PartCtr {
  PC_FN0 = 0,      // next frontier fill, bin 0 / 1
  PC_FN1 = 1,
  PC_RT0 = 2,      // round-list tails, bin 0 / 1
  PC_RT1 = 3,
  PC_ACTIVE = 4,   // active vertices discovered by the global relabel
  PC_REACHED = 5,  // vertices reached (bases + discoveries)
  PC_OVF = 6,      // round-list overflow
  PC_BASES = 7,
  PC_BAD = 8,      // link: slots without a reverse
  PC_OB0 = 16,     // outbox fill toward part q: PC_OB0 + q (reset by q once applied)
  PC_N = 24
};
// per-part 64-bit statistics (local writes only)
enum PartStat { PS_PUSH = 0, PS_RELABEL, PS_REPAIR, PS_BYTES, PS_FLOW, PS_CUT, PS_ACTIVE, PS_N = 8 };
// batch error block (int64), LLONG_MAX = none
enum PartErr { PE_NEG = 0, PE_UNKNOWN, PE_DUPSLOT, PE_DUPK, PE_OVER, PE_N = 8 };

struct PeerTab {
  int P;
  int n;  // global vertex count
  int lo[kMaxParts + 1];
  const int *off[kMaxParts];
  const int *adj[kMaxParts];
  const int *cap0[kMaxParts];
  int *pc[kMaxParts];
  int *cf[kMaxParts];
  long long *ex[kMaxParts];
  int *h[kMaxParts];
  unsigned *mark[kMaxParts];
  int *F[kMaxParts][2][2];  // [part][buffer][bin]
  int *R[kMaxParts][2];     // [part][bin]
  int *ctr[kMaxParts];
  int4 *out[kMaxParts];  // cut-slot push outboxes, obox_cap(nl) entries per destination
  int obox;              // 1: cut-slot pushes go through the outboxes
  int ostride;           // entries per destination: obox_cap(largest part), same on every part
  // own part only: vertices relabeled in the current round (the repair scope);
  // rl_cnt[1] counts the hub rows (> kPartHuge slots) among them, listed in rl_hub
  int *rl_list, *rl_flag, *rl_cnt, *rl_hub;
};

// device buffers of one part; the order here is the IPC export order
enum PartBuf {
  B_OFF = 0, B_ADJ, B_CAP0, B_PC, B_CF, B_EX, B_H, B_MARK, B_F00, B_F01, B_F10, B_F11, B_R0, B_R1,
  B_CTR, B_OUT, B_NBUF
};

// Outbox entries per destination part: pushes along cut slots in one push
// phase are buffered as (reverse slot, local vertex, amount) in the pushing
// part's own memory and applied by the owner after the phase barrier (one
// coalesced peer read per entry instead of two remote atomics and a remote
// activation per push).  A full outbox falls back to the direct remote update.
__host__ __device__ __forceinline__ int obox_cap(int nl) {
  return nl < 1024 ? 1024 : (nl > (1 << 22) ? (1 << 22) : nl);
}

struct PartObj {
  int device = 0;
  int P = 1, rank = 0;
  long long n = 0;
  int lo = 0, hi = 0, nl = 0;  // owned vertex range, local row count
  int S = 0;                   // local slots
  long long slot_base = 0;     // global index of local slot 0
  int m_original = 0;          // local original slots
  int s = -1, t = -1;
  int rcap = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 0;
  void *buf[B_NBUF] = {};
  size_t bytes[B_NBUF] = {};
  // local-only
  int *rev = nullptr;
  uint8_t *orig = nullptr;
  int *bases = nullptr;
  int *src = nullptr;           // local row of every slot (slot-parallel finalize)
  int *heavy = nullptr;         // rows longer than kPartHeavy
  int nheavy = 0;
  int *huge = nullptr;          // rows longer than kPartHuge
  int nhuge = 0;
  int *rl_list = nullptr, *rl_flag = nullptr, *rl_cnt = nullptr, *rl_hub = nullptr;
  // hub push scratch (capacity nhuge)
  int *hub_list = nullptr, *hub_cnt = nullptr;
  unsigned long long *hub_best = nullptr;
  long long *hub_taken = nullptr, *hub_snap = nullptr;
  unsigned long long *stat = nullptr;
  long long *err = nullptr;
  int *slot_first = nullptr;
  int *bslot = nullptr;        // batch scratch
  long long *bbuf = nullptr;   // batch staging: u, v, cap, global index
  long long bcap = 0;
  int bk = 0;
  PeerTab tab;
  bool opened[kMaxParts][B_NBUF] = {};  // IPC mappings to close
  bool inbox_pending = false;  // a push phase ran since the last swap
  unsigned push_stamp = 0;
  ~PartObj();
};

PartObj::~PartObj() {
  cudaSetDevice(device);
  for (int p = 0; p < kMaxParts; ++p)
    for (int b = 0; b < B_NBUF; ++b)
      if (opened[p][b]) {
        void *ptr = nullptr;
        switch (b) {
          case B_OFF: ptr = (void *)tab.off[p]; break;
          case B_ADJ: ptr = (void *)tab.adj[p]; break;
          case B_CAP0: ptr = (void *)tab.cap0[p]; break;
          case B_PC: ptr = tab.pc[p]; break;
          case B_CF: ptr = tab.cf[p]; break;
          case B_EX: ptr = tab.ex[p]; break;
          case B_H: ptr = tab.h[p]; break;
          case B_MARK: ptr = tab.mark[p]; break;
          case B_F00: ptr = tab.F[p][0][0]; break;
          case B_F01: ptr = tab.F[p][0][1]; break;
          case B_F10: ptr = tab.F[p][1][0]; break;
          case B_F11: ptr = tab.F[p][1][1]; break;
          case B_R0: ptr = tab.R[p][0]; break;
          case B_R1: ptr = tab.R[p][1]; break;
          case B_CTR: ptr = tab.ctr[p]; break;
          case B_OUT: ptr = tab.out[p]; break;
        }
        if (ptr) cudaIpcCloseMemHandle(ptr);
      }
  for (int b = 0; b < B_NBUF; ++b)
    if (buf[b]) cudaFree(buf[b]);
  for (void *p : {(void *)rev, (void *)orig, (void *)bases, (void *)src, (void *)heavy, (void *)huge, (void *)hub_list, (void *)hub_cnt,
                  (void *)hub_best, (void *)hub_taken, (void *)hub_snap, (void *)stat, (void *)err,
                  (void *)slot_first, (void *)bslot, (void *)bbuf, (void *)rl_list,
                  (void *)rl_flag, (void *)rl_cnt, (void *)rl_hub})
    if (p) cudaFree(p);
  if (stream) cudaStreamDestroy(stream);
}

static void tab_set_self(PartObj &o, int p) {
  PeerTab &T = o.tab;
  T.off[p] = (const int *)o.buf[B_OFF];
  T.adj[p] = (const int *)o.buf[B_ADJ];
  T.cap0[p] = (const int *)o.buf[B_CAP0];
  T.pc[p] = (int *)o.buf[B_PC];
  T.cf[p] = (int *)o.buf[B_CF];
  T.ex[p] = (long long *)o.buf[B_EX];
  T.h[p] = (int *)o.buf[B_H];
  T.mark[p] = (unsigned *)o.buf[B_MARK];
  T.F[p][0][0] = (int *)o.buf[B_F00];
  T.F[p][0][1] = (int *)o.buf[B_F01];
  T.F[p][1][0] = (int *)o.buf[B_F10];
  T.F[p][1][1] = (int *)o.buf[B_F11];
  T.R[p][0] = (int *)o.buf[B_R0];
  T.R[p][1] = (int *)o.buf[B_R1];
  T.ctr[p] = (int *)o.buf[B_CTR];
  T.out[p] = (int4 *)o.buf[B_OUT];
}

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
#define PGS_LOOP(i, cnt)                                                          \
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (cnt); \
       i += (long long)gridDim.x * blockDim.x)

__device__ __forceinline__ int owner_of(const PeerTab &T, int v) {
  int p = 0;
#pragma unroll
  for (int q = 1; q < kMaxParts; ++q)
    if (q < T.P && v >= T.lo[q]) p = q;
  return p;
}
__device__ __forceinline__ int vol_ld(const int *p) { return *(const volatile int *)p; }
__device__ __forceinline__ long long vol_ld(const long long *p) {
  return *(const volatile long long *)p;
}
__device__ __forceinline__ int sys_add(int *p, int v) { return atomicAdd_system(p, v); }
__device__ __forceinline__ long long sys_add(long long *p, long long v) {
  return (long long)atomicAdd_system((unsigned long long *)p, (unsigned long long)v);
}
__device__ __forceinline__ int heavy_of(const PeerTab &T, int p, int vl) {
  return (T.off[p][vl + 1] - T.off[p][vl]) > kPartHeavy ? 1 : 0;
}

// ---------------------------------------------------------------------------
// build helpers
// ---------------------------------------------------------------------------
__global__ void part_flag_kernel(long long m, const long long *us, const long long *vs, long long lo,
                                 long long hi, char *flag) {
  PGS_LOOP(i, m) {
    long long u = us[i], v = vs[i];
    flag[i] = (u >= lo && u < hi) || (v >= lo && v < hi);
  }
}

__global__ void part_slice_kernel(int nl, int lo, const int *goff, int *off) {
  PGS_LOOP(i, (long long)nl + 1) off[i] = goff[lo + i] - goff[lo];
}

__global__ void part_copy_slots_kernel(long long S, long long base, const int *gadj,
                                       const long long *gcap, const uint8_t *gorig, int *adj,
                                       int *cap0, uint8_t *orig, unsigned long long *bad) {
  PGS_LOOP(i, S) {
    adj[i] = gadj[base + i];
    long long c = gcap[base + i];
    if (c >= (1ll << 30)) atomicAdd(bad, 1ull);
    cap0[i] = (int)c;
    orig[i] = gorig[base + i];
  }
}

// rev[i]: slot of (adj[i], u) inside the part owning adj[i] (graph.py:171)
__global__ void part_rev_kernel(PeerTab T, int me, int nl, long long S, const int *off,
                                const int *adj, int *rev, int *ctr) {
  PGS_LOOP(i, S) {
    int a = 0, b = nl;  // row u: last row with off[u] <= i
    while (b - a > 1) {
      int mid = (a + b) >> 1;
      if (off[mid] <= (int)i) a = mid;
      else b = mid;
    }
    int ug = T.lo[me] + a;
    int x = adj[i];
    int p = owner_of(T, x);
    int xl = x - T.lo[p];
    const int *po = T.off[p], *pa = T.adj[p];
    int lo = po[xl], hi = po[xl + 1];
    while (lo < hi) {
      int mid = lo + ((hi - lo) >> 1);
      if (pa[mid] < ug) lo = mid + 1;
      else hi = mid;
    }
    if (lo < po[xl + 1] && pa[lo] == ug) rev[i] = lo;
    else {
      rev[i] = -1;
      atomicAdd(ctr + PC_BAD, 1);
    }
  }
}

__global__ void part_pc_kernel(PeerTab T, int me, long long S, const int *rev, int *ctr) {
  const int *adj = T.adj[me], *cap0 = T.cap0[me];
  int *pc = T.pc[me];
  PGS_LOOP(i, S) {
    int p = owner_of(T, adj[i]);
    long long s2 = (long long)cap0[i] + (long long)T.cap0[p][rev[i]];
    if (s2 >= (1ll << 31)) atomicAdd(ctr + PC_BAD, 1);
    pc[i] = (int)s2;
  }
}

// ---------------------------------------------------------------------------
// state
// ---------------------------------------------------------------------------
__global__ void part_init_kernel(PeerTab T, int me, int nl, long long S) {
  PGS_LOOP(i, S) T.cf[me][i] = T.cap0[me][i];
  PGS_LOOP(v, nl) {
    T.ex[me][v] = 0;
    T.h[me][v] = 0;
    T.mark[me][v] = 0;
  }
}

// saturate_source (state.py:42-59) on the part owning s: one CTA per chunk
__global__ void part_saturate_kernel(PeerTab T, int me, int sl, const int *rev,
                                     const long long *gate) {
  if (gate && (gate[PE_NEG] != LLONG_MAX || gate[PE_UNKNOWN] != LLONG_MAX ||
               gate[PE_DUPK] != LLONG_MAX || gate[PE_OVER] != LLONG_MAX))
    return;
  __shared__ long long part[kPartBlock / 32];
  const int lo = T.off[me][sl], hi = T.off[me][sl + 1];
  long long sum = 0;
  for (long long i = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < hi;
       i += (long long)gridDim.x * blockDim.x) {
    int d = T.cf[me][i];
    if (d > 0) {
      T.cf[me][i] = 0;
      int v = T.adj[me][i];
      int p = owner_of(T, v);
      sys_add(T.cf[p] + rev[i], d);
      sys_add(T.ex[p] + (v - T.lo[p]), (long long)d);
      sum += d;
    }
  }
  sum = warp_sum(sum);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int w = 0; w < kPartBlock / 32; ++w) tot += part[w];
    if (tot) sys_add(T.ex[me] + sl, -tot);
  }
}

// ---------------------------------------------------------------------------
// global relabel: level-synchronous BFS (kernels.py:168-215)
// ---------------------------------------------------------------------------
__global__ void part_bfs_init_kernel(PeerTab T, int me, int nl, int s, int t, int dyn,
                                     int forbidden, int *bases) {
  const int n = T.n, lo = T.lo[me];
  int *ctr = T.ctr[me];
  PGS_LOOP(v, nl) {
    int g = lo + (int)v;
    bool base = g == t || (dyn && g != s && vol_ld(T.ex[me] + v) < 0);
    if (g == forbidden) base = false;
    T.h[me][v] = base ? 0 : n;
    if (base) {
      int b = heavy_of(T, me, (int)v);
      T.F[me][0][b][atomicAdd(ctr + PC_FN0 + b, 1)] = (int)v;
      bases[atomicAdd(ctr + PC_BASES, 1)] = (int)v;
      atomicAdd(ctr + PC_REACHED, 1);
    }
  }
}

// Discovery through slot i of a frontier row (warp-synchronous: every lane of
// the warp calls, `valid` lanes hold a slot).  The owner's height is claimed
// by a system-scope CAS per discovery; the owner-side counters (next-frontier
// append, reached, active count, round-list append) take ONE system-scope
// atomic per (owner, degree class) group of the warp instead of one per
// discovery: over NVLink every remote atomic is a round trip to the owner's
// L2, and all of a level's discoveries hit the same few counter words.
__device__ __forceinline__ void part_discover_w(const PeerTab &T, int me, bool valid, int i, int L,
                                                int cur, int s, int t, int forbidden, int rcap) {
  const unsigned FULLM = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  int p = 0, vl = 0, b = 0;
  bool disc = false, act = false;
  if (valid) {
    const int v = T.adj[me][i];
    if (v != forbidden && T.pc[me][i] - vol_ld(T.cf[me] + i) > 0) {  // reverse residual cf[rev i]
      p = owner_of(T, v);
      vl = v - T.lo[p];
      int *hp = T.h[p] + vl;
      if (vol_ld(hp) == T.n && atomicCAS_system(hp, T.n, L + 1) == T.n) {
        disc = true;
        b = heavy_of(T, p, vl);
        act = v != s && v != t && vol_ld(T.ex[p] + vl) > 0;
      }
    }
  }
  if (!__any_sync(FULLM, disc)) return;
  const unsigned lt = lanemask_lt();
  {  // next frontier of the owner, per (owner, class)
    const unsigned g = __match_any_sync(FULLM, disc ? (unsigned)(p * 2 + b) : ~0u);
    const int ld = __ffs(g) - 1;
    int pos = 0;
    if (disc && lane == ld) pos = atomicAdd_system(T.ctr[p] + PC_FN0 + b, __popc(g));
    pos = __shfl_sync(FULLM, pos, ld) + __popc(g & lt);
    if (disc) T.F[p][cur ^ 1][b][pos] = vl;
  }
  {  // reached, per owner
    const unsigned g = __match_any_sync(FULLM, disc ? (unsigned)p : ~0u);
    if (disc && lane == __ffs(g) - 1) atomicAdd_system(T.ctr[p] + PC_REACHED, __popc(g));
  }
  if (!__any_sync(FULLM, act)) return;
  {  // active: the owner's round list, per (owner, class), and its count, per owner
    const unsigned g = __match_any_sync(FULLM, act ? (unsigned)(p * 2 + b) : ~0u);
    const int ld = __ffs(g) - 1;
    int q = 0;
    if (act && lane == ld) q = atomicAdd_system(T.ctr[p] + PC_RT0 + b, __popc(g));
    q = __shfl_sync(FULLM, q, ld) + __popc(g & lt);
    if (act) {
      if (q < rcap) T.R[p][b][q] = vl;
      else atomicExch_system(T.ctr[p] + PC_OVF, 1);
    }
    const unsigned g2 = __match_any_sync(FULLM, act ? (unsigned)p : ~0u);
    if (act && lane == __ffs(g2) - 1) atomicAdd_system(T.ctr[p] + PC_ACTIVE, __popc(g2));
  }
}

__global__ void part_bfs_expand_kernel(PeerTab T, int me, int L, int cur, int cnt0, int cnt1,
                                       int s, int t, int forbidden, int rcap, const int *huge,
                                       int nhuge) {
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int gwarps = (gridDim.x * blockDim.x) >> 5;
  const int *F0 = T.F[me][cur][0], *F1 = T.F[me][cur][1];
  for (int j = gwarp; j < cnt0; j += gwarps) {  // warp per light row
    int u = F0[j];
    int lo = T.off[me][u], hi = T.off[me][u + 1];
    for (int i0 = lo; i0 < hi; i0 += 32)
      part_discover_w(T, me, i0 + lane < hi, i0 + lane, L, cur, s, t, forbidden, rcap);
  }
  for (int j = blockIdx.x; j < cnt1; j += gridDim.x) {  // CTA per heavy row
    int u = F1[j];
    int lo = T.off[me][u], hi = T.off[me][u + 1];
    if (hi - lo > kPartHuge) continue;  // hubs: below
    for (int i0 = lo + (threadIdx.x & ~31); i0 < hi; i0 += blockDim.x) {  // warp-uniform trips
      const int i = i0 + (threadIdx.x & 31);
      part_discover_w(T, me, i < hi, i, L, cur, s, t, forbidden, rcap);
    }
  }
  // hubs of this level (the frontier of a level-synchronous BFS is {h == L}):
  // the whole grid per row
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gthreads = gridDim.x * blockDim.x;
  for (int j = 0; j < nhuge; ++j) {
    const int u = huge[j];
    if (vol_ld(T.h[me] + u) != L) continue;
    const int lo = T.off[me][u], hi = T.off[me][u + 1];
    for (int i0 = lo + (gtid & ~31); i0 < hi; i0 += gthreads) {
      const int i = i0 + (gtid & 31);
      part_discover_w(T, me, i < hi, i, L, cur, s, t, forbidden, rcap);
    }
  }
}

// Bottom-up step of the same level (direction-optimising BFS): every
// unreached own vertex v scans its own row for a residual slot v -> u into
// the frontier {h == L} and stops at the first one.  On R-MAT's wide middle
// levels most unreached vertices hit within their first 32 slots, instead of
// the frontier rows being scanned whole.  The heights are the same BFS
// distances as the top-down step's; v is written by its own warp only.
__global__ void part_bfs_bottomup_kernel(PeerTab T, int me, int nl, int L, int cur, int s, int t,
                                         int forbidden, int rcap) {
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int gwarps = (gridDim.x * blockDim.x) >> 5;
  const int n = T.n, lo_g = T.lo[me];
  int *ctr = T.ctr[me];
  for (int v0 = gwarp * 32; v0 < nl; v0 += gwarps * 32) {
    const int vme = v0 + lane;
    const bool open = vme < nl && vol_ld(T.h[me] + vme) == n && lo_g + vme != forbidden;
    unsigned todo = __ballot_sync(0xffffffffu, open);
    while (todo) {  // the warp scans each open vertex's row in turn
      const int k = __ffs(todo) - 1;
      todo &= todo - 1;
      const int v = v0 + k;
      const int lo = T.off[me][v], hi = T.off[me][v + 1];
      bool found = false;
      for (int i0 = lo; i0 < hi && !found; i0 += 32) {
        const int i = i0 + lane;
        bool hit = false;
        if (i < hi && vol_ld(T.cf[me] + i) > 0) {
          const int u = T.adj[me][i];
          const int p = owner_of(T, u);
          hit = vol_ld(T.h[p] + (u - T.lo[p])) == L;
        }
        found = __any_sync(0xffffffffu, hit);
      }
      if (found && lane == 0) {
        T.h[me][v] = L + 1;
        const int b = (hi - lo) > kPartHeavy ? 1 : 0;
        T.F[me][cur ^ 1][b][atomicAdd(ctr + PC_FN0 + b, 1)] = v;
        atomicAdd(ctr + PC_REACHED, 1);
        const int g = lo_g + v;
        if (g != s && g != t && vol_ld(T.ex[me] + v) > 0) {
          atomicAdd(ctr + PC_ACTIVE, 1);
          const int q = atomicAdd(ctr + PC_RT0 + b, 1);
          if (q < rcap) T.R[me][b][q] = v;
          else atomicExch(ctr + PC_OVF, 1);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// push wave (kernels.py:19-67): cooperative per row (warp or CTA), pushing
// along every admissible slot at the minimum residual height in slot order
// ---------------------------------------------------------------------------
// u (own, local) was relabeled below n: its row is in this round's repair
// scope.  A residual slot becomes steep (h(u) > h(v) + 1) only when its tail
// is raised -- heads only rise within a round, and a push v -> u is decided on
// h(v) > h(u) -- so the relabeled rows hold every slot the repair can find.
__device__ __forceinline__ void part_relabeled(const PeerTab &T, int me, int u) {
  if (atomicExch(T.rl_flag + u, 1) != 0) return;
  if (T.off[me][u + 1] - T.off[me][u] > kPartHuge) T.rl_hub[atomicAdd(T.rl_cnt + 1, 1)] = u;
  else T.rl_list[atomicAdd(T.rl_cnt, 1)] = u;
}

__device__ __forceinline__ void part_activate(const PeerTab &T, int v, unsigned stamp, int s, int t,
                                              int rcap) {
  if (v == s || v == t) return;
  int p = owner_of(T, v);
  int vl = v - T.lo[p];
  if (atomicMax_system(T.mark[p] + vl, stamp) >= stamp) return;  // already in the next wave
  int b = heavy_of(T, p, vl);
  int q = atomicAdd_system(T.ctr[p] + PC_RT0 + b, 1);
  if (q < rcap) T.R[p][b][q] = vl;
  else atomicExch_system(T.ctr[p] + PC_OVF, 1);
}

// Warp-synchronous part_activate (every lane calls; `pred` lanes activate v):
// the per-vertex stamp stays one atomic each, the owner's round-list append
// is one system-scope atomic per (owner, class) group of the warp.
__device__ __forceinline__ void part_activate_w(const PeerTab &T, bool pred, int v, unsigned stamp,
                                                int s, int t, int rcap) {
  const unsigned FULLM = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  int p = 0, vl = 0, b = 0;
  if (pred && (v == s || v == t)) pred = false;
  if (pred) {
    p = owner_of(T, v);
    vl = v - T.lo[p];
    pred = atomicMax_system(T.mark[p] + vl, stamp) < stamp;  // not yet in the next wave
    if (pred) b = heavy_of(T, p, vl);
  }
  if (!__any_sync(FULLM, pred)) return;
  const unsigned g = __match_any_sync(FULLM, pred ? (unsigned)(p * 2 + b) : ~0u);
  const int ld = __ffs(g) - 1;
  int q = 0;
  if (pred && lane == ld) q = atomicAdd_system(T.ctr[p] + PC_RT0 + b, __popc(g));
  q = __shfl_sync(FULLM, q, ld) + __popc(g & lanemask_lt());
  if (pred) {
    if (q < rcap) T.R[p][b][q] = vl;
    else atomicExch_system(T.ctr[p] + PC_OVF, 1);
  }
}

template <int G>
__device__ void part_push_row(const PeerTab &T, int me, int u, int kc, unsigned stamp, int s, int t,
                              int rcap, const int *rev, unsigned long long *loc,
                              long long *s_red) {
  const int n = T.n;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int tid = G == 32 ? lane : threadIdx.x;
  const int ug = T.lo[me] + u;
  const int lo = T.off[me][u], hi = T.off[me][u + 1];
  int *cf = T.cf[me];
  const int *adj = T.adj[me];
  // one read, broadcast: every thread of the group must take the same loop
  // decisions (the CTA variant synchronises inside the loop)
  int hu;
  long long eu;
  if (G == 32) {
    hu = __shfl_sync(0xffffffffu, lane == 0 ? vol_ld(T.h[me] + u) : 0, 0);
    eu = __shfl_sync(0xffffffffu, lane == 0 ? vol_ld(T.ex[me] + u) : 0ll, 0);
  } else {
    __syncthreads();
    if (threadIdx.x == 0) {
      s_red[0] = vol_ld(T.h[me] + u);
      s_red[1] = vol_ld(T.ex[me] + u);
    }
    __syncthreads();
    hu = (int)s_red[0];
    eu = s_red[1];
    __syncthreads();
  }
  for (int cnt = 0; cnt < kc; ++cnt) {
    if (eu <= 0 || hu >= n) break;
    unsigned long long best = ~0ull;  // (height, slot) of the first minimum (kernels.py:40-48)
    for (int i = lo + tid; i < hi; i += G) {
      if (vol_ld(cf + i) > 0) {
        int v = adj[i];
        int p = owner_of(T, v);
        unsigned hv = (unsigned)vol_ld(T.h[p] + (v - T.lo[p]));
        unsigned long long key = ((unsigned long long)hv << 32) | (unsigned)(i - lo);
        best = key < best ? key : best;
      }
    }
    best = warp_min_u64(best);
    if (G > 32) {
      __syncthreads();
      if (lane == 0) s_red[wib] = (long long)best;
      __syncthreads();
      best = ~0ull;
      for (int w = 0; w < G / 32; ++w)
        best = (unsigned long long)s_red[w] < best ? (unsigned long long)s_red[w] : best;
      __syncthreads();
    }
    if (tid == 0) loc[PS_BYTES] += 20 + 12ull * (hi - lo);
    if (best == ~0ull) {  // no residual out-slot
      hu = n;
      if (tid == 0) {
        T.h[me][u] = n;
        loc[PS_RELABEL]++;
      }
      break;
    }
    int bh = (int)(best >> 32);
    if (hu <= bh) {  // relabel from the scan snapshot
      hu = bh + 1 > n ? n : bh + 1;
      if (tid == 0) {
        T.h[me][u] = hu;
        loc[PS_RELABEL]++;
        if (hu < n) part_relabeled(T, me, u);
      }
      continue;
    }
    int first = lo + (int)(best & 0xFFFFFFFFu);
    long long carry = 0;
    for (int i0 = first - ((first - lo) % G); i0 < hi && carry < eu; i0 += G) {
      int i = i0 + tid;
      long long c = 0;
      int v = 0, p = 0;
      if (i < hi && i >= first) {
        c = vol_ld(cf + i);
        if (c > 0) {
          v = adj[i];
          p = owner_of(T, v);
          if (vol_ld(T.h[p] + (v - T.lo[p])) != bh) c = 0;
        }
      }
      long long incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        long long w = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += w;
      }
      long long tot;
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
        __syncthreads();
      } else {
        tot = __shfl_sync(0xffffffffu, incl, 31);
      }
      long long room = eu - carry - (incl - c);
      long long amt = room <= 0 ? 0 : (room < c ? room : c);
      long long old = 1;
      if (amt > 0) {
        atomicAdd(cf + i, (int)-amt);
        int q = INT_MAX;
        if (p != me && T.obox) q = atomicAdd(T.ctr[me] + PC_OB0 + p, 1);
        if (q < T.ostride) {  // applied (and v activated) by p after the barrier
          T.out[me][(size_t)p * T.ostride + q] = make_int4(rev[i], v - T.lo[p], (int)amt, 0);
          loc[PS_BYTES] += 16;
        } else {
          sys_add(T.cf[p] + rev[i], (int)amt);
          old = sys_add(T.ex[p] + (v - T.lo[p]), amt);
          loc[PS_BYTES] += 28;
        }
        loc[PS_PUSH]++;
      }
      part_activate_w(T, amt > 0 && old <= 0, v, stamp, s, t, rcap);  // (warp-uniform loop)
      carry += tot;
    }
    long long moved = carry < eu ? carry : eu;
    if (tid == 0 && moved > 0) sys_add(T.ex[me] + u, -moved);
    eu -= moved;
  }
  if (G > 32) __syncthreads();
  if (tid == 0 && hu < n && vol_ld(T.ex[me] + u) > 0) part_activate(T, ug, stamp, s, t, rcap);
}

// The owner's half of the buffered cut-slot pushes (after the push phase's
// barrier): every peer's outbox toward `me`, read over P2P in entry order.
__global__ void part_inbox_kernel(PeerTab T, int me, unsigned stamp, int s, int t, int rcap,
                                  unsigned long long *stat) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  unsigned long long bytes = 0;
  for (int p = 0; p < T.P; ++p) {
    if (p == me) continue;
    const int cnt = min(vol_ld(T.ctr[p] + PC_OB0 + me), T.ostride);
    const int4 *box = T.out[p] + (size_t)me * T.ostride;
    for (int j0 = gw * 32; j0 < cnt; j0 += nw * 32) {  // (warp-uniform trip count)
      const int j = j0 + lane;
      long long old = 1;
      int v = 0;
      if (j < cnt) {
        const int4 e = __ldcv(box + j);
        v = e.y;
        sys_add(T.cf[me] + e.x, e.z);
        old = sys_add(T.ex[me] + v, (long long)e.z);
        bytes += 16 + 16;
      }
      part_activate_w(T, j < cnt && old <= 0, T.lo[me] + v, stamp, s, t, rcap);
    }
  }
  bytes = warp_sum(bytes);
  if (lane == 0 && bytes) atomicAdd(stat + PS_BYTES, bytes);
}
__global__ void part_inbox_reset_kernel(PeerTab T, int me) {
  const int p = threadIdx.x;
  if (p < T.P && p != me) atomicExch_system(T.ctr[p] + PC_OB0 + me, 0);
}

__global__ void part_push_kernel(PeerTab T, int me, int b0, int e0, int b1, int e1, int kc,
                                 unsigned stamp, int s, int t, int rcap, const int *rev,
                                 unsigned long long *stat, int *hub_list, int *hub_cnt,
                                 unsigned long long *hub_best, long long *hub_taken) {
  __shared__ long long s_red[kPartBlock / 32 + 2];
  unsigned long long loc[PS_N] = {};
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int gwarps = (gridDim.x * blockDim.x) >> 5;
  for (int j = b0 + gwarp; j < e0; j += gwarps)
    part_push_row<32>(T, me, T.R[me][0][j], kc, stamp, s, t, rcap, rev, loc, s_red);
  for (int j = b1 + blockIdx.x; j < e1; j += gridDim.x) {
    const int u = T.R[me][1][j];
    if (T.off[me][u + 1] - T.off[me][u] > kPartHuge) {  // hub: whole grid, next kernels
      if (threadIdx.x == 0) {
        const int q = atomicAdd(hub_cnt, 1);
        hub_list[q] = u;
        hub_best[q] = ~0ull;
        hub_taken[q] = 0;
      }
      continue;
    }
    part_push_row<kPartBlock>(T, me, u, kc, stamp, s, t, rcap, rev, loc, s_red);
  }
  for (int k = 0; k < 4; ++k) {
    unsigned long long x = warp_sum(loc[k]);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd(stat + k, x);
  }
}

// One push-or-relabel step for hub rows (> kPartHuge slots) with the whole
// grid: (1) first-minimum (height, slot) over the residual slots by a 64-bit
// atomicMin, with u's height and excess snapshotted once; (2) relabel from
// the scan, or push along every slot at the minimum height, each slot
// claiming its share of the snapshot excess through an atomic ticket.
__global__ void part_hub_scan_kernel(PeerTab T, int me, const int *hub_list, const int *hub_cnt,
                                     unsigned long long *hub_best, long long *hub_snap) {
  const int nh = *hub_cnt;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gthreads = gridDim.x * blockDim.x;
  for (int j = 0; j < nh; ++j) {
    const int u = hub_list[j];
    const int lo = T.off[me][u], hi = T.off[me][u + 1];
    if (gtid == 0) {
      hub_snap[2 * j] = vol_ld(T.h[me] + u);
      hub_snap[2 * j + 1] = vol_ld(T.ex[me] + u);
    }
    unsigned long long best = ~0ull;
    for (int i = lo + gtid; i < hi; i += gthreads) {
      if (vol_ld(T.cf[me] + i) > 0) {
        const int v = T.adj[me][i];
        const int p = owner_of(T, v);
        const unsigned hv = (unsigned)vol_ld(T.h[p] + (v - T.lo[p]));
        const unsigned long long key = ((unsigned long long)hv << 32) | (unsigned)(i - lo);
        best = key < best ? key : best;
      }
    }
    best = warp_min_u64(best);
    if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(hub_best + j, best);
  }
}

__global__ void part_hub_push_kernel(PeerTab T, int me, const int *hub_list, const int *hub_cnt,
                                     const unsigned long long *hub_best, const long long *hub_snap,
                                     long long *hub_taken, unsigned stamp, int s, int t, int rcap,
                                     const int *rev, unsigned long long *stat) {
  const int n = T.n, nh = *hub_cnt;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gthreads = gridDim.x * blockDim.x;
  unsigned long long pushes = 0;
  for (int j = 0; j < nh; ++j) {
    const int u = hub_list[j];
    const int hu = (int)hub_snap[2 * j];
    const long long eu = hub_snap[2 * j + 1];
    const unsigned long long best = hub_best[j];
    if (eu <= 0 || hu >= n) continue;
    if (best == ~0ull || hu <= (int)(best >> 32)) {  // relabel (kernels.py:49-53, 62-66)
      if (gtid == 0) {
        const int nh2 = best == ~0ull ? n : ((int)(best >> 32) + 1 > n ? n : (int)(best >> 32) + 1);
        T.h[me][u] = nh2;
        atomicAdd(stat + PS_RELABEL, 1ull);
        if (nh2 < n) part_relabeled(T, me, u);
        if (nh2 < n) part_activate(T, T.lo[me] + u, stamp, s, t, rcap);
      }
      continue;
    }
    const int bh = (int)(best >> 32);
    const int lo = T.off[me][u], hi = T.off[me][u + 1];
    for (int i = lo + gtid; i < hi; i += gthreads) {
      const long long c = vol_ld(T.cf[me] + i);
      if (c <= 0) continue;
      const int v = T.adj[me][i];
      const int p = owner_of(T, v);
      if (vol_ld(T.h[p] + (v - T.lo[p])) != bh) continue;
      const long long before = atomicAdd((unsigned long long *)(hub_taken + j),
                                         (unsigned long long)c);
      long long amt = eu - before;
      amt = amt < 0 ? 0 : (amt < c ? amt : c);
      if (amt <= 0) continue;
      atomicAdd(T.cf[me] + i, (int)-amt);
      sys_add(T.cf[p] + rev[i], (int)amt);
      const long long old = sys_add(T.ex[p] + (v - T.lo[p]), amt);
      sys_add(T.ex[me] + u, -amt);
      ++pushes;
      if (old <= 0) part_activate(T, v, stamp, s, t, rcap);
    }
  }
  pushes = warp_sum(pushes);
  if ((threadIdx.x & 31) == 0 && pushes) atomicAdd(stat + PS_PUSH, pushes);
}

// still overflowing after its step: the hub joins the next wave
__global__ void part_hub_tail_kernel(PeerTab T, int me, const int *hub_list, const int *hub_cnt,
                                     unsigned stamp, int s, int t, int rcap) {
  const int nh = *hub_cnt;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nh; j += gridDim.x * blockDim.x) {
    const int u = hub_list[j];
    if (vol_ld(T.h[me] + u) < T.n && vol_ld(T.ex[me] + u) > 0)
      part_activate(T, T.lo[me] + u, stamp, s, t, rcap);
  }
}

// repair (kernels.py:70-93).  The reference repairs every vertex that ran in
// the round; only relabeled rows can hold a steep residual slot (see
// part_relabeled), so the scope is the round's relabel list -- on R-MAT 26
// the round lists repeat hub rows every wave.  Clears the list's flags.
__global__ void part_repair_kernel(PeerTab T, int me, const int *rev, unsigned long long *stat) {
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int gwarps = (gridDim.x * blockDim.x) >> 5;
  const int nr = *T.rl_cnt;
  unsigned long long reps = 0;
  auto slot = [&](int u, int hu, int i) {
    if (vol_ld(T.cf[me] + i) <= 0) return;
    int v = T.adj[me][i];
    int p = owner_of(T, v);
    int vl = v - T.lo[p];
    if (hu > vol_ld(T.h[p] + vl) + 1) {
      int amt = atomicExch(T.cf[me] + i, 0);
      if (amt > 0) {
        sys_add(T.cf[p] + rev[i], amt);
        sys_add(T.ex[me] + u, -(long long)amt);
        sys_add(T.ex[p] + vl, (long long)amt);
        ++reps;
      }
    }
  };
  for (int j = gwarp; j < nr; j += gwarps) {  // warp per light row
    int u = T.rl_list[j];
    int lo = T.off[me][u], hi = T.off[me][u + 1];
    if (hi - lo > kPartHeavy) continue;
    int hu = vol_ld(T.h[me] + u);
    for (int i = lo + lane; i < hi; i += 32) slot(u, hu, i);
    if (lane == 0) T.rl_flag[u] = 0;
  }
  for (int j = blockIdx.x; j < nr; j += gridDim.x) {  // CTA per heavy row
    int u = T.rl_list[j];
    int lo = T.off[me][u], hi = T.off[me][u + 1];
    if (hi - lo <= kPartHeavy) continue;
    int hu = vol_ld(T.h[me] + u);
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) slot(u, hu, i);
    if (threadIdx.x == 0) T.rl_flag[u] = 0;
  }
  // hub rows (R-MAT 26: millions of slots): the whole grid per row
  const int nh = T.rl_cnt[1];
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gthreads = gridDim.x * blockDim.x;
  for (int j = 0; j < nh; ++j) {
    int u = T.rl_hub[j];
    int lo = T.off[me][u], hi = T.off[me][u + 1];
    int hu = vol_ld(T.h[me] + u);
    for (int i = lo + gtid; i < hi; i += gthreads) slot(u, hu, i);
    if (gtid == 0) T.rl_flag[u] = 0;
  }
  reps = warp_sum(reps);
  if (lane == 0 && reps) atomicAdd(stat + PS_REPAIR, reps);
}

// flow over the local bases (dynamic.py:141-143) and the local part of the cut
// (solver.py:178-184): original slots from A = {h == n} into B
__global__ void part_final_kernel(PeerTab T, int me, long long S, int nb, const int *bases,
                                  const uint8_t *orig, const int *src,
                                  unsigned long long *stat) {
  const int n = T.n, lane = threadIdx.x & 31;
  long long f = 0, c = 0;
  PGS_LOOP(j, nb) f += vol_ld(T.ex[me] + bases[j]);
  PGS_LOOP(i, S) {  // slot-parallel: original slots from A = {h == n} into B
    if (!orig[i] || vol_ld(T.h[me] + src[i]) != n) continue;
    const int v = T.adj[me][i];
    const int p = owner_of(T, v);
    if (vol_ld(T.h[p] + (v - T.lo[p])) != n) c += T.cap0[me][i];
  }
  f = warp_sum(f);
  c = warp_sum(c);
  if (lane == 0) {
    if (f) atomicAdd(stat + PS_FLOW, (unsigned long long)f);
    if (c) atomicAdd(stat + PS_CUT, (unsigned long long)c);
  }
}

__global__ void part_src_kernel(const int *off, int nl, int *src) {
  const int lane = threadIdx.x & 31;
  for (int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < nl;
       u += (gridDim.x * blockDim.x) >> 5)
    for (int i = off[u] + lane; i < off[u + 1]; i += 32) src[i] = u;
}

__global__ void part_heavy_list_kernel(const int *off, int nl, int *list, int *cnt, int *huge,
                                       int *hcnt) {
  PGS_LOOP(u, nl) {
    int d = off[u + 1] - off[u];
    if (d > kPartHeavy) list[atomicAdd(cnt, 1)] = (int)u;
    if (d > kPartHuge) huge[atomicAdd(hcnt, 1)] = (int)u;
  }
}

// topology mode (solver.py:167-175): the round's worklist is every owned
// vertex but s and t, binned like the relabel's appends
__global__ void part_topo_seed_kernel(PeerTab T, int me, int nl, int s, int t, int rcap) {
  int *ctr = T.ctr[me];
  PGS_LOOP(v, nl) {
    const int g = T.lo[me] + (int)v;
    if (g == s || g == t) continue;
    const int b = heavy_of(T, me, (int)v);
    const int q = atomicAdd(ctr + PC_RT0 + b, 1);
    if (q < rcap) T.R[me][b][q] = (int)v;
    else atomicExch(ctr + PC_OVF, 1);
  }
}

__global__ void part_active_kernel(PeerTab T, int me, int nl, int s, int t,
                                   unsigned long long *stat) {
  unsigned long long a = 0;
  PGS_LOOP(v, nl) {
    int g = T.lo[me] + (int)v;
    if (g != s && g != t && T.ex[me][v] > 0 && T.h[me][v] < T.n) ++a;
  }
  a = warp_sum(a);
  if ((threadIdx.x & 31) == 0 && a) atomicAdd(stat + PS_ACTIVE, a);
}

// ---------------------------------------------------------------------------
// dynamic batch (dynamic.py:63-116): the host routes update j to the part
// owning us[j]; validation first (no mutation), apply only if every part's
// share of the batch is valid
// ---------------------------------------------------------------------------
__global__ void part_batch_resolve_kernel(PeerTab T, int me, long long k, const long long *bu,
                                          const long long *bv, const long long *bc,
                                          const long long *bj, const uint8_t *orig,
                                          const int *rev, int *slot, int *first, long long *err) {
  PGS_LOOP(j, k) {
    long long c = bc[j], gj = bj[j];
    if (c < 0) atomicMin(err + PE_NEG, gj);
    int ul = (int)(bu[j] - T.lo[me]);
    long long v = bv[j];
    int i = -1;
    if (v >= 0 && v < T.n) {
      int lo = T.off[me][ul], hi = T.off[me][ul + 1];
      while (lo < hi) {
        int mid = lo + ((hi - lo) >> 1);
        if (T.adj[me][mid] < (int)v) lo = mid + 1;
        else hi = mid;
      }
      if (lo < T.off[me][ul + 1] && T.adj[me][lo] == (int)v) i = lo;
    }
    slot[j] = i;
    if (i < 0 || !orig[i]) {
      atomicMin(err + PE_UNKNOWN, gj);
    } else {
      atomicMin(first + i, (int)gj);
      if (c >= 0) {
        int p = owner_of(T, (int)v);
        if (c >= (1ll << 30) || c + (long long)T.cap0[p][rev[i]] >= (1ll << 31))
          atomicMin(err + PE_OVER, gj);
      }
    }
  }
}

__global__ void part_batch_dup_kernel(long long k, long long slot_base, const int *slot,
                                      const int *first, const long long *bj, long long *err) {
  PGS_LOOP(j, k) {
    int i = slot[j];
    if (i >= 0 && first[i] != (int)bj[j]) atomicMin(err + PE_DUPSLOT, slot_base + i);
  }
}

__global__ void part_batch_dupidx_kernel(long long k, long long slot_base, const int *slot,
                                         const int *first, const long long *bj, long long *err) {
  long long ds = err[PE_DUPSLOT];
  if (ds == LLONG_MAX) return;
  PGS_LOOP(j, k) {
    int i = slot[j];
    if (i >= 0 && slot_base + i == ds && first[i] != (int)bj[j]) atomicMin(err + PE_DUPK, bj[j]);
  }
}

__global__ void part_batch_apply_kernel(PeerTab T, int me, long long k, const long long *bc,
                                        const int *slot, int *first, int apply) {
  PGS_LOOP(j, k) {
    int i = slot[j];
    if (i < 0) continue;
    first[i] = kFirstNone;
    if (apply) {
      int nc = (int)bc[j];
      T.cf[me][i] += nc - T.cap0[me][i];
      ((int *)T.cap0[me])[i] = nc;
    }
  }
}

// after every part applied: pair sums of touched pairs and the negative
// residual repair (flow reversal, dynamic.py:105-109) with its excess move
__global__ void part_batch_fix_kernel(PeerTab T, int me, long long k, const long long *bu,
                                      const int *slot, const int *rev) {
  PGS_LOOP(j, k) {
    int i = slot[j];
    int v = T.adj[me][i];
    int p = owner_of(T, v);
    int r = rev[i];
    int pcv = T.cap0[me][i] + T.cap0[p][r];
    T.pc[me][i] = pcv;
    T.pc[p][r] = pcv;
    int c = T.cf[me][i];
    if (c < 0) {
      T.cf[me][i] = 0;
      sys_add(T.cf[p] + r, c);
      sys_add(T.ex[me] + (int)(bu[j] - T.lo[me]), -(long long)c);
      sys_add(T.ex[p] + (v - T.lo[p]), (long long)c);
    }
  }
}

// ---------------------------------------------------------------------------
// device batch sampler for the largest graphs (gen.py fast_batch semantics:
// exponential-race keys E/w over the original slots, w = bias on s-out / t-in
// edges; decrements on positive capacities, new in [0, old); increments on
// the rest, new in [old+1, 2 old + 10]).  Candidates below a threshold are
// compacted and only they are sorted.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long smix(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ int row_of(const int *off, int nl, int i) {
  int a = 0, b = nl;
  while (b - a > 1) {
    int mid = (a + b) >> 1;
    if (off[mid] <= i) a = mid;
    else b = mid;
  }
  return a;
}

__global__ void part_sample_kernel(PeerTab T, int me, int nl, long long S, const uint8_t *orig,
                                   const uint8_t *taken, int s, int t, double bias,
                                   unsigned long long seed, int dec, double tau, int cap,
                                   unsigned long long *cand, int *cnt) {
  const int *off = T.off[me], *adj = T.adj[me], *cap0 = T.cap0[me];
  PGS_LOOP(i, S) {
    if (!orig[i] || taken[i] || (dec && cap0[i] <= 0)) continue;
    unsigned long long hsh = smix(seed ^ smix((unsigned long long)(T.lo[me]) * 0x100000001ull + i));
    double uu = ((double)(hsh >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    double w = 1.0;
    if (adj[i] == t) w = bias;
    else if (s >= T.lo[me] && s < T.lo[me + 1] && off[s - T.lo[me]] <= i && i < off[s - T.lo[me] + 1])
      w = bias;
    double key = -log(uu) / w;
    if (key < tau) {
      int q = atomicAdd(cnt, 1);
      if (q < cap) {
        float kf = (float)key;
        cand[q] = ((unsigned long long)__float_as_uint(kf) << 32) | (unsigned)i;
      }
    }
  }
}

__global__ void part_sample_emit_kernel(PeerTab T, int me, int nl, const int *slots, int k,
                                        int dec, unsigned long long seed, uint8_t *taken,
                                        long long *ou, long long *ov, long long *oc) {
  const int *off = T.off[me], *adj = T.adj[me], *cap0 = T.cap0[me];
  PGS_LOOP(j, k) {
    int i = slots[j];
    taken[i] = 1;
    long long old = cap0[i];
    unsigned long long hsh = smix(seed ^ 0xD1B54A32D192ED03ull ^ smix((unsigned long long)i + 1));
    ou[j] = T.lo[me] + row_of(off, nl, i);
    ov[j] = adj[i];
    oc[j] = dec ? (long long)(hsh % (unsigned long long)old)
                : old + 1 + (long long)(hsh % (unsigned long long)(old + 10));
  }
}

__global__ void part_untake_kernel(const int *slots, int k, uint8_t *taken) {
  PGS_LOOP(j, k) taken[slots[j]] = 0;
}

__global__ void part_weight_kernel(PeerTab T, int me, long long S, const uint8_t *orig, int s, int t,
                                   double bias, unsigned long long *acc) {
  const int *off = T.off[me], *adj = T.adj[me];
  unsigned long long a = 0;
  PGS_LOOP(i, S) {
    if (!orig[i]) continue;
    bool hub = adj[i] == t || (s >= T.lo[me] && s < T.lo[me + 1] && off[s - T.lo[me]] <= i &&
                               i < off[s - T.lo[me] + 1]);
    a += hub ? (unsigned long long)bias : 1ull;
  }
  a = warp_sum(a);
  if ((threadIdx.x & 31) == 0 && a) atomicAdd(acc, a);
}

static inline int pgrid(long long work, int sms) {
  long long g = (work + kPartBlock - 1) / kPartBlock;
  long long cap = (long long)sms * 8;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace mfx

// ===========================================================================
// C-ABI
// ===========================================================================
using namespace mfx;

struct mfx_part {
  PartObj o;
};

namespace mfx {
static int part_fail(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}
}  // namespace mfx

#define PCK(x)                                                                         \
  do {                                                                                 \
    cudaError_t _e = (x);                                                              \
    if (_e != cudaSuccess)                                                             \
      return part_fail(MFX_CUDA_ERROR, "CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), \
                       __FILE__, __LINE__, cudaGetErrorString(_e));                    \
  } while (0)

static int part_build(PartObj &o, long long m, const int64_t *d_us, const int64_t *d_vs,
                      const int64_t *d_caps) {
  cudaStream_t st = o.stream;
  // edges incident to the owned range
  char *flag = nullptr;
  int64_t *sel = nullptr;
  int *nsel = nullptr;
  size_t M = (size_t)(m > 0 ? m : 1);
  PCK(cudaMalloc(&flag, M));
  PCK(cudaMalloc(&sel, 3 * M * sizeof(int64_t)));
  PCK(cudaMalloc(&nsel, sizeof(int) * 4));
  long long msel = 0;
  if (m > 0) {
    part_flag_kernel<<<pgrid(m, o.num_sms), kPartBlock, 0, st>>>(m, (const long long *)d_us,
                                                               (const long long *)d_vs, o.lo, o.hi,
                                                               flag);
    size_t tb = 0;
    PCK(cub::DeviceSelect::Flagged(nullptr, tb, d_us, flag, sel, nsel, (int64_t)m, st));
    void *tmp = nullptr;
    PCK(cudaMalloc(&tmp, tb));
    const int64_t *src[3] = {d_us, d_vs, d_caps};
    int cnt[3];
    for (int k = 0; k < 3; ++k) {
      size_t t2 = tb;
      PCK(cub::DeviceSelect::Flagged(tmp, t2, src[k], flag, sel + k * M, nsel + k, (int64_t)m, st));
    }
    PCK(cudaMemcpyAsync(cnt, nsel, sizeof(cnt), cudaMemcpyDeviceToHost, st));
    PCK(cudaStreamSynchronize(st));
    cudaFree(tmp);
    msel = cnt[0];
    count_launch(4);
  }
  cudaFree(flag);
  cudaFree(nsel);
  // Bi-CSR of the selected edges over all n vertices: the owned rows are
  // exactly the owned rows of the global layout (every edge touching them)
  Topology topo;
  topo.device = o.device;
  topo.stream = st;
  topo.num_sms = o.num_sms;
  int64_t err[2];
  int64_t *gcap = nullptr;
  cudaError_t e = build_bicsr_device(o.n, msel, sel, sel + M, sel + 2 * M, topo, &gcap, err, nullptr);
  cudaFree(sel);
  topo.stream = nullptr;  // owned by the part
  PCK(e);
  if (err[0]) {
    if (gcap) cudaFree(gcap);
    if (err[0] == 5)
      return part_fail(MFX_VALUE_ERROR, "partition exceeds the int32 slot layout of one device");
    return part_fail(MFX_GRAPH_ERROR, "invalid edge list (kind %lld at selected edge %lld)",
                     (long long)err[0], (long long)err[1]);
  }
  int glo = 0, ghi = 0;
  PCK(cudaMemcpy(&glo, topo.off + o.lo, sizeof(int), cudaMemcpyDeviceToHost));
  PCK(cudaMemcpy(&ghi, topo.off + o.hi, sizeof(int), cudaMemcpyDeviceToHost));
  o.S = ghi - glo;
  size_t SS = (size_t)(o.S > 0 ? o.S : 1), NL = (size_t)(o.nl > 0 ? o.nl : 1);
  o.rcap = (int)std::min<long long>(4ll * NL + 4096, INT_MAX);
  size_t sizes[B_NBUF] = {sizeof(int) * (NL + 1), sizeof(int) * SS, sizeof(int) * SS,
                          sizeof(int) * SS, sizeof(int) * SS, sizeof(long long) * NL,
                          sizeof(int) * NL, sizeof(unsigned) * NL, sizeof(int) * NL,
                          sizeof(int) * NL, sizeof(int) * NL, sizeof(int) * NL,
                          sizeof(int) * (size_t)o.rcap, sizeof(int) * (size_t)o.rcap,
                          sizeof(int) * PC_N,
                          sizeof(int4) * (size_t)o.tab.ostride * (o.P > 1 ? o.P : 1)};
  for (int b = 0; b < B_NBUF; ++b) {
    o.bytes[b] = sizes[b];
    PCK(cudaMalloc(&o.buf[b], sizes[b]));
  }
  PCK(cudaMemsetAsync(o.buf[B_CTR], 0, sizeof(int) * PC_N, st));
  PCK(cudaMalloc(&o.rev, sizeof(int) * SS));
  PCK(cudaMalloc(&o.orig, SS));
  PCK(cudaMalloc(&o.bases, sizeof(int) * NL));
  PCK(cudaMalloc(&o.heavy, sizeof(int) * NL));
  PCK(cudaMalloc(&o.src, sizeof(int) * SS));
  PCK(cudaMalloc(&o.huge, sizeof(int) * NL));
  PCK(cudaMalloc(&o.rl_list, sizeof(int) * NL));
  PCK(cudaMalloc(&o.rl_flag, sizeof(int) * NL));
  PCK(cudaMalloc(&o.rl_cnt, 2 * sizeof(int)));
  PCK(cudaMalloc(&o.rl_hub, sizeof(int) * NL));
  PCK(cudaMemsetAsync(o.rl_flag, 0, sizeof(int) * NL, st));
  PCK(cudaMemsetAsync(o.rl_cnt, 0, 2 * sizeof(int), st));
  PCK(cudaMalloc(&o.stat, sizeof(unsigned long long) * PS_N));
  PCK(cudaMalloc(&o.err, sizeof(long long) * PE_N));
  PCK(cudaMalloc(&o.slot_first, sizeof(int) * SS));
  PCK(cudaMemsetAsync(o.slot_first, 0x7f, sizeof(int) * SS, st));
  unsigned long long *bad = nullptr;
  PCK(cudaMalloc(&bad, sizeof(unsigned long long)));
  PCK(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), st));
  part_slice_kernel<<<pgrid(o.nl + 1, o.num_sms), kPartBlock, 0, st>>>(o.nl, o.lo, topo.off,
                                                                      (int *)o.buf[B_OFF]);
  if (o.S > 0)
    part_copy_slots_kernel<<<pgrid(o.S, o.num_sms), kPartBlock, 0, st>>>(
        o.S, glo, topo.adj, (const long long *)gcap, topo.orig, (int *)o.buf[B_ADJ],
        (int *)o.buf[B_CAP0], o.orig, bad);
  unsigned long long hb = 0;
  PCK(cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, st));
  PCK(cudaStreamSynchronize(st));
  count_launch(2);
  cudaFree(bad);
  cudaFree(gcap);
  if (hb)
    return part_fail(MFX_VALUE_ERROR,
                     "the partitioned engine stores int32 residuals: capacities must stay below 2^30");
  // local original slots
  {
    std::vector<uint8_t> h((size_t)o.S);
    if (o.S > 0) PCK(cudaMemcpy(h.data(), o.orig, (size_t)o.S, cudaMemcpyDeviceToHost));
    long long mo = 0;
    for (uint8_t x : h) mo += x != 0;
    o.m_original = (int)mo;
  }
  return MFX_OK;
}

extern "C" {

int mfx_part_create(int64_t n, int nparts, int rank, const int64_t *bounds, int64_t m,
                    const int64_t *d_us, const int64_t *d_vs, const int64_t *d_caps,
                    int64_t source, int64_t sink, int device, mfx_part **out) {
  *out = nullptr;
  if (n <= 0) return part_fail(MFX_GRAPH_ERROR, "vertex count must be positive, got %lld", (long long)n);
  if (n >= INT_MAX) return part_fail(MFX_VALUE_ERROR, "vertex ids must fit int32");
  if (nparts < 1 || nparts > kMaxParts)
    return part_fail(MFX_VALUE_ERROR, "nparts must be in [1, %d], got %d", kMaxParts, nparts);
  if (rank < 0 || rank >= nparts) return part_fail(MFX_VALUE_ERROR, "rank %d out of range", rank);
  if (bounds[0] != 0 || bounds[nparts] != n)
    return part_fail(MFX_VALUE_ERROR, "partition bounds must start at 0 and end at n");
  for (int p = 0; p < nparts; ++p)
    if (bounds[p + 1] <= bounds[p])
      return part_fail(MFX_VALUE_ERROR, "partition bounds must be strictly increasing");
  if (source < 0 || source >= n || sink < 0 || sink >= n || source == sink)
    return part_fail(MFX_VALUE_ERROR, "invalid source/sink (%lld, %lld)", (long long)source,
                     (long long)sink);
  int count = 0;
  PCK(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count)
    return part_fail(MFX_VALUE_ERROR, "device %d out of range [0, %d)", device, count);
  PCK(cudaSetDevice(device));
  mfx_part *P = new mfx_part();
  PartObj &o = P->o;
  o.device = device;
  o.P = nparts;
  o.rank = rank;
  o.n = n;
  o.lo = (int)bounds[rank];
  o.hi = (int)bounds[rank + 1];
  o.nl = o.hi - o.lo;
  o.s = (int)source;
  o.t = (int)sink;
  memset(&o.tab, 0, sizeof(o.tab));
  o.tab.P = nparts;
  o.tab.n = (int)n;
  {
    // MFX_PART_OUTBOX: 0 = every cut-slot push updates the peer directly;
    // k >= 2 = outboxes of k entries (tests: overflow into the direct path)
    const char *ob = getenv("MFX_PART_OUTBOX");
    const int obv = ob ? atoi(ob) : 1;
    o.tab.obox = obv != 0;
    long long big = 0;
    for (int p = 0; p < nparts; ++p) big = std::max<long long>(big, bounds[p + 1] - bounds[p]);
    o.tab.ostride = obv >= 2 ? obv : obox_cap((int)big);
  }
  for (int p = 0; p <= nparts; ++p) o.tab.lo[p] = (int)bounds[p];
  for (int p = nparts + 1; p <= kMaxParts; ++p) o.tab.lo[p] = (int)n;
  cudaError_t e = cudaStreamCreateWithFlags(&o.stream, cudaStreamNonBlocking);
  if (!e) e = cudaDeviceGetAttribute(&o.num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e) {
    delete P;
    PCK(e);
  }
  int rc = part_build(o, m, d_us, d_vs, d_caps);
  if (rc) {
    delete P;
    return rc;
  }
  {  // rows long enough for whole-grid treatment in repair / finalize
    int *cnt = nullptr;
    cudaError_t e2 = cudaMalloc(&cnt, 2 * sizeof(int));
    if (!e2) e2 = cudaMemsetAsync(cnt, 0, 2 * sizeof(int), o.stream);
    if (!e2 && o.nl > 0) {
      part_heavy_list_kernel<<<pgrid(o.nl, o.num_sms), kPartBlock, 0, o.stream>>>(
          (const int *)o.buf[B_OFF], o.nl, o.heavy, cnt, o.huge, cnt + 1);
      part_src_kernel<<<o.num_sms * 8, kPartBlock, 0, o.stream>>>((const int *)o.buf[B_OFF], o.nl,
                                                                   o.src);
      count_launch();
    }
    int hc[2] = {0, 0};
    if (!e2) e2 = cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, o.stream);
    if (!e2) e2 = cudaStreamSynchronize(o.stream);
    o.nheavy = hc[0];
    o.nhuge = hc[1];
    if (cnt) cudaFree(cnt);
    const size_t H = (size_t)(o.nhuge > 0 ? o.nhuge : 1);
    if (!e2) e2 = cudaMalloc(&o.hub_list, sizeof(int) * H);
    if (!e2) e2 = cudaMalloc(&o.hub_cnt, sizeof(int));
    if (!e2) e2 = cudaMalloc(&o.hub_best, sizeof(unsigned long long) * H);
    if (!e2) e2 = cudaMalloc(&o.hub_taken, sizeof(long long) * H);
    if (!e2) e2 = cudaMalloc(&o.hub_snap, sizeof(long long) * 2 * H);
    count_launch();
    if (e2) {
      delete P;
      PCK(e2);
    }
  }
  tab_set_self(o, rank);
  o.tab.rl_list = o.rl_list;
  o.tab.rl_flag = o.rl_flag;
  o.tab.rl_cnt = o.rl_cnt;
  o.tab.rl_hub = o.rl_hub;
  *out = P;
  return MFX_OK;
}

int mfx_part_create_host(int64_t n, int nparts, int rank, const int64_t *bounds, int64_t m,
                         const int64_t *us, const int64_t *vs, const int64_t *caps,
                         int64_t source, int64_t sink, int device, mfx_part **out) {
  *out = nullptr;
  PCK(cudaSetDevice(device));
  size_t M = (size_t)(m > 0 ? m : 1);
  int64_t *d = nullptr;
  PCK(cudaMalloc(&d, 3 * M * sizeof(int64_t)));
  if (m > 0) {
    PCK(cudaMemcpy(d, us, m * sizeof(int64_t), cudaMemcpyHostToDevice));
    PCK(cudaMemcpy(d + M, vs, m * sizeof(int64_t), cudaMemcpyHostToDevice));
    PCK(cudaMemcpy(d + 2 * M, caps, m * sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  int rc = mfx_part_create(n, nparts, rank, bounds, m, d, d + M, d + 2 * M, source, sink, device, out);
  cudaFree(d);
  return rc;
}

void mfx_part_free(mfx_part *p) { delete p; }

int mfx_part_info(const mfx_part *p, int64_t *info) {
  const PartObj &o = p->o;
  info[0] = o.lo;
  info[1] = o.hi;
  info[2] = o.S;
  info[3] = o.m_original;
  info[4] = o.rcap;
  info[5] = o.device;
  info[6] = o.P;
  info[7] = o.rank;
  return MFX_OK;
}

int mfx_part_export(const mfx_part *p, void *blob, int64_t cap, int64_t *len) {
  const PartObj &o = p->o;
  int64_t need = (int64_t)(B_NBUF * sizeof(cudaIpcMemHandle_t));
  *len = need;
  if (cap < need) return part_fail(MFX_VALUE_ERROR, "export blob needs %lld bytes", (long long)need);
  PCK(cudaSetDevice(o.device));
  for (int b = 0; b < B_NBUF; ++b) {
    cudaIpcMemHandle_t h;
    PCK(cudaIpcGetMemHandle(&h, o.buf[b]));
    memcpy((char *)blob + b * sizeof(h), &h, sizeof(h));
  }
  return MFX_OK;
}

int mfx_part_attach(mfx_part *p, int peer, const void *blob, int64_t len) {
  PartObj &o = p->o;
  if (peer < 0 || peer >= o.P || peer == o.rank)
    return part_fail(MFX_VALUE_ERROR, "peer %d invalid for rank %d of %d", peer, o.rank, o.P);
  if (len < (int64_t)(B_NBUF * sizeof(cudaIpcMemHandle_t)))
    return part_fail(MFX_VALUE_ERROR, "short peer blob");
  PCK(cudaSetDevice(o.device));
  void *ptr[B_NBUF];
  for (int b = 0; b < B_NBUF; ++b) {
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char *)blob + b * sizeof(h), sizeof(h));
    PCK(cudaIpcOpenMemHandle(&ptr[b], h, cudaIpcMemLazyEnablePeerAccess));
    o.opened[peer][b] = true;
  }
  PeerTab &T = o.tab;
  T.off[peer] = (const int *)ptr[B_OFF];
  T.adj[peer] = (const int *)ptr[B_ADJ];
  T.cap0[peer] = (const int *)ptr[B_CAP0];
  T.pc[peer] = (int *)ptr[B_PC];
  T.cf[peer] = (int *)ptr[B_CF];
  T.ex[peer] = (long long *)ptr[B_EX];
  T.h[peer] = (int *)ptr[B_H];
  T.mark[peer] = (unsigned *)ptr[B_MARK];
  T.F[peer][0][0] = (int *)ptr[B_F00];
  T.F[peer][0][1] = (int *)ptr[B_F01];
  T.F[peer][1][0] = (int *)ptr[B_F10];
  T.F[peer][1][1] = (int *)ptr[B_F11];
  T.R[peer][0] = (int *)ptr[B_R0];
  T.R[peer][1] = (int *)ptr[B_R1];
  T.ctr[peer] = (int *)ptr[B_CTR];
  T.out[peer] = (int4 *)ptr[B_OUT];
  return MFX_OK;
}

int mfx_part_attach_local(mfx_part *p, const mfx_part *q) {
  PartObj &o = p->o;
  const PartObj &r = q->o;
  if (r.P != o.P || r.rank == o.rank || r.n != o.n)
    return part_fail(MFX_VALUE_ERROR, "parts do not belong to the same partition set");
  if (r.device != o.device) {  // NVLink P2P between the GPUs of one process
    PCK(cudaSetDevice(o.device));
    cudaError_t e = cudaDeviceEnablePeerAccess(r.device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) PCK(e);
    cudaGetLastError();
  }
  const PeerTab &R = r.tab;  // r's own entry was set when r was created
  PeerTab &T = o.tab;
  const int k = r.rank;
  T.off[k] = R.off[k];
  T.adj[k] = R.adj[k];
  T.cap0[k] = R.cap0[k];
  T.pc[k] = R.pc[k];
  T.cf[k] = R.cf[k];
  T.ex[k] = R.ex[k];
  T.h[k] = R.h[k];
  T.mark[k] = R.mark[k];
  for (int a = 0; a < 2; ++a) {
    for (int b = 0; b < 2; ++b) T.F[k][a][b] = R.F[k][a][b];
    T.R[k][a] = R.R[k][a];
  }
  T.ctr[k] = R.ctr[k];
  T.out[k] = R.out[k];
  return MFX_OK;
}

// Phases.  args/out are 8 x int64; see include/mfx.h for the meaning.
int mfx_part_sync(mfx_part *pp) {
  PartObj &o = pp->o;
  PCK(cudaSetDevice(o.device));
  PCK(cudaStreamSynchronize(o.stream));
  PCK(cudaGetLastError());
  return MFX_OK;
}

int mfx_part_phase(mfx_part *pp, int phase, const int64_t *args, int64_t *out) {
  const bool async = (phase & MFX_PH_ASYNC) != 0;
  phase &= ~MFX_PH_ASYNC;
  if (async && (phase == MFX_PH_LINK || phase == MFX_PH_LINK_PC || phase == MFX_PH_SWAP ||
                phase == MFX_PH_FINAL || phase == MFX_PH_ACTIVE || phase == MFX_PH_BATCH_RESOLVE))
    return part_fail(MFX_VALUE_ERROR, "partition phase %d returns results: no async form", phase);
  PartObj &o = pp->o;
  PCK(cudaSetDevice(o.device));
  cudaStream_t st = o.stream;
  const PeerTab &T = o.tab;
  const int me = o.rank;
  int *ctr = (int *)o.buf[B_CTR];
  const int G = o.num_sms * 4;
  for (int k = 0; k < 8; ++k) out[k] = 0;
  for (int p = 0; p < o.P; ++p)
    if (!T.off[p]) return part_fail(MFX_VALUE_ERROR, "part %d not attached to peer %d", me, p);
  switch (phase) {
    case MFX_PH_LINK: {
      PCK(cudaMemsetAsync(ctr + PC_BAD, 0, sizeof(int), st));
      if (o.S > 0)
        part_rev_kernel<<<pgrid(o.S, o.num_sms), kPartBlock, 0, st>>>(
            T, me, o.nl, o.S, (const int *)o.buf[B_OFF], (const int *)o.buf[B_ADJ], o.rev, ctr);
      count_launch();
      break;
    }
    case MFX_PH_LINK_PC: {
      if (o.S > 0)
        part_pc_kernel<<<pgrid(o.S, o.num_sms), kPartBlock, 0, st>>>(T, me, o.S, o.rev, ctr);
      count_launch();
      break;
    }
    case MFX_PH_INIT: {
      part_init_kernel<<<pgrid((long long)o.S + o.nl, o.num_sms), kPartBlock, 0, st>>>(T, me, o.nl, o.S);
      PCK(cudaMemsetAsync(o.stat, 0, sizeof(unsigned long long) * PS_N, st));
      count_launch();
      break;
    }
    case MFX_PH_SATURATE: {
      if (o.s >= o.lo && o.s < o.hi) {
        part_saturate_kernel<<<o.num_sms, kPartBlock, 0, st>>>(T, me, o.s - o.lo, o.rev,
                                                                args[0] ? o.err : nullptr);
        count_launch();
      }
      break;
    }
    case MFX_PH_BFS_INIT: {  // args: dyn
      PCK(cudaMemsetAsync(ctr, 0, sizeof(int) * PC_N, st));
      int forbidden = args[0] ? o.s : -1;
      part_bfs_init_kernel<<<pgrid(o.nl, o.num_sms), kPartBlock, 0, st>>>(
          T, me, o.nl, o.s, o.t, (int)args[0], forbidden, o.bases);
      count_launch();
      break;
    }
    case MFX_PH_BFS_EXPAND: {  // args: L, cur, cnt0, cnt1, dyn, bottom-up
      int forbidden = args[4] ? o.s : -1;
      if (args[5]) {  // the level's frontier is {h == L} on every part
        part_bfs_bottomup_kernel<<<G, kPartBlock, 0, st>>>(T, me, o.nl, (int)args[0], (int)args[1],
                                                           o.s, o.t, forbidden, o.rcap);
        count_launch();
      } else if (args[2] + args[3] > 0) {
        part_bfs_expand_kernel<<<G, kPartBlock, 0, st>>>(T, me, (int)args[0], (int)args[1],
                                                         (int)args[2], (int)args[3], o.s, o.t,
                                                         forbidden, o.rcap, o.huge, o.nhuge);
        count_launch();
      }
      break;
    }
    case MFX_PH_SWAP: {  // -> out: next frontier per bin, round-list tails, active, reached, ovf, bases
      if (o.inbox_pending && o.P > 1) {  // the last push phase's buffered cut-slot pushes
        part_inbox_kernel<<<G, kPartBlock, 0, st>>>(T, me, o.push_stamp, o.s, o.t, o.rcap, o.stat);
        part_inbox_reset_kernel<<<1, 32, 0, st>>>(T, me);
        count_launch(2);
      }
      o.inbox_pending = false;
      int h[PC_N];
      PCK(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, st));
      PCK(cudaStreamSynchronize(st));
      PCK(cudaMemsetAsync(ctr + PC_FN0, 0, 2 * sizeof(int), st));
      for (int k = 0; k < 8; ++k) out[k] = h[k];
      break;
    }
    case MFX_PH_PUSH: {  // args: b0, e0, b1, e1, kc, stamp
      int b0 = (int)args[0], e0 = (int)std::min<int64_t>(args[1], o.rcap);
      int b1 = (int)args[2], e1 = (int)std::min<int64_t>(args[3], o.rcap);
      o.inbox_pending = true;  // (peers may buffer pushes toward this part)
      o.push_stamp = (unsigned)args[5];
      if (e0 > b0 || e1 > b1) {
        PCK(cudaMemsetAsync(o.hub_cnt, 0, sizeof(int), st));
        part_push_kernel<<<G, kPartBlock, 0, st>>>(T, me, b0, e0, b1, e1, (int)args[4],
                                                   (unsigned)args[5], o.s, o.t, o.rcap, o.rev,
                                                   o.stat, o.hub_list, o.hub_cnt, o.hub_best,
                                                   o.hub_taken);
        part_hub_scan_kernel<<<G, kPartBlock, 0, st>>>(T, me, o.hub_list, o.hub_cnt, o.hub_best,
                                                       o.hub_snap);
        part_hub_push_kernel<<<G, kPartBlock, 0, st>>>(T, me, o.hub_list, o.hub_cnt, o.hub_best,
                                                       o.hub_snap, o.hub_taken, (unsigned)args[5],
                                                       o.s, o.t, o.rcap, o.rev, o.stat);
        part_hub_tail_kernel<<<o.num_sms, kPartBlock, 0, st>>>(T, me, o.hub_list, o.hub_cnt,
                                                               (unsigned)args[5], o.s, o.t, o.rcap);
        count_launch(4);
      }
      break;
    }
    case MFX_PH_REPAIR: {  // args: e0, e1
      int e0 = (int)std::min<int64_t>(args[0], o.rcap), e1 = (int)std::min<int64_t>(args[1], o.rcap);
      if (e0 + e1 > 0) {  // (the scope is the round's relabel list)
        part_repair_kernel<<<G, kPartBlock, 0, st>>>(T, me, o.rev, o.stat);
        PCK(cudaMemsetAsync(o.rl_cnt, 0, 2 * sizeof(int), st));
        count_launch();
      }
      break;
    }
    case MFX_PH_FINAL: {  // args: #bases -> out[0] flow partial, out[1] cut partial
      PCK(cudaMemsetAsync(o.stat + PS_FLOW, 0, 2 * sizeof(unsigned long long), st));
      part_final_kernel<<<G, kPartBlock, 0, st>>>(T, me, o.S, (int)args[0], o.bases, o.orig, o.src,
                                                  o.stat);
      count_launch();
      break;
    }
    case MFX_PH_TOPO_SEED: {
      PCK(cudaMemsetAsync(ctr + PC_RT0, 0, 2 * sizeof(int), st));
      part_topo_seed_kernel<<<pgrid(o.nl, o.num_sms), kPartBlock, 0, st>>>(T, me, o.nl, o.s, o.t,
                                                                           o.rcap);
      count_launch();
      break;
    }
    case MFX_PH_ACTIVE: {
      PCK(cudaMemsetAsync(o.stat + PS_ACTIVE, 0, sizeof(unsigned long long), st));
      part_active_kernel<<<pgrid(o.nl, o.num_sms), kPartBlock, 0, st>>>(T, me, o.nl, o.s, o.t, o.stat);
      count_launch();
      break;
    }
    case MFX_PH_BATCH_RESOLVE: {
      long long init[PE_N];
      for (int k = 0; k < PE_N; ++k) init[k] = LLONG_MAX;
      PCK(cudaMemcpyAsync(o.err, init, sizeof(init), cudaMemcpyHostToDevice, st));
      long long k = o.bk;
      if (k > 0) {
        const long long *B = (const long long *)o.bbuf;
        int g = pgrid(k, o.num_sms);
        part_batch_resolve_kernel<<<g, kPartBlock, 0, st>>>(T, me, k, B, B + o.bcap, B + 2 * o.bcap,
                                                            B + 3 * o.bcap, o.orig, o.rev, o.bslot,
                                                            o.slot_first, o.err);
        part_batch_dup_kernel<<<g, kPartBlock, 0, st>>>(k, o.slot_base, o.bslot, o.slot_first,
                                                        B + 3 * o.bcap, o.err);
        part_batch_dupidx_kernel<<<g, kPartBlock, 0, st>>>(k, o.slot_base, o.bslot, o.slot_first,
                                                           B + 3 * o.bcap, o.err);
        count_launch(3);
      }
      long long h[PE_N];
      PCK(cudaMemcpyAsync(h, o.err, sizeof(h), cudaMemcpyDeviceToHost, st));
      PCK(cudaStreamSynchronize(st));
      for (int q = 0; q < 8; ++q) out[q] = h[q];
      break;
    }
    case MFX_PH_BATCH_APPLY: {  // args: apply (0 = only restore scratch)
      long long k = o.bk;
      if (k > 0) {
        const long long *B = (const long long *)o.bbuf;
        part_batch_apply_kernel<<<pgrid(k, o.num_sms), kPartBlock, 0, st>>>(
            T, me, k, B + 2 * o.bcap, o.bslot, o.slot_first, (int)args[0]);
        count_launch();
      }
      break;
    }
    case MFX_PH_BATCH_FIX: {
      long long k = o.bk;
      if (k > 0) {
        const long long *B = (const long long *)o.bbuf;
        part_batch_fix_kernel<<<pgrid(k, o.num_sms), kPartBlock, 0, st>>>(T, me, k, B, o.bslot, o.rev);
        count_launch();
      }
      break;
    }
    default:
      return part_fail(MFX_VALUE_ERROR, "unknown partition phase %d", phase);
  }
  PCK(cudaGetLastError());
  if (async) return MFX_OK;  // (enqueued; mfx_part_sync waits, nothing is read back)
  PCK(cudaStreamSynchronize(st));
  if (phase == MFX_PH_LINK || phase == MFX_PH_LINK_PC) {
    int bad = 0;
    PCK(cudaMemcpy(&bad, ctr + PC_BAD, sizeof(int), cudaMemcpyDeviceToHost));
    if (bad)
      return part_fail(MFX_VALUE_ERROR,
                       phase == MFX_PH_LINK ? "%d slots without a reverse slot in the owning part"
                                            : "%d pair capacities overflow int32 residual storage",
                       bad);
  }
  if (phase == MFX_PH_FINAL || phase == MFX_PH_ACTIVE || phase == MFX_PH_PUSH ||
      phase == MFX_PH_REPAIR || phase == MFX_PH_INIT) {
    unsigned long long h[PS_N];
    PCK(cudaMemcpy(h, o.stat, sizeof(h), cudaMemcpyDeviceToHost));
    if (phase == MFX_PH_FINAL) {
      out[0] = (int64_t)h[PS_FLOW];
      out[1] = (int64_t)h[PS_CUT];
    } else if (phase == MFX_PH_ACTIVE) {
      out[0] = (int64_t)h[PS_ACTIVE];
    } else {
      out[0] = (int64_t)h[PS_PUSH];
      out[1] = (int64_t)h[PS_RELABEL];
      out[2] = (int64_t)h[PS_REPAIR];
      out[3] = (int64_t)h[PS_BYTES];
    }
  }
  return MFX_OK;
}

// Stage this part's share of an update batch (host arrays; gidx = the
// update's index in the whole batch, for reference-identical error reports).
int mfx_part_stage_batch(mfx_part *pp, int64_t k, const int64_t *us, const int64_t *vs,
                         const int64_t *caps, const int64_t *gidx, int64_t slot_base) {
  PartObj &o = pp->o;
  PCK(cudaSetDevice(o.device));
  for (int64_t j = 0; j < k; ++j)
    if (us[j] < o.lo || us[j] >= o.hi)
      return part_fail(MFX_VALUE_ERROR, "update %lld routed to the wrong part", (long long)gidx[j]);
  if (k > o.bcap) {
    if (o.bbuf) cudaFree(o.bbuf);
    if (o.bslot) cudaFree(o.bslot);
    o.bbuf = nullptr;
    o.bslot = nullptr;
    long long cap = k > 1024 ? k : 1024;
    PCK(cudaMalloc(&o.bbuf, sizeof(long long) * 4 * (size_t)cap));
    PCK(cudaMalloc(&o.bslot, sizeof(int) * (size_t)cap));
    o.bcap = cap;
  }
  o.bk = (int)k;
  o.slot_base = slot_base;
  if (k > 0) {
    long long *B = o.bbuf;
    PCK(cudaMemcpyAsync(B, us, sizeof(int64_t) * k, cudaMemcpyHostToDevice, o.stream));
    PCK(cudaMemcpyAsync(B + o.bcap, vs, sizeof(int64_t) * k, cudaMemcpyHostToDevice, o.stream));
    PCK(cudaMemcpyAsync(B + 2 * o.bcap, caps, sizeof(int64_t) * k, cudaMemcpyHostToDevice, o.stream));
    PCK(cudaMemcpyAsync(B + 3 * o.bcap, gidx, sizeof(int64_t) * k, cudaMemcpyHostToDevice, o.stream));
    PCK(cudaStreamSynchronize(o.stream));
  }
  return MFX_OK;
}

// Download the local arrays (any may be NULL): off[nl+1], adj/rev/cap0/cf[S]
// (int64, rev as local slot indices of the owner), orig[S], excess/height[nl].
// Sample k_dec decrements then k_inc increments from this part's original
// slots (host output arrays of k_dec + k_inc entries, (u, v)-sorted within
// each kind); *got = updates produced.
int mfx_part_sample_batch(mfx_part *pp, int64_t k_dec, int64_t k_inc, uint64_t seed, double bias,
                          int64_t *us, int64_t *vs, int64_t *caps, int64_t *got) {
  PartObj &o = pp->o;
  PCK(cudaSetDevice(o.device));
  cudaStream_t st = o.stream;
  *got = 0;
  const long long S = o.S;
  if (S == 0 || k_dec + k_inc == 0) return MFX_OK;
  uint8_t *taken = nullptr;
  PCK(cudaMalloc(&taken, (size_t)S));
  PCK(cudaMemsetAsync(taken, 0, (size_t)S, st));
  unsigned long long *acc = nullptr;
  PCK(cudaMalloc(&acc, sizeof(unsigned long long)));
  PCK(cudaMemsetAsync(acc, 0, sizeof(unsigned long long), st));
  part_weight_kernel<<<pgrid(S, o.num_sms), kPartBlock, 0, st>>>(o.tab, o.rank, S, o.orig, o.s, o.t,
                                                               bias, acc);
  unsigned long long W = 0;
  PCK(cudaMemcpyAsync(&W, acc, sizeof(W), cudaMemcpyDeviceToHost, st));
  PCK(cudaStreamSynchronize(st));
  long long done = 0;
  std::vector<int> all_slots;
  for (int kind = 0; kind < 2; ++kind) {
    const long long want = kind == 0 ? k_dec : k_inc;
    if (want <= 0) continue;
    const int cap = (int)std::min<long long>(8 * want + 4096, S);
    unsigned long long *cand = nullptr, *sorted = nullptr;
    int *cnt = nullptr;
    PCK(cudaMalloc(&cand, sizeof(unsigned long long) * cap));
    PCK(cudaMalloc(&sorted, sizeof(unsigned long long) * cap));
    PCK(cudaMalloc(&cnt, sizeof(int)));
    double tau = 3.0 * (double)want / (double)(W > 0 ? W : 1) + 1e-12;
    int c = 0;
    for (int it = 0; it < 60; ++it) {
      PCK(cudaMemsetAsync(cnt, 0, sizeof(int), st));
      part_sample_kernel<<<pgrid(S, o.num_sms), kPartBlock, 0, st>>>(
          o.tab, o.rank, o.nl, S, o.orig, taken, o.s, o.t, bias, seed * 2 + kind, kind == 0, tau,
          cap, cand, cnt);
      PCK(cudaMemcpyAsync(&c, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
      PCK(cudaStreamSynchronize(st));
      count_launch();
      if (c > cap) tau *= 0.5;                       // too many candidates
      else if (c < want && tau < 1e30) tau *= 4.0;  // too few: widen (or nothing left)
      else break;
      if (c < want && tau >= 1e30) break;
    }
    if (c > cap) c = cap;
    size_t tb = 0;
    PCK(cub::DeviceRadixSort::SortKeys(nullptr, tb, cand, sorted, c, 0, 64, st));
    void *tmp = nullptr;
    PCK(cudaMalloc(&tmp, tb > 0 ? tb : 1));
    PCK(cub::DeviceRadixSort::SortKeys(tmp, tb, cand, sorted, c, 0, 64, st));
    std::vector<unsigned long long> h((size_t)c);
    PCK(cudaMemcpyAsync(h.data(), sorted, sizeof(unsigned long long) * (size_t)c,
                        cudaMemcpyDeviceToHost, st));
    PCK(cudaStreamSynchronize(st));
    long long take = std::min<long long>(want, c);
    std::vector<int> slots((size_t)take);
    for (long long j = 0; j < take; ++j) slots[j] = (int)(h[j] & 0xFFFFFFFFull);
    std::sort(slots.begin(), slots.end());
    int *d_slots = nullptr;
    long long *d_out = nullptr;
    PCK(cudaMalloc(&d_slots, sizeof(int) * (size_t)(take > 0 ? take : 1)));
    PCK(cudaMalloc(&d_out, sizeof(long long) * 3 * (size_t)(take > 0 ? take : 1)));
    if (take > 0) {
      PCK(cudaMemcpyAsync(d_slots, slots.data(), sizeof(int) * take, cudaMemcpyHostToDevice, st));
      part_sample_emit_kernel<<<pgrid(take, o.num_sms), kPartBlock, 0, st>>>(
          o.tab, o.rank, o.nl, d_slots, (int)take, kind == 0, seed * 2 + kind, taken, d_out,
          d_out + take, d_out + 2 * take);
      PCK(cudaMemcpyAsync(us + done, d_out, sizeof(long long) * take, cudaMemcpyDeviceToHost, st));
      PCK(cudaMemcpyAsync(vs + done, d_out + take, sizeof(long long) * take, cudaMemcpyDeviceToHost, st));
      PCK(cudaMemcpyAsync(caps + done, d_out + 2 * take, sizeof(long long) * take,
                          cudaMemcpyDeviceToHost, st));
      PCK(cudaStreamSynchronize(st));
      count_launch();
    }
    done += take;
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
  return MFX_OK;
}

int mfx_part_download(const mfx_part *pp, int64_t *off, int64_t *adj, int64_t *rev, int64_t *cap0,
                      int64_t *cf, uint8_t *orig, int64_t *excess, int64_t *height) {
  const PartObj &o = pp->o;
  PCK(cudaSetDevice(o.device));
  auto widen = [&](const void *d, int64_t *h, size_t cnt) -> int {
    if (!h || cnt == 0) return MFX_OK;
    std::vector<int> tmp(cnt);
    PCK(cudaMemcpy(tmp.data(), d, sizeof(int) * cnt, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < cnt; ++i) h[i] = tmp[i];
    return MFX_OK;
  };
  int rc;
  if ((rc = widen(o.buf[B_OFF], off, (size_t)o.nl + 1))) return rc;
  if ((rc = widen(o.buf[B_ADJ], adj, (size_t)o.S))) return rc;
  if ((rc = widen(o.rev, rev, (size_t)o.S))) return rc;
  if ((rc = widen(o.buf[B_CAP0], cap0, (size_t)o.S))) return rc;
  if ((rc = widen(o.buf[B_CF], cf, (size_t)o.S))) return rc;
  if ((rc = widen(o.buf[B_H], height, (size_t)o.nl))) return rc;
  if (orig && o.S > 0) PCK(cudaMemcpy(orig, o.orig, (size_t)o.S, cudaMemcpyDeviceToHost));
  if (excess && o.nl > 0)
    PCK(cudaMemcpy(excess, o.buf[B_EX], sizeof(int64_t) * (size_t)o.nl, cudaMemcpyDeviceToHost));
  return MFX_OK;
}

}  // extern "C"
