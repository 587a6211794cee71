// build.cu -- GPU Bi-CSR builder (build_bicsr, graph.py:126-174).
//
// The reference normalises with np.unique twice plus np.add.at and finds the
// reverse slot with a global searchsorted.  On the device:
//   validate   first bad source / target / capacity index (graph.py:48-61)
//   keys       (u << vb) | v, self-loops mapped to a sentinel that sorts last
//   sort       CUB radix sort of (key, cap) over the significant bits only
//   merge      reduce-by-key: parallel edges summed (graph.py:143-147)
//   closure    append every swapped key with cap 0, sort, reduce-by-key with
//              payload cap*2 + origin so caps sum and origin flags OR
//              (graph.py:152-163)
//   decode     adj / cap0 / is_original; row offsets by binary search of the
//              sorted keys (graph.py:167-168)
//   rev        binary search of u inside row v (graph.py:171)
// The slot order equals the reference's (u*n + v order), so every array is
// bit-identical to the reference's.
#include <limits.h>

#include <cub/cub.cuh>

#include "engine.h"

namespace mfx {

static inline int grid_for(long long work, int num_sms) {
  long long g = (work + kBlock - 1) / kBlock;
  long long cap = (long long)num_sms * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

static int bitlen(unsigned long long x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

#define GS_LOOP(i, cnt)                                                        \
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (cnt); \
       i += (long long)gridDim.x * blockDim.x)

__global__ void validate_kernel(long long n, long long m, const long long *us, const long long *vs,
                                const long long *caps, long long *err) {
  GS_LOOP(i, m) {
    if (us[i] < 0 || us[i] >= n) atomicMin(err + 0, i);
    if (vs[i] < 0 || vs[i] >= n) atomicMin(err + 1, i);
    if (caps[i] < 0) atomicMin(err + 2, i);
  }
}

__global__ void make_keys_kernel(long long m, const long long *us, const long long *vs,
                                 const long long *caps, int vb, unsigned long long sentinel,
                                 unsigned long long *keys, long long *vals,
                                 unsigned long long *selfloops) {
  unsigned long long sl = 0;
  GS_LOOP(i, m) {
    long long u = us[i], v = vs[i];
    if (u == v) {
      keys[i] = sentinel;
      ++sl;
    } else {
      keys[i] = ((unsigned long long)u << vb) | (unsigned long long)v;
    }
    vals[i] = caps[i];
  }
  sl = warp_sum(sl);
  if ((threadIdx.x & 31) == 0 && sl) atomicAdd(selfloops, sl);
}

// first half: merged original edges (payload cap*2+1); second half: swapped
// zero-capacity candidates (payload 0)
__global__ void closure_kernel(long long m1, const unsigned long long *ukeys, const long long *ucaps,
                               int vb, unsigned long long *keys2, long long *vals2) {
  unsigned long long vmask = (1ull << vb) - 1;
  GS_LOOP(i, m1) {
    unsigned long long k = ukeys[i];
    keys2[i] = k;
    vals2[i] = ucaps[i] * 2 + 1;
    keys2[m1 + i] = ((k & vmask) << vb) | (k >> vb);
    vals2[m1 + i] = 0;
  }
}

__global__ void decode_kernel(long long S, const unsigned long long *skeys, const long long *svals,
                              int vb, int *adj, long long *cap0, uint8_t *orig) {
  unsigned long long vmask = (1ull << vb) - 1;
  GS_LOOP(i, S) {
    adj[i] = (int)(skeys[i] & vmask);
    cap0[i] = svals[i] >> 1;
    orig[i] = (uint8_t)(svals[i] & 1);
  }
}

// off[u] = first slot whose tail >= u (lower bound on the sorted keys)
__global__ void offsets_kernel(long long n, long long S, const unsigned long long *skeys, int vb,
                               int *off) {
  GS_LOOP(u, n + 1) {
    unsigned long long want = (unsigned long long)u << vb;
    long long lo = 0, hi = S;
    while (lo < hi) {
      long long mid = (lo + hi) >> 1;
      if (skeys[mid] < want) lo = mid + 1;
      else hi = mid;
    }
    off[u] = (int)lo;
  }
}

// rev[i]: slot of (adj[i], src[i]) found inside row adj[i]
__global__ void rev_kernel(long long S, const unsigned long long *skeys, int vb, const int *off,
                           const int *adj, int *rev) {
  GS_LOOP(i, S) {
    int u = (int)(skeys[i] >> vb), v = adj[i];
    int lo = off[v], hi = off[v + 1];
    while (lo < hi) {
      int mid = lo + ((hi - lo) >> 1);
      if (adj[mid] < u) lo = mid + 1;
      else hi = mid;
    }
    rev[i] = lo;
  }
}

__global__ void pair_max_kernel(long long S, const int *rev, const long long *cap0,
                                unsigned long long *out) {
  unsigned long long mx = 0;
  GS_LOOP(i, S) {
    unsigned long long p = (unsigned long long)(cap0[i] + cap0[rev[i]]);
    mx = p > mx ? p : mx;
  }
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = w > mx ? w : mx;
  }
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, mx);
}

__global__ void src_kernel(long long S, long long n, const int *off, long long *src) {
  GS_LOOP(i, S) {
    long long lo = 0, hi = n;  // largest u with off[u] <= i
    while (lo < hi) {
      long long mid = (lo + hi + 1) >> 1;
      if (off[mid] <= i) lo = mid;
      else hi = mid - 1;
    }
    src[i] = lo;
  }
}

__global__ void narrow_idx_kernel(long long cnt, const long long *src, int *dst) {
  GS_LOOP(i, cnt) dst[i] = (int)src[i];
}

struct DevBuf {
  void *p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 16); }
  template <typename T>
  T *as() const {
    return (T *)p;
  }
};

#define CKE(x)                           \
  do {                                   \
    cudaError_t _e = (x);                \
    if (_e != cudaSuccess) return _e;    \
  } while (0)

cudaError_t build_bicsr_device(int64_t n, int64_t m, const int64_t *d_us, const int64_t *d_vs,
                               const int64_t *d_caps, Topology &topo, int64_t **d_cap0_out,
                               int64_t err[2], int *launches) {
  cudaStream_t st = topo.stream;
  err[0] = 0;
  err[1] = -1;
  if (n <= 0) {
    err[0] = 1;
    return cudaSuccess;
  }
  const long long *us = (const long long *)d_us, *vs = (const long long *)d_vs,
                  *caps = (const long long *)d_caps;
  int nl = 0;
  // ---- validate ----
  DevBuf e3;
  CKE(e3.alloc(4 * sizeof(long long)));
  {
    long long init[4] = {LLONG_MAX, LLONG_MAX, LLONG_MAX, 0};
    CKE(cudaMemcpyAsync(e3.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
  }
  if (m > 0) {
    validate_kernel<<<grid_for(m, topo.num_sms), kBlock, 0, st>>>(n, m, us, vs, caps,
                                                                  e3.as<long long>());
    ++nl;
  }
  long long hv[4];
  CKE(cudaMemcpyAsync(hv, e3.p, sizeof(hv), cudaMemcpyDeviceToHost, st));
  CKE(cudaStreamSynchronize(st));
  for (int k = 0; k < 3; ++k)
    if (hv[k] != LLONG_MAX) {
      err[0] = 2 + k;
      err[1] = hv[k];
      return cudaSuccess;
    }
  int vb = bitlen((unsigned long long)n);           // v < 2^vb (and n itself fits)
  int ub = bitlen((unsigned long long)n);           // u <= n (sentinel u = n)
  int end_bit = vb + ub;
  unsigned long long sentinel = (unsigned long long)n << vb;

  // ---- keys + first sort/merge ----
  size_t M = (size_t)(m > 0 ? m : 1);
  DevBuf k0, k1, v0, v1, cnt;
  CKE(k0.alloc(M * 16));  // room for the closure (2 * m1 <= 2 * m)
  CKE(k1.alloc(M * 16));
  CKE(v0.alloc(M * 16));
  CKE(v1.alloc(M * 16));
  CKE(cnt.alloc(4 * sizeof(unsigned long long)));
  CKE(cudaMemsetAsync(cnt.p, 0, 4 * sizeof(unsigned long long), st));
  unsigned long long *K0 = k0.as<unsigned long long>(), *K1 = k1.as<unsigned long long>();
  long long *V0 = v0.as<long long>(), *V1 = v1.as<long long>();
  unsigned long long *C = cnt.as<unsigned long long>();
  if (m > 0) {
    make_keys_kernel<<<grid_for(m, topo.num_sms), kBlock, 0, st>>>(m, us, vs, caps, vb, sentinel,
                                                                   K0, V0, C + 0);
    ++nl;
  }
  size_t tmp_bytes = 0, tb = 0;
  CKE(cub::DeviceRadixSort::SortPairs(nullptr, tb, K0, K1, V0, V1, (int64_t)(2 * M), 0, end_bit, st));
  tmp_bytes = tb;
  CKE(cub::DeviceReduce::ReduceByKey(nullptr, tb, K1, K0, V1, V0, (long long *)(C + 1),
                                     ::cuda::std::plus<long long>{}, (int64_t)(2 * M), st));
  tmp_bytes = tb > tmp_bytes ? tb : tmp_bytes;
  DevBuf tmp;
  CKE(tmp.alloc(tmp_bytes));
  unsigned long long h_sl = 0;
  long long m1 = 0, S = 0;
  if (m > 0) {
    tb = tmp_bytes;
    CKE(cub::DeviceRadixSort::SortPairs(tmp.p, tb, K0, K1, V0, V1, (int64_t)m, 0, end_bit, st));
    CKE(cudaMemcpyAsync(&h_sl, C + 0, sizeof(h_sl), cudaMemcpyDeviceToHost, st));
    CKE(cudaStreamSynchronize(st));
    long long kept = m - (long long)h_sl;
    if (kept > 0) {
      tb = tmp_bytes;
      CKE(cub::DeviceReduce::ReduceByKey(tmp.p, tb, K1, K0, V1, V0, (long long *)(C + 1),
                                         ::cuda::std::plus<long long>{}, (int64_t)kept, st));
      CKE(cudaMemcpyAsync(&m1, C + 1, sizeof(m1), cudaMemcpyDeviceToHost, st));
      CKE(cudaStreamSynchronize(st));
    }
    nl += 4;
  }
  // ---- closure + second sort/merge ----
  if (m1 > 0) {
    closure_kernel<<<grid_for(m1, topo.num_sms), kBlock, 0, st>>>(m1, K0, V0, vb, K1, V1);
    tb = tmp_bytes;
    CKE(cub::DeviceRadixSort::SortPairs(tmp.p, tb, K1, K0, V1, V0, (int64_t)(2 * m1), 0, end_bit, st));
    tb = tmp_bytes;
    CKE(cub::DeviceReduce::ReduceByKey(tmp.p, tb, K0, K1, V0, V1, (long long *)(C + 2),
                                       ::cuda::std::plus<long long>{}, (int64_t)(2 * m1), st));
    CKE(cudaMemcpyAsync(&S, C + 2, sizeof(S), cudaMemcpyDeviceToHost, st));
    CKE(cudaStreamSynchronize(st));
    nl += 5;
  }
  if (S >= INT_MAX || n >= INT_MAX) {
    err[0] = 5;  // exceeds the int32 slot-index layout of one device
    return cudaSuccess;
  }
  // ---- decode into the topology ----
  topo.n = (int)n;
  topo.S = (int)S;
  topo.m_original = (int)m1;
  topo.diag[0] = (int64_t)h_sl;
  topo.diag[1] = (m - (int64_t)h_sl) - m1;
  topo.diag[2] = S - m1;
  CKE(cudaMalloc(&topo.off, sizeof(int) * (size_t)(n + 1)));
  CKE(cudaMalloc(&topo.adj, sizeof(int) * (size_t)(S > 0 ? S : 1)));
  CKE(cudaMalloc(&topo.rev, sizeof(int) * (size_t)(S > 0 ? S : 1)));
  CKE(cudaMalloc(&topo.orig, (size_t)(S > 0 ? S : 1)));
  int64_t *cap0 = nullptr;
  CKE(cudaMalloc(&cap0, sizeof(int64_t) * (size_t)(S > 0 ? S : 1)));
  *d_cap0_out = cap0;
  if (S > 0)
    decode_kernel<<<grid_for(S, topo.num_sms), kBlock, 0, st>>>(S, K1, V1, vb, topo.adj,
                                                                (long long *)cap0, topo.orig);
  offsets_kernel<<<grid_for(n + 1, topo.num_sms), kBlock, 0, st>>>(n, S, K1, vb, topo.off);
  if (S > 0)
    rev_kernel<<<grid_for(S, topo.num_sms), kBlock, 0, st>>>(S, K1, vb, topo.off, topo.adj, topo.rev);
  nl += 3;
  CKE(cudaGetLastError());
  CKE(cudaStreamSynchronize(st));
  if (launches) *launches += nl;
  count_launch(nl);
  return cudaSuccess;
}

cudaError_t topology_from_bicsr(int64_t n, int64_t S, const int64_t *d_off, const int64_t *d_adj,
                                const int64_t *d_rev, const uint8_t *d_orig, Topology &topo) {
  cudaStream_t st = topo.stream;
  topo.n = (int)n;
  topo.S = (int)S;
  CKE(cudaMalloc(&topo.off, sizeof(int) * (size_t)(n + 1)));
  CKE(cudaMalloc(&topo.adj, sizeof(int) * (size_t)(S > 0 ? S : 1)));
  CKE(cudaMalloc(&topo.rev, sizeof(int) * (size_t)(S > 0 ? S : 1)));
  CKE(cudaMalloc(&topo.orig, (size_t)(S > 0 ? S : 1)));
  narrow_idx_kernel<<<grid_for(n + 1, topo.num_sms), kBlock, 0, st>>>(n + 1, (const long long *)d_off,
                                                                      topo.off);
  if (S > 0) {
    narrow_idx_kernel<<<grid_for(S, topo.num_sms), kBlock, 0, st>>>(S, (const long long *)d_adj,
                                                                    topo.adj);
    narrow_idx_kernel<<<grid_for(S, topo.num_sms), kBlock, 0, st>>>(S, (const long long *)d_rev,
                                                                    topo.rev);
    CKE(cudaMemcpyAsync(topo.orig, d_orig, (size_t)S, cudaMemcpyDeviceToDevice, st));
  }
  count_launch(3);
  return cudaGetLastError();
}

cudaError_t download_src(const Topology &topo, int64_t *d_src) {
  if (topo.S == 0) return cudaSuccess;
  src_kernel<<<grid_for(topo.S, topo.num_sms), kBlock, 0, topo.stream>>>(topo.S, topo.n, topo.off,
                                                                         (long long *)d_src);
  count_launch();
  return cudaGetLastError();
}

cudaError_t pair_max_int64(const Topology &topo, const int64_t *d_cap0, unsigned long long *d_out) {
  CKE(cudaMemsetAsync(d_out, 0, sizeof(unsigned long long), topo.stream));
  if (topo.S == 0) return cudaSuccess;
  pair_max_kernel<<<grid_for(topo.S, topo.num_sms), kBlock, 0, topo.stream>>>(
      topo.S, topo.rev, (const long long *)d_cap0, d_out);
  count_launch();
  return cudaGetLastError();
}

}  // namespace mfx
