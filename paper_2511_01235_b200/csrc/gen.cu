// gen.cu -- device-side synthetic input for the largest configuration (C5,
// R-MAT scale 26: 1.07 B edges, which numpy on the host would take minutes
// and ~25 GB of host memory to draw) and the slot-balanced vertex-range cut
// for the partitioned engine.
//
// The R-MAT recursion is the one of paper_2511_01235_b200/gen.py rmat_graph
// (SURVEY Appendix B): per bit, r ~ U[0,1); u gets the bit when r >= a+b, v
// when a <= r < a+b or r >= a+b+c; caps U[1,100]; s = argmax out-degree, t =
// argmax in-degree != s.  Only the random stream differs (a counter-based
// splitmix64 hash of (seed, edge, bit) instead of numpy's PCG64), so a device
// graph is reproducible from its seed on any number of GPUs.
#include <limits.h>

#include <cub/cub.cuh>

#include "../../include/mfx.h"
#include "engine.h"

namespace mfx {

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ double u01(unsigned long long x) {
  return (double)(splitmix64(x) >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void rmat_kernel(long long m, int scale, unsigned long long seed, double a, double b,
                            double c, long long *us, long long *vs, long long *caps,
                            int *outdeg, int *indeg) {
  const double ab = a + b, abc = a + b + c;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    unsigned long long base = splitmix64(seed ^ 0x5851F42D4C957F2Dull) + (unsigned long long)e * 64ull;
    long long u = 0, v = 0;
    for (int bit = 0; bit < scale; ++bit) {
      double r = u01(base + bit);
      u |= (long long)(r >= ab) << bit;
      v |= (long long)((r >= a && r < ab) || r >= abc) << bit;
    }
    us[e] = u;
    vs[e] = v;
    caps[e] = 1 + (long long)(splitmix64(base + 63) % 100ull);
    atomicAdd(outdeg + u, 1);
    atomicAdd(indeg + v, 1);
  }
}

__global__ void exclude_kernel(int *deg, const cub::KeyValuePair<int, int> *s) { deg[s->key] = -1; }

// slot weight of a row: out-degree + in-degree (reverse stubs) + 1, as
// partition.balanced_bounds on the host
__global__ void slots_kernel(long long n, const int *deg, long long *w) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    w[i] = (long long)deg[i] + 1;
}

__global__ void degree_kernel(long long m, const long long *us, const long long *vs, int *deg) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    atomicAdd(deg + us[e], 1);
    atomicAdd(deg + vs[e], 1);
  }
}

static int ggrid(long long work, int sms) {
  long long g = (work + 255) / 256, cap = (long long)sms * 16;
  return (int)(g < 1 ? 1 : g > cap ? cap : g);
}

// bounds[0..P]: first vertex whose prefix slot weight reaches p/P of the total
static cudaError_t cut_bounds(long long n, const long long *d_w, int nparts, int sms,
                              cudaStream_t st, int64_t *bounds) {
  long long *scan = nullptr;
  cudaError_t e = cudaMalloc(&scan, sizeof(long long) * (size_t)n);
  if (e) return e;
  size_t tb = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, d_w, scan, (int64_t)n, st);
  void *tmp = nullptr;
  if ((e = cudaMalloc(&tmp, tb))) return e;
  cub::DeviceScan::InclusiveSum(tmp, tb, d_w, scan, (int64_t)n, st);
  long long total = 0;
  cudaMemcpyAsync(&total, scan + n - 1, sizeof(total), cudaMemcpyDeviceToHost, st);
  e = cudaStreamSynchronize(st);
  bounds[0] = 0;
  for (int p = 1; p < nparts; ++p) {  // host binary search over the device scan
    long long want = (long long)((double)total * p / nparts), lo = 0, hi = n;
    while (lo < hi) {
      long long mid = (lo + hi) / 2, x = 0;
      cudaMemcpy(&x, scan + mid, sizeof(x), cudaMemcpyDeviceToHost);
      if (x < want) lo = mid + 1;
      else hi = mid;
    }
    long long b = lo + 1;
    if (b <= bounds[p - 1]) b = bounds[p - 1] + 1;
    if (b > n - (nparts - p)) b = n - (nparts - p);
    bounds[p] = b;
  }
  bounds[nparts] = n;
  cudaFree(tmp);
  cudaFree(scan);
  count_launch(2);
  return e;
}

}  // namespace mfx

using namespace mfx;

extern "C" {

int mfx_rmat_device(int scale, int64_t edge_factor, uint64_t seed, double a, double b, double c,
                    int device, int64_t *d_us, int64_t *d_vs, int64_t *d_caps, int64_t *source,
                    int64_t *sink) {
  if (scale < 1 || scale > 30) {
    g_last_error = "R-MAT scale must be in [1, 30]";
    return MFX_VALUE_ERROR;
  }
  cudaError_t e = cudaSetDevice(device);
  int sms = 0;
  if (!e) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const long long n = 1ll << scale, m = n * edge_factor;
  int *deg = nullptr;
  if (!e) e = cudaMalloc(&deg, sizeof(int) * 2 * (size_t)n);
  if (!e) e = cudaMemset(deg, 0, sizeof(int) * 2 * (size_t)n);
  if (e) {
    g_last_error = cudaGetErrorString(e);
    return MFX_CUDA_ERROR;
  }
  rmat_kernel<<<ggrid(m, sms), 256>>>(m, scale, seed, a, b, c, (long long *)d_us,
                                      (long long *)d_vs, (long long *)d_caps, deg, deg + n);
  cub::KeyValuePair<int, int> *kv = nullptr;
  cudaMalloc(&kv, 2 * sizeof(*kv));
  size_t tb = 0;
  cub::DeviceReduce::ArgMax(nullptr, tb, deg, kv, (int)n);
  void *tmp = nullptr;
  cudaMalloc(&tmp, tb);
  cub::DeviceReduce::ArgMax(tmp, tb, deg, kv, (int)n);            // s: max out-degree
  exclude_kernel<<<1, 1>>>(deg + n, kv);                           // t != s
  cub::DeviceReduce::ArgMax(tmp, tb, deg + n, kv + 1, (int)n);    // t: max in-degree
  cub::KeyValuePair<int, int> h[2];
  e = cudaMemcpy(h, kv, sizeof(h), cudaMemcpyDeviceToHost);
  count_launch(4);
  cudaFree(tmp);
  cudaFree(kv);
  cudaFree(deg);
  if (!e) e = cudaGetLastError();
  if (e) {
    g_last_error = cudaGetErrorString(e);
    return MFX_CUDA_ERROR;
  }
  *source = h[0].key;
  *sink = h[1].key;
  return MFX_OK;
}

int mfx_part_bounds_device(int64_t n, int64_t m, const int64_t *d_us, const int64_t *d_vs,
                           int nparts, int device, int64_t *bounds) {
  if (nparts < 1 || nparts > 8 || nparts > n) {
    g_last_error = "nparts must be in [1, min(8, n)]";
    return MFX_VALUE_ERROR;
  }
  cudaError_t e = cudaSetDevice(device);
  int sms = 0;
  if (!e) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  int *deg = nullptr;
  long long *w = nullptr;
  if (!e) e = cudaMalloc(&deg, sizeof(int) * (size_t)n);
  if (!e) e = cudaMalloc(&w, sizeof(long long) * (size_t)n);
  if (!e) e = cudaMemset(deg, 0, sizeof(int) * (size_t)n);
  if (!e && m > 0)
    degree_kernel<<<ggrid(m, sms), 256>>>(m, (const long long *)d_us, (const long long *)d_vs, deg);
  if (!e) slots_kernel<<<ggrid(n, sms), 256>>>(n, deg, w);
  if (!e) e = cudaDeviceSynchronize();
  if (!e) e = cut_bounds(n, w, nparts, sms, 0, bounds);
  count_launch(2);
  cudaFree(deg);
  cudaFree(w);
  if (e) {
    g_last_error = cudaGetErrorString(e);
    return MFX_CUDA_ERROR;
  }
  return MFX_OK;
}

}  // extern "C"
