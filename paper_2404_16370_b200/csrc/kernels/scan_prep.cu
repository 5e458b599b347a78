// Device scan input pipeline: make_scan_cloud
// (filter.cpp:86-100) on the GPU — voxel downsample with leaf doubling
// (gaussian_cloud.cpp:110-144), kNN plane-model covariances
// (gaussian_cloud.cpp:36-90), the sensor-noise term, and the engine's
// per-scan records (plane-model parameters for the fast likelihood path).
//
// Compiled with -fmad=false (Makefile): every double operation is a single
// IEEE rounding in the source order, as in the -ffp-contract=off host build,
// so the prepared scan is bit-identical to host make_scan_cloud
// (tests/test_gpu_scan_prep.py).
//
//   voxel_downsample: 63-bit voxel key per point, stable CUB radix sort of
//     (key, index), one thread per voxel sums its points in input order; the
//     voxels are emitted in order of first appearance (flag + scan), which is
//     the reference's insertion order.
//   k_nearest (point_grid.cpp:51-107): the reference visits grid rings
//     outwards (z, y, x, then ascending index inside a cell), keeps the first
//     k+1 visited sorted stably by distance and replaces the last entry only
//     on a strictly smaller distance. Its result is therefore the k+1 smallest
//     (d2, visit rank) pairs, rank = (Chebyshev ring of the cells, z, y, x,
//     index); a scan has <= n_scan_max points, so each query ranks all of them.
//   covariance: canonical (x, y, z) order of the k neighbours, mean and
//     outer-product sums in that order, Jacobi eigen-decomposition (host
//     sym_eig3), Sigma = V diag(eps l, l, l) V^T + noise^2 I.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "../engine.cuh"
#include "../kernels.cuh"

namespace smcl {

namespace {

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

constexpr int64_t kKeyBias = int64_t(1) << 20;  // 21-bit key fields

// gaussian_cloud.cpp:117-121: floor(p / leaf) per axis, packed.
__global__ void k_voxel_keys(const double* __restrict__ p, int n, double leaf, uint64_t* __restrict__ key,
                             int32_t* __restrict__ iota, int* __restrict__ overflow) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t k = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double f = floor(p[3 * i + a] / leaf);
    int64_t c = (f >= -9.2e18 && f <= 9.2e18) ? static_cast<int64_t>(f) : INT64_MIN;
    c += kKeyBias;
    if (c < 0 || c >= 2 * kKeyBias) {
      atomicExch(overflow, 1);
      c = 0;
    }
    k = (k << 21) | static_cast<uint64_t>(c);
  }
  key[i] = k;
  iota[i] = i;
}

__global__ void k_voxel_heads(const uint64_t* __restrict__ skey, const int32_t* __restrict__ sidx, int n,
                              int32_t* __restrict__ head, int32_t* __restrict__ first_flag) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const bool h = p == 0 || skey[p] != skey[p - 1];
  head[p] = h ? 1 : 0;
  first_flag[sidx[p]] = h ? 1 : 0;  // first (lowest) input index of its voxel
}

// One thread per sorted position that starts a voxel: centroid in input order.
__global__ void k_voxel_centroids(const double* __restrict__ p, const uint64_t* __restrict__ skey,
                                  const int32_t* __restrict__ sidx, const int32_t* __restrict__ head, int n,
                                  const int32_t* __restrict__ out_pos_excl, double* __restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n || !head[s]) return;
  double sx = 0.0, sy = 0.0, sz = 0.0;
  int c = 0;
  for (int q = s; q < n && (q == s || skey[q] == skey[s]); ++q) {
    const int32_t i = sidx[q];
    sx = sx + p[3 * i];
    sy = sy + p[3 * i + 1];
    sz = sz + p[3 * i + 2];
    ++c;
  }
  const double d = static_cast<double>(c);
  const int o = out_pos_excl[sidx[s]];
  out[3 * o] = sx / d;
  out[3 * o + 1] = sy / d;
  out[3 * o + 2] = sz / d;
}

// Whole downsample_to (gaussian_cloud.cpp:134-144) in one block for n <=
// kBlockItems points: keys, stable block radix sort, voxel heads, leaf
// doubling until <= max_points voxels, first-appearance positions, centroids
// in input order, and the bounds of the result (kNN grid). One launch, no host
// round trip between leaf levels.
constexpr int kBlockThreads = 512, kBlockIpt = 8, kBlockItems = kBlockThreads * kBlockIpt;
using BlockSort = cub::BlockRadixSort<uint64_t, kBlockThreads, kBlockIpt, int32_t>;
using BlockScanI = cub::BlockScan<int32_t, kBlockThreads>;
struct BlockSmem {
  union {
    typename BlockSort::TempStorage sort;
    typename BlockScanI::TempStorage scan;
  } tmp;
  uint64_t key[kBlockItems];
  int32_t idx[kBlockItems];
  int32_t flag[kBlockItems];  // first-appearance flag by input index, then its exclusive scan
  int count, overflow;
  double lo[3][kBlockThreads / 32], hi[3][kBlockThreads / 32];
};

__global__ void __launch_bounds__(kBlockThreads) k_downsample_block(const double* __restrict__ p, int n, double leaf0,
                                                                   int max_points, double* __restrict__ out,
                                                                   int* __restrict__ info, double* __restrict__ bounds) {
  extern __shared__ __align__(16) unsigned char ds_raw[];
  BlockSmem& sm = *reinterpret_cast<BlockSmem*>(ds_raw);
  const int t = threadIdx.x;
  double leaf = leaf0;
  if (t == 0) {
    sm.count = 0;
    sm.overflow = 0;
  }
  __syncthreads();
  for (int level = 0; level < 64; ++level) {
    uint64_t keys[kBlockIpt];
    int32_t vals[kBlockIpt];
#pragma unroll
    for (int u = 0; u < kBlockIpt; ++u) {
      const int i = t * kBlockIpt + u;
      vals[u] = i;
      keys[u] = ~0ull;
      if (i < n) {
        uint64_t k = 0;
        for (int a = 0; a < 3; ++a) {
          const double f = floor(p[3 * i + a] / leaf);
          int64_t c = (f >= -9.2e18 && f <= 9.2e18) ? static_cast<int64_t>(f) : INT64_MIN;
          c += kKeyBias;
          if (c < 0 || c >= 2 * kKeyBias) {
            sm.overflow = 1;
            c = 0;
          }
          k = (k << 21) | static_cast<uint64_t>(c);
        }
        keys[u] = k;
      }
    }
    __syncthreads();
    BlockSort(sm.tmp.sort).Sort(keys, vals, 0, 64);  // stable; padding keys (all ones) sort last
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kBlockIpt; ++u) {
      sm.key[t * kBlockIpt + u] = keys[u];
      sm.idx[t * kBlockIpt + u] = vals[u];
    }
    __syncthreads();
    int heads = 0;
#pragma unroll
    for (int u = 0; u < kBlockIpt; ++u) {
      const int q = t * kBlockIpt + u;
      if (q < n) {
        const bool h = q == 0 || sm.key[q] != sm.key[q - 1];
        sm.flag[sm.idx[q]] = h ? 1 : 0;
        heads += h;
      }
    }
    atomicAdd(&sm.count, heads);
    __syncthreads();
    if (sm.overflow || sm.count <= max_points) break;
    leaf *= 2.0;
    __syncthreads();  // everyone has read count/overflow
    if (t == 0) sm.count = 0;
    __syncthreads();
  }
  const int m = sm.count;
  if (sm.overflow) {
    if (t == 0) {
      info[0] = m;
      info[1] = 1;
    }
    return;
  }
  // exclusive scan of the first-appearance flags in input order -> output position
  int32_t f[kBlockIpt];
#pragma unroll
  for (int u = 0; u < kBlockIpt; ++u) {
    const int i = t * kBlockIpt + u;
    f[u] = i < n ? sm.flag[i] : 0;
  }
  BlockScanI(sm.tmp.scan).ExclusiveSum(f, f);
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kBlockIpt; ++u) sm.flag[t * kBlockIpt + u] = f[u];
  __syncthreads();
  double lo[3] = {1e308, 1e308, 1e308}, hi[3] = {-1e308, -1e308, -1e308};
#pragma unroll
  for (int u = 0; u < kBlockIpt; ++u) {
    const int s = t * kBlockIpt + u;
    if (s >= n || !(s == 0 || sm.key[s] != sm.key[s - 1])) continue;
    double sx = 0.0, sy = 0.0, sz = 0.0;
    int c = 0;
    for (int q = s; q < n && (q == s || sm.key[q] == sm.key[s]); ++q) {
      const int32_t i = sm.idx[q];
      sx = sx + p[3 * i];
      sy = sy + p[3 * i + 1];
      sz = sz + p[3 * i + 2];
      ++c;
    }
    const double d = static_cast<double>(c);
    const double v[3] = {sx / d, sy / d, sz / d};
    const int o = sm.flag[sm.idx[s]];
    for (int a = 0; a < 3; ++a) {
      out[3 * o + a] = v[a];
      lo[a] = fmin(lo[a], v[a]);
      hi[a] = fmax(hi[a], v[a]);
    }
  }
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  if ((t & 31) == 0)
    for (int a = 0; a < 3; ++a) {
      sm.lo[a][t >> 5] = lo[a];
      sm.hi[a][t >> 5] = hi[a];
    }
  __syncthreads();
  if (t == 0) {
    for (int a = 0; a < 3; ++a) {
      double l = sm.lo[a][0], h = sm.hi[a][0];
      for (int w = 1; w < kBlockThreads / 32; ++w) {
        l = fmin(l, sm.lo[a][w]);
        h = fmax(h, sm.hi[a][w]);
      }
      bounds[a] = l;
      bounds[3 + a] = h;
    }
    info[0] = m;
    info[1] = 0;
  }
}

__global__ void k_bounds(const double* __restrict__ p, int n, double* __restrict__ b) {
  // single block: min/max per axis (exact)
  __shared__ double s_lo[3][256], s_hi[3][256];
  double lo[3] = {p[0], p[1], p[2]}, hi[3] = {p[0], p[1], p[2]};
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    for (int a = 0; a < 3; ++a) {
      lo[a] = fmin(lo[a], p[3 * i + a]);
      hi[a] = fmax(hi[a], p[3 * i + a]);
    }
  for (int a = 0; a < 3; ++a) {
    s_lo[a][threadIdx.x] = lo[a];
    s_hi[a][threadIdx.x] = hi[a];
  }
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int a = 0; a < 3; ++a) {
        s_lo[a][threadIdx.x] = fmin(s_lo[a][threadIdx.x], s_lo[a][threadIdx.x + o]);
        s_hi[a][threadIdx.x] = fmax(s_hi[a][threadIdx.x], s_hi[a][threadIdx.x + o]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int a = 0; a < 3; ++a) {
      b[a] = s_lo[a][0];
      b[3 + a] = s_hi[a][0];
    }
}

// prep.cpp sym_eig3 (cyclic Jacobi, ascending eigenvalues, eigenvectors in columns).
__device__ void sym_eig3_dev(const double a_in[9], double w[3], double v[9]) {
  double a[3][3], V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a[i][j] = a_in[i * 3 + j];
  for (int sweep = 0; sweep < 50; ++sweep) {
    const double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
    const double scale = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]);
    if (off == 0.0 || off <= 1e-300 || off < 1e-18 * scale) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (a[p][q] == 0.0) continue;
        const double th = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {
          const double x = a[k][p], y = a[k][q];
          a[k][p] = c * x - s * y;
          a[k][q] = s * x + c * y;
        }
        for (int k = 0; k < 3; ++k) {
          const double x = a[p][k], y = a[q][k];
          a[p][k] = c * x - s * y;
          a[q][k] = s * x + c * y;
        }
        for (int k = 0; k < 3; ++k) {
          const double x = V[k][p], y = V[k][q];
          V[k][p] = c * x - s * y;
          V[k][q] = s * x + c * y;
        }
      }
  }
  // std::sort of three indices by diagonal (insertion sort: stable)
  int ord[3] = {0, 1, 2};
  for (int i = 1; i < 3; ++i) {
    const int x = ord[i];
    int j = i;
    while (j > 0 && a[x][x] < a[ord[j - 1]][ord[j - 1]]) {
      ord[j] = ord[j - 1];
      --j;
    }
    ord[j] = x;
  }
  for (int c = 0; c < 3; ++c) {
    w[c] = a[ord[c]][ord[c]];
    for (int r = 0; r < 3; ++r) v[r * 3 + c] = V[r][ord[c]];
  }
}

struct KnnGrid {
  double org[3];
  double cell;
  int dims[3];
};

__device__ __forceinline__ void grid_cell(const KnnGrid& g, const double* p, int c[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int v = static_cast<int>(floor((p[a] - g.org[a]) / g.cell));
    c[a] = v < 0 ? 0 : (v > g.dims[a] - 1 ? g.dims[a] - 1 : v);
  }
}

constexpr int kKnnMax = 16;  // k + 1 <= kKnnMax (std::sort of <= 16 items is a stable insertion sort)

// (d2, rank, index) lexicographic order of the reference's stable top-K.
struct KnnKey {
  double d2;
  uint64_t rank;
  int32_t j;
};
__device__ __forceinline__ bool knn_less(const KnnKey& a, const KnnKey& b) {
  return a.d2 < b.d2 || (a.d2 == b.d2 && (a.rank < b.rank || (a.rank == b.rank && a.j < b.j)));
}

// Grid cell of every scan point (point_grid.cpp:45-49).
__global__ void k_scan_cells(const double* __restrict__ p, int n, KnnGrid g, int4* __restrict__ cell) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c[3];
  grid_cell(g, p + 3 * i, c);
  cell[i] = make_int4(c[0], c[1], c[2], 0);
}

// Covariance + structure record of point i from its k neighbours (one lane).
__device__ void cov_and_record(const double* __restrict__ p, int i, const int32_t* nbi, int m, double eps,
                               double noise_var, double* __restrict__ sigma, float4* __restrict__ rec,
                               int* __restrict__ not_structured, unsigned long long* __restrict__ l1max_bits) {
  double nb[kKnnMax][3];
  for (int s = 0; s < m; ++s)
    for (int a = 0; a < 3; ++a) nb[s][a] = p[3 * nbi[s] + a];
  // canonical order (x, y, z) — insertion sort
  for (int s = 1; s < m; ++s) {
    const double x0 = nb[s][0], x1 = nb[s][1], x2 = nb[s][2];
    int t = s;
    while (t > 0 && (x0 < nb[t - 1][0] || (x0 == nb[t - 1][0] && (x1 < nb[t - 1][1] ||
                                                                   (x1 == nb[t - 1][1] && x2 < nb[t - 1][2]))))) {
      nb[t][0] = nb[t - 1][0];
      nb[t][1] = nb[t - 1][1];
      nb[t][2] = nb[t - 1][2];
      --t;
    }
    nb[t][0] = x0;
    nb[t][1] = x1;
    nb[t][2] = x2;
  }
  double mean[3] = {0.0, 0.0, 0.0};
  for (int s = 0; s < m; ++s)
    for (int a = 0; a < 3; ++a) mean[a] = mean[a] + nb[s][a];
  const double cntd = static_cast<double>(m);
  for (int a = 0; a < 3; ++a) mean[a] = mean[a] / cntd;
  double cov[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int s = 0; s < m; ++s) {
    const double d[3] = {nb[s][0] - mean[0], nb[s][1] - mean[1], nb[s][2] - mean[2]};
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) cov[r * 3 + c] = cov[r * 3 + c] + d[r] * d[c];
  }
  for (int e = 0; e < 9; ++e) cov[e] = cov[e] / cntd;
  double w[3], v[9];
  sym_eig3_dev(cov, w, v);
  const double lmax = fmax(w[2], 1e-12);
  const double reg[3] = {eps * lmax, lmax, lmax};
  double sg[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      sg[r * 3 + c] = ((v[r * 3 + 0] * reg[0]) * v[c * 3 + 0] + (v[r * 3 + 1] * reg[1]) * v[c * 3 + 1]) +
                      (v[r * 3 + 2] * reg[2]) * v[c * 3 + 2];
  if (noise_var > 0.0)
    for (int d = 0; d < 3; ++d) sg[4 * d] = sg[4 * d] + noise_var;
  for (int e = 0; e < 9; ++e) sigma[9 * i + e] = sg[e];
  // engine.cu structure_ab on the final covariance -> fast-path record
  sym_eig3_dev(sg, w, v);
  double mx = 0.0;
  for (int e = 0; e < 9; ++e) mx = fmax(mx, fabs(sg[e]));
  const double a = 0.5 * (w[1] + w[2]), sv = w[0];
  const double ax[3] = {v[0], v[3], v[6]};
  double err = 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      const double recv = (r == c ? a : 0.0) - (a - sv) * ax[r] * ax[c];
      err = fmax(err, fabs(recv - sg[r * 3 + c]));
    }
  if (!(err <= 1e-10 * mx) || !(sv >= 0.0) || !(a > 0.0)) atomicExch(not_structured, 1);
  const double* mu = p + 3 * i;
  rec[2 * i] = make_float4(static_cast<float>(mu[0]), static_cast<float>(mu[1]), static_cast<float>(mu[2]),
                           static_cast<float>(a - sv));
  rec[2 * i + 1] = make_float4(static_cast<float>(ax[0]), static_cast<float>(ax[1]), static_cast<float>(ax[2]),
                               static_cast<float>(sv));
  const double l1 = (fabs(mu[0]) + fabs(mu[1])) + fabs(mu[2]);
  atomicMax(l1max_bits, static_cast<unsigned long long>(__double_as_longlong(l1)));  // l1 >= 0: bit order = value order
}

// gaussian_cloud.cpp:36-90 + filter.cpp:95-98: warp per query point. Lanes
// stride over the candidates keeping a private stable top-K; the warp merges
// the 32 sorted lists by K rounds of a lexicographic warp minimum.
__global__ void __launch_bounds__(128) k_scan_knn_cov(const double* __restrict__ p, const int4* __restrict__ cell,
                                                     int n, int k, double eps, double noise_var,
                                                     double* __restrict__ sigma, float4* __restrict__ rec,
                                                     int* __restrict__ not_structured,
                                                     unsigned long long* __restrict__ l1max_bits) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;  // warp-uniform
  const int K = k + 1;
  const double q[3] = {p[3 * i], p[3 * i + 1], p[3 * i + 2]};
  const int4 c0 = cell[i];
  KnnKey best[kKnnMax];
  int cnt = 0;
  for (int j = lane; j < n; j += 32) {
    const double dx = p[3 * j] - q[0], dy = p[3 * j + 1] - q[1], dz = p[3 * j + 2] - q[2];
    KnnKey e;
    e.d2 = (dx * dx + dy * dy) + dz * dz;
    const int4 cj = cell[j];
    const int ring = max(abs(cj.x - c0.x), max(abs(cj.y - c0.y), abs(cj.z - c0.z)));
    e.rank = (static_cast<uint64_t>(ring) << 48) | (static_cast<uint64_t>(cj.z) << 32) |
             (static_cast<uint64_t>(cj.y) << 16) | static_cast<uint64_t>(cj.x);
    e.j = j;
    int pos;
    if (cnt < K) {
      pos = cnt++;
    } else {
      if (!knn_less(e, best[K - 1])) continue;
      pos = K - 1;
    }
    while (pos > 0 && knn_less(e, best[pos - 1])) {
      best[pos] = best[pos - 1];
      --pos;
    }
    best[pos] = e;
  }
  // merge: K rounds of the warp-wide minimum of the list heads
  int head = 0;
  int32_t nbi[kKnnMax];
  int m = 0;
  for (int r = 0; r < K; ++r) {
    KnnKey h;
    h.d2 = __longlong_as_double(0x7ff0000000000000ll);
    h.rank = ~0ull;
    h.j = 0x7fffffff;
    if (head < cnt) h = best[head];
    KnnKey mn = h;
    for (int o = 16; o > 0; o >>= 1) {
      KnnKey other;
      other.d2 = __shfl_xor_sync(FULL, mn.d2, o);
      other.rank = __shfl_xor_sync(FULL, mn.rank, o);
      other.j = __shfl_xor_sync(FULL, mn.j, o);
      if (knn_less(other, mn)) mn = other;
    }
    if (head < cnt && h.j == mn.j) ++head;  // the owning lane pops its head (indices are unique)
    if (mn.j != i && m < k) nbi[m++] = mn.j;  // the point itself is skipped (gaussian_cloud.cpp:55-59)
  }
  if (lane == 0) cov_and_record(p, i, nbi, m, eps, noise_var, sigma, rec, not_structured, l1max_bits);
}

// engine.cu structure_ab on the device: plane-model parameters of a scan
// covariance + the fast-path record; flags non-structured covariances.
__global__ void k_scan_records(const double* __restrict__ mu, const double* __restrict__ sigma, int n,
                               float4* __restrict__ rec, int* __restrict__ not_structured, double* __restrict__ l1) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const double* sig = sigma + 9 * q;
  double w[3], v[9];
  sym_eig3_dev(sig, w, v);
  double mx = 0.0;
  for (int e = 0; e < 9; ++e) mx = fmax(mx, fabs(sig[e]));
  const double a = 0.5 * (w[1] + w[2]), sv = w[0];
  const double ax[3] = {v[0], v[3], v[6]};
  double err = 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      const double recv = (r == c ? a : 0.0) - (a - sv) * ax[r] * ax[c];
      err = fmax(err, fabs(recv - sig[r * 3 + c]));
    }
  if (!(err <= 1e-10 * mx) || !(sv >= 0.0) || !(a > 0.0)) atomicExch(not_structured, 1);
  rec[2 * q] = make_float4(static_cast<float>(mu[3 * q]), static_cast<float>(mu[3 * q + 1]),
                           static_cast<float>(mu[3 * q + 2]), static_cast<float>(a - sv));
  rec[2 * q + 1] = make_float4(static_cast<float>(ax[0]), static_cast<float>(ax[1]), static_cast<float>(ax[2]),
                               static_cast<float>(sv));
  l1[q] = (fabs(mu[3 * q]) + fabs(mu[3 * q + 1])) + fabs(mu[3 * q + 2]);
}

__global__ void k_gather_stride(const double* __restrict__ mu, const double* __restrict__ sigma, int n_out,
                                int stride, double* __restrict__ mu_out, double* __restrict__ sigma_out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n_out) return;
  for (int a = 0; a < 3; ++a) mu_out[3 * q + a] = mu[3 * (q * stride) + a];
  for (int a = 0; a < 9; ++a) sigma_out[9 * q + a] = sigma[9 * (q * stride) + a];
}

#define SP_CK(x)                        \
  do {                                  \
    const cudaError_t e_ = (x);         \
    if (e_ != cudaSuccess) return e_;   \
  } while (0)

template <class T>
cudaError_t grow(T*& p, size_t& cap, size_t n, cudaStream_t st) {
  if (n <= cap && p) return cudaSuccess;
  if (p) SP_CK(cudaFreeAsync(p, st));
  p = nullptr;
  cap = std::max<size_t>(n, 1);
  return cudaMallocAsync(reinterpret_cast<void**>(&p), cap * sizeof(T), st);
}

}  // namespace

// Scratch reused across frames.
struct ScanPrepWork {
  uint64_t *key = nullptr, *skey = nullptr;
  int32_t *iota = nullptr, *sidx = nullptr, *head = nullptr, *first = nullptr, *pos = nullptr;
  int* flag = nullptr;  // [0] overflow / count, [1] not structured, [2] not structured (kNN path)
  int4* cells = nullptr;
  unsigned long long* l1bits = nullptr;
  size_t c_cells = 0, c_l1bits = 0;
  double* bounds = nullptr;
  void* temp = nullptr;
  size_t cap = 0, temp_cap = 0, c_key = 0, c_skey = 0, c_iota = 0, c_sidx = 0, c_head = 0, c_first = 0, c_pos = 0;
  size_t c_flag = 0, c_bounds = 0;
};

ScanPrepWork* scan_prep_create() { return new ScanPrepWork(); }
void scan_prep_destroy(ScanPrepWork* w) {
  if (!w) return;
  for (void* p : {static_cast<void*>(w->key), static_cast<void*>(w->skey), static_cast<void*>(w->iota),
                  static_cast<void*>(w->sidx), static_cast<void*>(w->head), static_cast<void*>(w->first),
                  static_cast<void*>(w->pos), static_cast<void*>(w->flag), static_cast<void*>(w->bounds),
                  static_cast<void*>(w->cells), static_cast<void*>(w->l1bits), w->temp})
    if (p) cudaFree(p);
  delete w;
}

// voxel_downsample(points, leaf) into d_out (capacity n points); returns the
// voxel count through *n_out (host, synchronous). *overflow: a voxel key does
// not fit 21 bits per axis (the caller falls back to the host path).
cudaError_t scan_voxel_downsample(ScanPrepWork* w, const double* d_pts, int n, double leaf, double* d_out,
                                  int* n_out, bool* overflow, cudaStream_t st) {
  const size_t un = static_cast<size_t>(std::max(n, 1));
  SP_CK(grow(w->key, w->c_key, un, st));
  SP_CK(grow(w->skey, w->c_skey, un, st));
  SP_CK(grow(w->iota, w->c_iota, un, st));
  SP_CK(grow(w->sidx, w->c_sidx, un, st));
  SP_CK(grow(w->head, w->c_head, un, st));
  SP_CK(grow(w->first, w->c_first, un, st));
  SP_CK(grow(w->pos, w->c_pos, un, st));
  SP_CK(grow(w->flag, w->c_flag, 2, st));
  size_t sb = 0, cb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sb, w->key, w->skey, w->iota, w->sidx, n, 0, 63);
  cub::DeviceScan::ExclusiveSum(nullptr, cb, w->first, w->pos, n);
  if (std::max(sb, cb) > w->temp_cap) {
    if (w->temp) SP_CK(cudaFreeAsync(w->temp, st));
    w->temp_cap = std::max(sb, cb);
    SP_CK(cudaMallocAsync(&w->temp, w->temp_cap, st));
  }
  SP_CK(cudaMemsetAsync(w->flag, 0, 2 * sizeof(int), st));
  count_launch();
  k_voxel_keys<<<blocks_for(n, 256), 256, 0, st>>>(d_pts, n, leaf, w->key, w->iota, w->flag);
  size_t tb = w->temp_cap;
  SP_CK(cub::DeviceRadixSort::SortPairs(w->temp, tb, w->key, w->skey, w->iota, w->sidx, n, 0, 63, st));
  count_launch();
  k_voxel_heads<<<blocks_for(n, 256), 256, 0, st>>>(w->skey, w->sidx, n, w->head, w->first);
  tb = w->temp_cap;
  SP_CK(cub::DeviceScan::ExclusiveSum(w->temp, tb, w->first, w->pos, n, st));
  count_launch();
  k_voxel_centroids<<<blocks_for(n, 128), 128, 0, st>>>(d_pts, w->skey, w->sidx, w->head, n, w->pos, d_out);
  int last[2], flags[2];
  SP_CK(cudaMemcpyAsync(&last[0], w->pos + (n - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
  SP_CK(cudaMemcpyAsync(&last[1], w->first + (n - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
  SP_CK(cudaMemcpyAsync(flags, w->flag, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  SP_CK(cudaStreamSynchronize(st));
  *n_out = last[0] + last[1];
  *overflow = flags[0] != 0;
  return cudaGetLastError();
}

// Bounds of d_pts (host, synchronous).
cudaError_t scan_bounds(ScanPrepWork* w, const double* d_pts, int n, double b[6], cudaStream_t st) {
  SP_CK(grow(w->bounds, w->c_bounds, 6, st));
  count_launch();
  k_bounds<<<1, 256, 0, st>>>(d_pts, n, w->bounds);
  SP_CK(cudaMemcpyAsync(b, w->bounds, 6 * sizeof(double), cudaMemcpyDeviceToHost, st));
  return cudaStreamSynchronize(st);
}

cudaError_t scan_records(ScanPrepWork* w, const double* d_mu, const double* d_sigma, int n, float4* d_rec,
                         double* d_l1, bool* structured, double* l1max, cudaStream_t st) {
  SP_CK(grow(w->flag, w->c_flag, 2, st));
  SP_CK(cudaMemsetAsync(w->flag + 1, 0, sizeof(int), st));
  count_launch();
  k_scan_records<<<blocks_for(n, 128), 128, 0, st>>>(d_mu, d_sigma, n, d_rec, w->flag + 1, d_l1);
  int ns = 0;
  SP_CK(cudaMemcpyAsync(&ns, w->flag + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  std::vector<double> l1(static_cast<size_t>(n));
  SP_CK(cudaMemcpyAsync(l1.data(), d_l1, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  SP_CK(cudaStreamSynchronize(st));
  *structured = ns == 0;
  double m = 0.0;
  for (double v : l1) m = std::max(m, v);
  *l1max = m;
  return cudaSuccess;
}

cudaError_t scan_downsample_block(ScanPrepWork* w, const double* d_pts, int n, double leaf0, int max_points,
                                  double* d_out, int* n_out, bool* overflow, double bounds[6], cudaStream_t st) {
  if (n > kBlockItems) return cudaErrorInvalidValue;
  SP_CK(grow(w->flag, w->c_flag, 4, st));
  SP_CK(grow(w->bounds, w->c_bounds, 6, st));
  const size_t smem = sizeof(BlockSmem);
  SP_CK(cudaFuncSetAttribute(k_downsample_block, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  count_launch();
  k_downsample_block<<<1, kBlockThreads, smem, st>>>(d_pts, n, leaf0, max_points, d_out, w->flag, w->bounds);
  SP_CK(cudaGetLastError());
  int info[2];
  SP_CK(cudaMemcpyAsync(info, w->flag, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  SP_CK(cudaMemcpyAsync(bounds, w->bounds, 6 * sizeof(double), cudaMemcpyDeviceToHost, st));
  SP_CK(cudaStreamSynchronize(st));
  *n_out = info[0];
  *overflow = info[1] != 0;
  return cudaSuccess;
}

cudaError_t scan_knn_cov_records(ScanPrepWork* w, const double* d_pts, int n, int k, double eps, double noise_var,
                                 const double grid_org[3], double grid_cell, const int grid_dims[3],
                                 double* d_sigma, float4* d_rec, bool* structured, double* l1max, cudaStream_t st) {
  if (k + 1 > kKnnMax) return cudaErrorInvalidValue;
  KnnGrid g;
  for (int a = 0; a < 3; ++a) {
    g.org[a] = grid_org[a];
    g.dims[a] = grid_dims[a];
  }
  g.cell = grid_cell;
  SP_CK(grow(w->cells, w->c_cells, static_cast<size_t>(n), st));
  SP_CK(grow(w->flag, w->c_flag, 4, st));
  SP_CK(cudaMemsetAsync(w->flag + 2, 0, 2 * sizeof(int), st));  // [2] not structured, [3] unused
  SP_CK(grow(w->l1bits, w->c_l1bits, 1, st));
  SP_CK(cudaMemsetAsync(w->l1bits, 0, sizeof(unsigned long long), st));
  count_launch(2);
  k_scan_cells<<<blocks_for(n, 128), 128, 0, st>>>(d_pts, n, g, w->cells);
  k_scan_knn_cov<<<blocks_for(static_cast<int64_t>(n) * 32, 128), 128, 0, st>>>(
      d_pts, w->cells, n, k, eps, noise_var, d_sigma, d_rec, w->flag + 2, w->l1bits);
  SP_CK(cudaGetLastError());
  int ns = 0;
  unsigned long long bits = 0;
  SP_CK(cudaMemcpyAsync(&ns, w->flag + 2, sizeof(int), cudaMemcpyDeviceToHost, st));
  SP_CK(cudaMemcpyAsync(&bits, w->l1bits, sizeof(bits), cudaMemcpyDeviceToHost, st));
  SP_CK(cudaStreamSynchronize(st));
  *structured = ns == 0;
  std::memcpy(l1max, &bits, sizeof(double));
  return cudaSuccess;
}

cudaError_t scan_gather_stride(const double* d_mu, const double* d_sigma, int n_out, int stride, double* mu_out,
                               double* sigma_out, cudaStream_t st) {
  count_launch();
  k_gather_stride<<<blocks_for(n_out, 128), 128, 0, st>>>(d_mu, d_sigma, n_out, stride, mu_out, sigma_out);
  return cudaGetLastError();
}

}  // namespace smcl
