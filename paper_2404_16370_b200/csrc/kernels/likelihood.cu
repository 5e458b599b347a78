// K1 / K2: per-particle GICP likelihood with Gauss-Newton accumulation
// (reference gicp.cpp:11-45 evaluate, 87-107 evaluate_all, 109-137
// evaluate_likelihoods) and the damped 6x6 solve (gicp.cpp:47-75).
//
// Two formulations:
//  * exact  — one thread per particle, fp64, the reference's world-frame
//             expressions in the oracle's evaluation order with unfused
//             multiplies/adds: bit-identical to the CPU oracle.
//  * fast   — one warp per particle, lanes stride over scan points. Phase A
//             transforms points in fp64 (exact voxel decision), gathers the
//             32-byte denormalised cell record and compacts matched points into
//             a per-warp shared-memory queue; phase B runs the body-frame,
//             structured-covariance (Woodbury) algebra in fp32 on full warps;
//             a shuffle reduction produces the 28 accumulators per particle.
// Both write the same per-particle system record; a thread-per-particle fp64
// kernel then does the LLT solve + gating exactly as the oracle.
#include <cuda_runtime.h>

#include <algorithm>

#include "../engine.cuh"
#include "../kernels.cuh"

namespace smcl {

namespace {

// ---------------------------------------------------------------- exact helpers
struct M3d {
  double m[9];
};

__device__ __forceinline__ void mul33(const double* a, const double* b, double* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r[i * 3 + j] = xadd(xadd(xmul(a[i * 3 + 0], b[0 * 3 + j]), xmul(a[i * 3 + 1], b[1 * 3 + j])),
                          xmul(a[i * 3 + 2], b[2 * 3 + j]));
}
// a * b^T
__device__ __forceinline__ void mul33t(const double* a, const double* b, double* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r[i * 3 + j] = xadd(xadd(xmul(a[i * 3 + 0], b[j * 3 + 0]), xmul(a[i * 3 + 1], b[j * 3 + 1])),
                          xmul(a[i * 3 + 2], b[j * 3 + 2]));
}
// a^T * b
__device__ __forceinline__ void mult33(const double* a, const double* b, double* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r[i * 3 + j] = xadd(xadd(xmul(a[0 * 3 + i], b[0 * 3 + j]), xmul(a[1 * 3 + i], b[1 * 3 + j])),
                          xmul(a[2 * 3 + i], b[2 * 3 + j]));
}
__device__ __forceinline__ double cof3(const double* m, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return xsub(xmul(m[i1 * 3 + j1], m[i2 * 3 + j2]), xmul(m[i1 * 3 + j2], m[i2 * 3 + j1]));
}
// Eigen 3x3 inverse (cofactors of column 0, invdet = 1/det).
__device__ __forceinline__ void inverse3(const double* m, double* r) {
  const double c00 = cof3(m, 0, 0), c10 = cof3(m, 1, 0), c20 = cof3(m, 2, 0);
  const double det = xadd(xadd(xmul(c00, m[0]), xmul(c10, m[3])), xmul(c20, m[6]));
  const double invdet = 1.0 / det;
  r[0] = xmul(c00, invdet);
  r[1] = xmul(c10, invdet);
  r[2] = xmul(c20, invdet);
  r[3] = xmul(cof3(m, 0, 1), invdet);
  r[4] = xmul(cof3(m, 1, 1), invdet);
  r[5] = xmul(cof3(m, 2, 1), invdet);
  r[6] = xmul(cof3(m, 0, 2), invdet);
  r[7] = xmul(cof3(m, 1, 2), invdet);
  r[8] = xmul(cof3(m, 2, 2), invdet);
}

// nnf.hpp:24-35 lookup, exact: floor((p - o) * inv) per axis, bounds check.
__device__ __forceinline__ int64_t nnf_cell(const NnfGeom& g, const double p[3], double frac[3]) {
  int64_t c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double x = xmul(xsub(p[a], g.origin[a]), g.inv_res);
    const double f = floor(x);
    if (!(f >= 0.0 && f < static_cast<double>(g.dims[a]))) return -1;
    c[a] = static_cast<int64_t>(f);
    frac[a] = xsub(x, f);
  }
  return (c[2] * g.dims[1] + c[1]) * g.dims[0] + c[0];
}

__device__ __forceinline__ void transform_x(const Pose& P, const double mu[3], double p[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
    p[i] = xadd(xadd(xadd(xmul(P.R[i * 3 + 0], mu[0]), xmul(P.R[i * 3 + 1], mu[1])), xmul(P.R[i * 3 + 2], mu[2])),
                P.t[i]);
}

// ---------------------------------------------------------------- exact kernel
template <bool GN>
__global__ void __launch_bounds__(128) k_gicp_exact(const Pose* __restrict__ poses, int64_t n, ScanView scan,
                                                    MapExact map, double* __restrict__ sys,
                                                    double* __restrict__ raw_ll, int32_t* __restrict__ nm_out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Pose P = poses[i];
  double htl[9], htr[9], hbr[9], b[6];
#pragma unroll
  for (int q = 0; q < 9; ++q) htl[q] = htr[q] = hbr[q] = 0.0;
#pragma unroll
  for (int q = 0; q < 6; ++q) b[q] = 0.0;
  double ll = 0.0;
  int nmatch = 0;
  for (int k = 0; k < scan.n; ++k) {
    const double mu[3] = {__ldg(scan.mu + 3 * k), __ldg(scan.mu + 3 * k + 1), __ldg(scan.mu + 3 * k + 2)};
    double p[3], frac[3];
    transform_x(P, mu, p);
    const int64_t cell = nnf_cell(map.g, p, frac);
    if (cell < 0) continue;
    const int32_t m = __ldg(map.cells + cell);
    if (m < 0) continue;
    const double e[3] = {xsub(__ldg(map.mu + 3 * m), p[0]), xsub(__ldg(map.mu + 3 * m + 1), p[1]),
                         xsub(__ldg(map.mu + 3 * m + 2), p[2])};
    double ss[9], sm[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      ss[q] = __ldg(scan.sigma + 9 * k + q);
      sm[q] = __ldg(map.sigma + 9 * static_cast<int64_t>(m) + q);
    }
    double rs[9], t[9], cm[9], om[9];
    mul33(P.R, ss, rs);
    mul33t(rs, P.R, t);
#pragma unroll
    for (int q = 0; q < 9; ++q) cm[q] = xadd(sm[q], t[q]);
    inverse3(cm, om);
    double oe[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) oe[r] = xadd(xadd(xmul(om[r * 3 + 0], e[0]), xmul(om[r * 3 + 1], e[1])), xmul(om[r * 3 + 2], e[2]));
    if (GN) {
      const double sk[9] = {0.0, -mu[2], mu[1], mu[2], 0.0, -mu[0], -mu[1], mu[0], 0.0};
      double a[9], oa[9], orr[9], t1[9], t2[9], t3[9];
      mul33(P.R, sk, a);
      mul33(om, a, oa);
      mul33(om, P.R, orr);
      mult33(a, oa, t1);
      mult33(a, orr, t2);
      mult33(P.R, orr, t3);
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        htl[q] = xadd(htl[q], t1[q]);
        htr[q] = xsub(htr[q], t2[q]);
        hbr[q] = xadd(hbr[q], t3[q]);
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double bt = xadd(xadd(xmul(a[0 * 3 + c], oe[0]), xmul(a[1 * 3 + c], oe[1])), xmul(a[2 * 3 + c], oe[2]));
        const double bb = xadd(xadd(xmul(P.R[0 * 3 + c], oe[0]), xmul(P.R[1 * 3 + c], oe[1])), xmul(P.R[2 * 3 + c], oe[2]));
        b[c] = xadd(b[c], bt);
        b[c + 3] = xsub(b[c + 3], bb);
      }
    }
    ll = xsub(ll, xadd(xadd(xmul(e[0], oe[0]), xmul(e[1], oe[1])), xmul(e[2], oe[2])));
    ++nmatch;
  }
  if (GN) {
    double* out = sys + i * kSysStride;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        out[r * 6 + c] = htl[r * 3 + c];
        out[r * 6 + c + 3] = htr[r * 3 + c];
        out[(r + 3) * 6 + c + 3] = hbr[r * 3 + c];
        out[(r + 3) * 6 + c] = htr[c * 3 + r];
      }
#pragma unroll
    for (int q = 0; q < 6; ++q) out[36 + q] = b[q];
  }
  raw_ll[i] = nmatch == 0 ? -1e30 : ll;
  nm_out[i] = nmatch;
}

// ---------------------------------------------------------------- solve
// Eigen LLT (lower, unblocked) + two triangular solves, oracle order.
// Packed lower triangle of a symmetric 6x6: element (i, j), j <= i.
__host__ __device__ constexpr int lp6(int i, int j) { return i * (i + 1) / 2 + j; }

// LLT solve on the packed lower triangle, the oracle's operation order
// (every entry it reads is on or below the diagonal). Register-resident:
// fully unrolled, constant indices. (Pivot reciprocals instead of the 27
// IEEE divisions would save ~25 us per step but break the bitwise equality
// with the oracle's solve that the parity tests pin.)
__device__ __forceinline__ bool llt6_solve_lower(const double (&A)[21], const double (&b)[6], double (&x)[6]) {
  double L[21];
#pragma unroll
  for (int q = 0; q < 21; ++q) L[q] = A[q];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    double xk = L[lp6(k, k)];
    if (k > 0) {
      double sq = 0.0;
#pragma unroll
      for (int j = 0; j < k; ++j) sq = xadd(sq, xmul(L[lp6(k, j)], L[lp6(k, j)]));
      xk = xsub(xk, sq);
    }
    if (xk <= 0.0) return false;
    xk = sqrt(xk);
    L[lp6(k, k)] = xk;
#pragma unroll
    for (int i = k + 1; i < 6; ++i) {
      if (k > 0) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < k; ++j) s = xadd(s, xmul(L[lp6(i, j)], L[lp6(k, j)]));
        L[lp6(i, k)] = xsub(L[lp6(i, k)], s);
      }
      L[lp6(i, k)] = L[lp6(i, k)] / xk;
    }
  }
  double y[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < i; ++j) s = xadd(s, xmul(L[lp6(i, j)], y[j]));
    y[i] = xsub(b[i], s) / L[lp6(i, i)];
  }
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    double s = 0.0;
#pragma unroll
    for (int j = i + 1; j < 6; ++j) s = xadd(s, xmul(L[lp6(j, i)], x[j]));
    x[i] = xsub(y[i], s) / L[lp6(i, i)];
  }
  return true;
}

// gicp.cpp:47-75 on the packed lower triangle of H.
__device__ __forceinline__ void solve_step_lower(const double (&H)[21], const double (&b)[6], double lambda,
                                                 double omax, double vmax, double (&step)[6]) {
#pragma unroll
  for (int c = 0; c < 6; ++c) step[c] = 0.0;
  bool zero = true;
#pragma unroll
  for (int c = 0; c < 6; ++c) zero = zero && (b[c] == 0.0);
  if (zero) return;
  double lm = lambda;
  bool solved = false;
#pragma unroll 1
  for (int attempt = 0; attempt < 4; ++attempt) {
    double D[21], x[6];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j) D[lp6(i, j)] = (i == j) ? xadd(H[lp6(i, j)], lm) : xadd(H[lp6(i, j)], 0.0);
    if (llt6_solve_lower(D, b, x)) {
      bool finite = true;
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        step[c] = -x[c];
        finite = finite && isfinite(step[c]);
      }
      if (finite) {
        solved = true;
        break;
      }
#pragma unroll
      for (int c = 0; c < 6; ++c) step[c] = 0.0;
    }
    lm = xmul(lm, 2.0);
  }
  if (!solved) {
#pragma unroll
    for (int c = 0; c < 6; ++c) step[c] = 0.0;
    return;
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    step[c] = fmin(fmax(step[c], -omax), omax);
    step[c + 3] = fmin(fmax(step[c + 3], -vmax), vmax);
  }
}

// Full row-major H (the batch primitive of the parity tests): its lower triangle.
__device__ __forceinline__ void solve_step_dev(const double* H, const double* b, double lambda, double omax,
                                               double vmax, double* step) {
  double Hl[21], bb[6], st[6];
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) Hl[lp6(i, j)] = H[i * 6 + j];
#pragma unroll
  for (int c = 0; c < 6; ++c) bb[c] = b[c];
  solve_step_lower(Hl, bb, lambda, omax, vmax, st);
#pragma unroll
  for (int c = 0; c < 6; ++c) step[c] = st[c];
}

__device__ __forceinline__ double gated(const GicpParamsDev& p, double raw, int nm) {
  if (nm < p.min_matched) return -1e30;
  return xsub(raw, xmul(p.miss_cost, xsub(static_cast<double>(p.scan_size), static_cast<double>(nm))));
}

// F32: the fast kernel's fp32 record (kSysF lanes), widened to fp64 as the
// kernel's own conversion would; else the exact kernel's fp64 record. Only
// the lower triangle of H is read (LLT, trace).
// nm_sum (optional): += sum of n_matched (the step profile's matched
// particle-points of the pass), one block-reduced atomic per block (a
// same-address atomic per warp had serialised ~32 k atomics at 1M).
template <bool F32>
__global__ void k_solve(const double* __restrict__ sys, const float* __restrict__ sysf,
                        const double* __restrict__ raw_ll, const int32_t* __restrict__ nm, int64_t n,
                        GicpParamsDev p, double* __restrict__ steps, double* __restrict__ ll,
                        unsigned long long* __restrict__ nm_sum) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int m = i < n ? nm[i] : 0;
  if (nm_sum) {  // block-uniform branch; launched with 128 threads
    __shared__ unsigned s_w[4];
    const unsigned w = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(m));
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = w;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned long long t = static_cast<unsigned long long>(s_w[0]) + s_w[1] + s_w[2] + s_w[3];
      if (t) atomicAdd(nm_sum, t);
    }
  }
  if (i >= n) return;
  ll[i] = gated(p, raw_ll[i], m);
  double step[6] = {0, 0, 0, 0, 0, 0};
  if (m != 0) {
    double Hl[21], bb[6];  // packed lower triangle of H, b
    if (F32) {
      constexpr int off[27] = SMCL_FAST_SYS_OFF;  // row-major H (lower) then b, in record order
      const float4* r = reinterpret_cast<const float4*>(sysf + i * kSysF);
      float v[28];
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        const float4 a = __ldg(r + q);
        v[4 * q] = a.x, v[4 * q + 1] = a.y, v[4 * q + 2] = a.z, v[4 * q + 3] = a.w;
      }
#pragma unroll
      for (int q = 0; q < 27; ++q) {
        if (off[q] < 36)
          Hl[lp6(off[q] / 6, off[q] % 6)] = static_cast<double>(v[q]);
        else
          bb[off[q] - 36] = static_cast<double>(v[q]);
      }
    } else {
      const double* s = sys + i * kSysStride;
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = 0; c <= r; ++c) Hl[lp6(r, c)] = s[r * 6 + c];
#pragma unroll
      for (int c = 0; c < 6; ++c) bb[c] = s[36 + c];
    }
    double tr = 0.0;
#pragma unroll
    for (int q = 0; q < 6; ++q) tr = xadd(tr, Hl[lp6(q, q)]);
    const double lambda = xmul(p.damping_scale, tr) / 6.0;
    solve_step_lower(Hl, bb, lambda, p.omega_max, p.v_max, step);
  }
#pragma unroll
  for (int q = 0; q < 6; ++q) steps[6 * i + q] = step[q];
}

// counts (optional): += (particles with a matched observation, sum of
// n_matched), the Bayes update's match counts (posterior.cpp:26-58), folded
// into the gate's sweep (one block reduction + two atomics per block).
__global__ void __launch_bounds__(256) k_gate(const double* __restrict__ raw_ll, const int32_t* __restrict__ nm,
                                              int64_t n, GicpParamsDev p, double* __restrict__ ll,
                                              unsigned long long* __restrict__ counts) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned a = 0, b = 0;
  if (i < n) {
    const int m = nm[i];
    const double g = gated(p, raw_ll[i], m);
    ll[i] = g;
    a = g > -1e30 ? 1u : 0u;
    b = static_cast<unsigned>(m);
  }
  if (!counts) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  __shared__ unsigned sa[8], sb[8];
  if ((threadIdx.x & 31) == 0) {
    sa[threadIdx.x >> 5] = a;
    sb[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long ta = 0, tb = 0;
    for (int w = 0; w < 8; ++w) {
      ta += sa[w];
      tb += sb[w];
    }
    if (ta) atomicAdd(counts, ta);
    if (tb) atomicAdd(counts + 1, tb);
  }
}

__global__ void k_solve_batch(const double* __restrict__ H, const double* __restrict__ b,
                              const double* __restrict__ lam, int64_t n, double omax, double vmax,
                              double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double h[36], bb[6], st[6];
  for (int q = 0; q < 36; ++q) h[q] = H[36 * i + q];
  for (int q = 0; q < 6; ++q) bb[q] = b[6 * i + q];
  solve_step_dev(h, bb, lam[i], omax, vmax, st);
  for (int q = 0; q < 6; ++q) out[6 * i + q] = st[q];
}

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

void launch_gicp_exact(bool gn, const Pose* poses, int64_t n, const ScanView& scan, const MapExact& map, double* sys,
                       double* raw_ll, int32_t* nm, cudaStream_t st) {
  count_launch();
  if (n <= 0) return;
  if (gn)
    k_gicp_exact<true><<<blocks_for(n, 128), 128, 0, st>>>(poses, n, scan, map, sys, raw_ll, nm);
  else
    k_gicp_exact<false><<<blocks_for(n, 128), 128, 0, st>>>(poses, n, scan, map, sys, raw_ll, nm);
}

void launch_solve(const double* sys, const float* sysf, const double* raw_ll, const int32_t* nm, int64_t n,
                  const GicpParamsDev& p, double* steps, double* ll, cudaStream_t st, unsigned long long* nm_sum) {
  count_launch();
  if (n <= 0) return;
  if (sysf)
    k_solve<true><<<blocks_for(n, 128), 128, 0, st>>>(nullptr, sysf, raw_ll, nm, n, p, steps, ll, nm_sum);
  else
    k_solve<false><<<blocks_for(n, 128), 128, 0, st>>>(sys, nullptr, raw_ll, nm, n, p, steps, ll, nm_sum);
}

void launch_gate_ll(const double* raw_ll, const int32_t* nm, int64_t n, const GicpParamsDev& p, double* ll,
                    cudaStream_t st, unsigned long long* counts) {
  count_launch();
  if (n <= 0) return;
  k_gate<<<blocks_for(n, 256), 256, 0, st>>>(raw_ll, nm, n, p, ll, counts);
}

void launch_solve_batch(const double* H, const double* b, const double* lam, int64_t n, double omax, double vmax,
                        double* out, cudaStream_t st) {
  count_launch();
  if (n <= 0) return;
  k_solve_batch<<<blocks_for(n, 128), 128, 0, st>>>(H, b, lam, n, omax, vmax, out);
}

}  // namespace smcl
