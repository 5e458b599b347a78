#include <cuda_runtime.h>
#include "../paper_2404_16370_b200/csrc/engine.cuh"
#include "../paper_2404_16370_b200/csrc/kernels.cuh"
namespace smcl {
// Float kernel value of a pair as the reference caches it
// (neighbor_graph.hpp:84-86, neighbor_search.cpp:161-166): 0 if the
// translation bound underflows, else (float)exp(-q) with q from the SE3 log.
//
// Fast evaluation. With Rrel = Ra^T Rb,
// vee = (Rrel - Rrel^T)^vee, s = |vee|/2, c = (tr Rrel - 1)/2, r = hypot(s, c),
// theta = atan2(s, c), the reference's log (se3.hpp:103-149) gives
// |w| = theta*r, and V^-1 acts as the identity along w and as a scaled
// rotation with |V^-1 x|^2 = |x|^2 (th/2)^2 / sin^2(th/2) across it, so
//   q = sr th^2 + st ( (u.w^)^2 + (|u|^2 - (u.w^)^2) th^2 / (4 sin^2(th/2)) ),
// u = Ra^T (tb - ta), th = theta*r. No sin/cos calls: sin/cos of th follow
// from s/r, c/r and the tiny th - theta. q agrees with the reference's to
// ~1e-14 relative; the float is returned only if exp(-q)*(1 -+ 4e-12) round
// to the same float, otherwise *ok = false and kval_of takes the reference-order log.
__device__ __forceinline__ float kval_fast(const Pose& a, const Pose& b, double sr, double st, bool* ok) {
  double m[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      m[i * 3 + j] = fma(a.R[0 * 3 + i], b.R[0 * 3 + j], fma(a.R[1 * 3 + i], b.R[1 * 3 + j], a.R[2 * 3 + i] * b.R[2 * 3 + j]));
  const double d0 = b.t[0] - a.t[0], d1 = b.t[1] - a.t[1], d2 = b.t[2] - a.t[2];
  double u[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) u[i] = fma(a.R[0 * 3 + i], d0, fma(a.R[1 * 3 + i], d1, a.R[2 * 3 + i] * d2));
  const double v0 = m[7] - m[5], v1 = m[2] - m[6], v2 = m[3] - m[1];
  const double vv = fma(v0, v0, fma(v1, v1, v2 * v2));  // |vee|^2 = 4 s^2
  const double c = fmin(1.0, fmax(-1.0, 0.5 * ((m[0] + m[4]) + m[8] - 1.0)));
  const double uu = fma(u[0], u[0], fma(u[1], u[1], u[2] * u[2]));
  double q;
  if (vv == 0.0) {  // identical rotations: w = 0, v = u
    q = st * uu;
  } else {
    const double ivs = rsqrt_nr(vv);  // 1 / |vee|
    const double s = 0.5 * (vv * ivs);
    const double theta = atan2(s, c);
    if (theta > 3.14159265358979323846 - 1e-2) {  // near the pi branch: reference path
      *ok = false;
      return 0.0f;
    }
    const double r2 = fma(s, s, c * c);
    const double inv_r = rsqrt_nr(r2);
    const double r = r2 * inv_r;
    const double th = theta * r;  // |w|
    const double th2 = th * th;
    const double uw = fma(u[0], v0, fma(u[1], v1, u[2] * v2)) * ivs;
    const double par = uw * uw;  // (u . w^)^2
    const double perp = fmax(uu - par, 0.0);
    double F;  // th^2 / (4 sin^2(th/2))
    if (th2 < 1e-6) {
      F = fma(th2, fma(th2, 1.0 / 240.0, 1.0 / 12.0), 1.0);
    } else {
      const double S = s * inv_r, Cc = c * inv_r, dl = theta * (r - 1.0);  // th = theta + dl
      const double sin_th = fma(dl, Cc, S) - 0.5 * dl * dl * S;
      const double cos_th = fma(-dl, S, Cc) - 0.5 * dl * dl * Cc;
      // 4 sin^2(th/2) = 2(1 - cos th) = 2 sin^2 th / (1 + cos th)
      F = cos_th < 0.0 ? th2 * rcp_nr(2.0 * (1.0 - cos_th)) : th2 * (1.0 + cos_th) * rcp_nr(2.0 * sin_th * sin_th);
    }
    q = fma(sr, th2, st * fma(perp, F, par));
  }
  if (!(q == q)) {
    *ok = false;
    return 0.0f;
  }
  const double k = exp(-q);
  const float lo = __double2float_rn(k * (1.0 - 4e-12)), hi = __double2float_rn(k * (1.0 + 4e-12));
  *ok = lo == hi;
  return hi;
}

// Kernel value of the pair as the reference computes it, via kval_fast when
// its float is provably the same.
__device__ __forceinline__ float kval_of(const Pose& a, const Pose& b, double sr, double st) {
  if (kernel_underflows(a, b, st)) return 0.0f;
  bool ok;
  const float f = kval_fast(a, b, sr, st, &ok);
  if (ok) return f;
  double d[6];
  se3_log(inv_compose_x(a, b), d);
  return __double2float_rn(exp(-kernel_q(d, sr, st)));
}


__global__ void k_pairs(const Pose* __restrict__ P, const int2* __restrict__ pr, int n, double sr, double st, float* out) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int2 q = pr[t];
  out[t] = kval_of(P[q.x], P[q.y], sr, st);
}
}
