// SE3 / RNG / small linear algebra for the B200 Stein-particle filter.
// __host__ __device__ so host setup (predict's Cholesky, LSH pass frames) and
// the sm_100a kernels evaluate identical code.
//
// Evaluation order: every formula follows the reference
// (/root/reference/proj/include/steinmcl/se3.hpp, rng.hpp) with left-to-right
// sums ((x0 + x1) + x2). Functions with the `_x` suffix ("exact") use
// __dmul_rn/__dadd_rn so nvcc cannot fuse them into FMAs: they are the ones
// whose results feed a discrete decision (voxel index, LSH cell) and must agree
// bit for bit with the CPU oracle. The others may contract to FMA (ulp-level
// differences only).
#pragma once

#include <cstdint>
#include <math.h>

#ifdef __CUDACC__
#define SMCL_HD __host__ __device__ __forceinline__
#define SMCL_ALIGN16 __align__(16)
#else
#define SMCL_HD inline
#define SMCL_ALIGN16 alignas(16)
#endif

namespace smcl {

#ifdef __CUDA_ARCH__
SMCL_HD double xmul(double a, double b) { return __dmul_rn(a, b); }
SMCL_HD double xadd(double a, double b) { return __dadd_rn(a, b); }
SMCL_HD double xsub(double a, double b) { return __dsub_rn(a, b); }
#else
// Host objects are compiled with -ffp-contract=off, so these stay unfused.
SMCL_HD double xmul(double a, double b) { return a * b; }
SMCL_HD double xadd(double a, double b) { return a + b; }
SMCL_HD double xsub(double a, double b) { return a - b; }
#endif

constexpr double kPi = 3.14159265358979323846;

#ifdef __CUDACC__
// Reciprocal / reciprocal square root: MUFU seed (~2^-22) + Newton steps
// (~1 ulp), no IEEE slow path. Arguments are positive normal numbers.
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
// atan2(s, c) for s >= 0 (angles in [0, pi]) at ~1 ulp: one division by a
// Newton reciprocal, octant reduction to |u| <= tan(pi/8) + eps, and
// atan(u) = u P(u^2) with a degree-11 near-minimax P on u^2 <= 0.18
// (scratch/atan_poly.py: max relative error 1.5e-16). No special cases: the
// callers pass finite (s, c) with s^2 + c^2 ~ 1.
__device__ __forceinline__ double atan2_pos(double s, double c) {
  constexpr double kT8 = 0.41421356237309504880;  // tan(pi/8)
  const double ac = fabs(c);
  double num, den, base;
  if (s <= kT8 * ac) {  // near 0 (c > 0) or near pi (c < 0): u = s / c
    num = s;
    den = c;
    base = c > 0.0 ? 0.0 : 3.14159265358979323846;
  } else if (ac <= kT8 * s) {  // near pi/2: u = -c / s
    num = -c;
    den = s;
    base = 1.57079632679489661923;
  } else if (c > 0.0) {  // near pi/4: u = (s - c) / (s + c)
    num = s - c;
    den = s + c;
    base = 0.78539816339744830962;
  } else {  // near 3pi/4: u = (s + c) / (c - s)
    num = s + c;
    den = c - s;
    base = 2.35619449019234492885;
  }
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
  double e = fma(-den, r, 1.0);
  r = fma(r, e, r);
  e = fma(-den, r, 1.0);
  r = fma(r, e, r);
  double u = num * r;
  u = fma(fma(-den, u, num), r, u);  // one correction step: u = num / den to ~1 ulp
  const double y = u * u;
  double p = -0.017085141492542092;
  p = fma(p, y, 0.037299486849215);
  p = fma(p, y, -0.05008578394066089);
  p = fma(p, y, 0.058409193896630636);
  p = fma(p, y, -0.06662122513410981);
  p = fma(p, y, 0.07691971387624114);
  p = fma(p, y, -0.09090892587575122);
  p = fma(p, y, 0.11111110595175504);
  p = fma(p, y, -0.14285714276163336);
  p = fma(p, y, 0.19999999999908397);
  p = fma(p, y, -0.3333333333333299);
  return fma(u * y, p, u) + base;  // u (1 + y p(y)) + base
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y * fma(-hx * y, y, 1.5);
}
#endif

// Pose: R row-major, t. 96 bytes, 16-byte aligned (6 x 128-bit loads).
struct SMCL_ALIGN16 Pose {
  double R[9];
  double t[3];
};

#ifdef __CUDACC__
// Read-only 96-byte pose as three 256-bit loads (sm_100 LDG.256; poses sit
// at 96-byte strides from a 256-byte aligned base, so every one is 32-byte
// aligned). A plain struct copy compiles to twelve 64-bit loads; the gather-
// heavy passes (neighbour pass, SVGD) are L1-wavefront bound.
__device__ __forceinline__ void ldg_v4d(const double* p, double& a, double& b, double& c, double& d) {
  // volatile: a non-volatile asm is a pure function to the compiler, which may
  // then hoist the load above the guard that makes the address valid.
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ Pose ldg_pose(const Pose* p) {
  const double* v = reinterpret_cast<const double*>(p);
  Pose q;
  ldg_v4d(v, q.R[0], q.R[1], q.R[2], q.R[3]);
  ldg_v4d(v + 4, q.R[4], q.R[5], q.R[6], q.R[7]);
  ldg_v4d(v + 8, q.R[8], q.t[0], q.t[1], q.t[2]);
  return q;
}
#endif

SMCL_HD Pose pose_identity() {
  Pose p;
#pragma unroll
  for (int i = 0; i < 9; ++i) p.R[i] = (i % 4 == 0) ? 1.0 : 0.0;
  p.t[0] = p.t[1] = p.t[2] = 0.0;
  return p;
}

// a.R * b.R, a.R * b.t + a.t  (se3.hpp:61-63), exact order.
SMCL_HD Pose compose_x(const Pose& a, const Pose& b) {
  Pose p;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j)
      p.R[i * 3 + j] = xadd(xadd(xmul(a.R[i * 3 + 0], b.R[0 * 3 + j]), xmul(a.R[i * 3 + 1], b.R[1 * 3 + j])),
                            xmul(a.R[i * 3 + 2], b.R[2 * 3 + j]));
    p.t[i] = xadd(xadd(xadd(xmul(a.R[i * 3 + 0], b.t[0]), xmul(a.R[i * 3 + 1], b.t[1])), xmul(a.R[i * 3 + 2], b.t[2])),
                  a.t[i]);
  }
  return p;
}

// inverse(a) * b without materialising the inverse: R = a.R^T b.R,
// t = a.R^T b.t + (-(a.R^T a.t)); identical rounding to compose(inverse(a), b).
SMCL_HD Pose inv_compose_x(const Pose& a, const Pose& b) {
  double it[3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    it[i] = -xadd(xadd(xmul(a.R[0 * 3 + i], a.t[0]), xmul(a.R[1 * 3 + i], a.t[1])), xmul(a.R[2 * 3 + i], a.t[2]));
  Pose p;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j)
      p.R[i * 3 + j] = xadd(xadd(xmul(a.R[0 * 3 + i], b.R[0 * 3 + j]), xmul(a.R[1 * 3 + i], b.R[1 * 3 + j])),
                            xmul(a.R[2 * 3 + i], b.R[2 * 3 + j]));
    p.t[i] = xadd(xadd(xadd(xmul(a.R[0 * 3 + i], b.t[0]), xmul(a.R[1 * 3 + i], b.t[1])), xmul(a.R[2 * 3 + i], b.t[2])),
                  it[i]);
  }
  return p;
}

// se3.hpp:44-46
SMCL_HD double rotation_drift(const Pose& p) {
  double mx = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double v = xadd(xadd(xmul(p.R[0 * 3 + i], p.R[0 * 3 + j]), xmul(p.R[1 * 3 + i], p.R[1 * 3 + j])),
                            xmul(p.R[2 * 3 + i], p.R[2 * 3 + j]));
      const double d = fabs(xsub(v, (i == j) ? 1.0 : 0.0));
      mx = d > mx ? d : mx;
    }
  return mx;
}

// Quaternion round trip of se3.hpp:48-52 (Eigen Quaternion(Matrix3) and
// toRotationMatrix), q = (x, y, z, w).
SMCL_HD void orthonormalize(Pose& p) {
  const double* m = p.R;
  double q[4];
  double t = xadd(xadd(m[0], m[4]), m[8]);
  if (t > 0.0) {
    t = sqrt(xadd(t, 1.0));
    q[3] = xmul(0.5, t);
    t = 0.5 / t;
    q[0] = xmul(xsub(m[7], m[5]), t);
    q[1] = xmul(xsub(m[2], m[6]), t);
    q[2] = xmul(xsub(m[3], m[1]), t);
  } else {
    int i = 0;
    if (m[4] > m[0]) i = 1;
    if (m[8] > m[i * 4]) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    t = sqrt(xadd(xsub(xsub(m[i * 4], m[j * 4]), m[k * 4]), 1.0));
    double qq[3];
    qq[i] = xmul(0.5, t);
    t = 0.5 / t;
    q[3] = xmul(xsub(m[k * 3 + j], m[j * 3 + k]), t);
    qq[j] = xmul(xadd(m[j * 3 + i], m[i * 3 + j]), t);
    qq[k] = xmul(xadd(m[k * 3 + i], m[i * 3 + k]), t);
    q[0] = qq[0];
    q[1] = qq[1];
    q[2] = qq[2];
  }
  const double n = sqrt(xadd(xadd(xadd(xmul(q[0], q[0]), xmul(q[1], q[1])), xmul(q[2], q[2])), xmul(q[3], q[3])));
  const double x = q[0] / n, y = q[1] / n, z = q[2] / n, w = q[3] / n;
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twx = xmul(tx, w), twy = xmul(ty, w), twz = xmul(tz, w);
  const double txx = xmul(tx, x), txy = xmul(ty, x), txz = xmul(tz, x);
  const double tyy = xmul(ty, y), tyz = xmul(tz, y), tzz = xmul(tz, z);
  p.R[0] = xsub(1.0, xadd(tyy, tzz));
  p.R[1] = xsub(txy, twz);
  p.R[2] = xadd(txz, twy);
  p.R[3] = xadd(txy, twz);
  p.R[4] = xsub(1.0, xadd(txx, tzz));
  p.R[5] = xsub(tyz, twx);
  p.R[6] = xsub(txz, twy);
  p.R[7] = xadd(tyz, twx);
  p.R[8] = xsub(1.0, xadd(txx, tyy));
}

SMCL_HD void renormalize_if_needed(Pose& p, double threshold = 1e-7) {
  if (rotation_drift(p) > threshold) orthonormalize(p);
}

// se3.hpp:73-97. Transcendentals are CUDA's (<= 2 ulp) on the device.
SMCL_HD Pose se3_exp(const double xi[6]) {
  const double w0 = xi[0], w1 = xi[1], w2 = xi[2];
  const double theta2 = xadd(xadd(xmul(w0, w0), xmul(w1, w1)), xmul(w2, w2));
  const double theta = sqrt(theta2);
  double a, b, c;
  if (theta < 1e-4) {
    const double t4 = xmul(theta2, theta2);
    a = xadd(xsub(1.0, theta2 / 6.0), t4 / 120.0);
    b = xadd(xsub(0.5, theta2 / 24.0), t4 / 720.0);
    c = xadd(xsub(1.0 / 6.0, theta2 / 120.0), t4 / 5040.0);
  } else {
    const double s_half = sin(xmul(0.5, theta));
    a = sin(theta) / theta;
    b = xmul(xmul(2.0, s_half), s_half) / theta2;
    c = xsub(1.0, a) / theta2;
  }
  // s = skew(w); s2 = s*s (full 3x3 product as the reference evaluates it).
  const double s[9] = {0.0, -w2, w1, w2, 0.0, -w0, -w1, w0, 0.0};
  double s2[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      s2[i * 3 + j] = xadd(xadd(xmul(s[i * 3 + 0], s[0 * 3 + j]), xmul(s[i * 3 + 1], s[1 * 3 + j])),
                           xmul(s[i * 3 + 2], s[2 * 3 + j]));
  Pose p;
  double vm[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const double id = (i % 4 == 0) ? 1.0 : 0.0;
    p.R[i] = xadd(xadd(id, xmul(a, s[i])), xmul(b, s2[i]));
    vm[i] = xadd(xadd(id, xmul(b, s[i])), xmul(c, s2[i]));
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
    p.t[i] = xadd(xadd(xmul(vm[i * 3 + 0], xi[3]), xmul(vm[i * 3 + 1], xi[4])), xmul(vm[i * 3 + 2], xi[5]));
  return p;
}

// se3.hpp:103-149.
SMCL_HD void se3_log(const Pose& p, double xi[6]) {
  const double* r = p.R;
  const double vee0 = xsub(r[7], r[5]), vee1 = xsub(r[2], r[6]), vee2 = xsub(r[3], r[1]);
  const double s = xmul(0.5, sqrt(xadd(xadd(xmul(vee0, vee0), xmul(vee1, vee1)), xmul(vee2, vee2))));
  const double tr = xadd(xadd(r[0], r[4]), r[8]);
  double cos_theta = xmul(0.5, xsub(tr, 1.0));
  cos_theta = fmin(1.0, fmax(-1.0, cos_theta));
  const double theta = atan2(s, cos_theta);
  double om0, om1, om2;
  if (theta > kPi - 1e-6) {
    double aat[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) aat[i] = xmul(0.5, xadd(r[i], (i % 4 == 0) ? 1.0 : 0.0));
    int k = 0;
    if (aat[4] > aat[0]) k = 1;
    if (aat[8] > aat[k * 4]) k = 2;
    double axis[3];
    axis[k] = sqrt(fmax(aat[k * 4], 0.0));
    const double inv = axis[k] > 0.0 ? 1.0 / axis[k] : 0.0;
#pragma unroll
    for (int j = 0; j < 3; ++j)
      if (j != k) axis[j] = xmul(aat[j * 3 + k], inv);
    const double n = sqrt(xadd(xadd(xmul(axis[0], axis[0]), xmul(axis[1], axis[1])), xmul(axis[2], axis[2])));
    if (n > 0.0) {
      axis[0] = axis[0] / n;
      axis[1] = axis[1] / n;
      axis[2] = axis[2] / n;
    }
    om0 = xmul(theta, axis[0]);
    om1 = xmul(theta, axis[1]);
    om2 = xmul(theta, axis[2]);
  } else if (theta < 1e-8) {
    om0 = xmul(0.5, vee0);
    om1 = xmul(0.5, vee1);
    om2 = xmul(0.5, vee2);
  } else {
    const double f = theta / xmul(2.0, sin(theta));
    om0 = xmul(f, vee0);
    om1 = xmul(f, vee1);
    om2 = xmul(f, vee2);
  }
  const double theta2 = xadd(xadd(xmul(om0, om0), xmul(om1, om1)), xmul(om2, om2));
  double coef;
  if (theta2 < 1e-8) {
    coef = xadd(1.0 / 12.0, theta2 / 720.0);
  } else {
    const double th = sqrt(theta2);
    const double a = sin(th) / th;
    const double s_half = sin(xmul(0.5, th));
    const double b = xmul(xmul(2.0, s_half), s_half) / theta2;
    coef = xsub(1.0, xmul(0.5, a) / b) / theta2;
  }
  const double sk[9] = {0.0, -om2, om1, om2, 0.0, -om0, -om1, om0, 0.0};
  double vi[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double s2 = xadd(xadd(xmul(sk[i * 3 + 0], sk[0 * 3 + j]), xmul(sk[i * 3 + 1], sk[1 * 3 + j])),
                             xmul(sk[i * 3 + 2], sk[2 * 3 + j]));
      const double id = (i == j) ? 1.0 : 0.0;
      vi[i * 3 + j] = xadd(xsub(id, xmul(0.5, sk[i * 3 + j])), xmul(coef, s2));
    }
  xi[0] = om0;
  xi[1] = om1;
  xi[2] = om2;
#pragma unroll
  for (int i = 0; i < 3; ++i)
    xi[3 + i] = xadd(xadd(xmul(vi[i * 3 + 0], p.t[0]), xmul(vi[i * 3 + 1], p.t[1])), xmul(vi[i * 3 + 2], p.t[2]));
}

// svgd.hpp:30-34: exp(-(sigma_r |w|^2 + sigma_t |v|^2)).
SMCL_HD double kernel_q(const double d[6], double sr, double st) {
  const double qr = xadd(xadd(xmul(d[0], d[0]), xmul(d[1], d[1])), xmul(d[2], d[2]));
  const double qt = xadd(xadd(xmul(d[3], d[3]), xmul(d[4], d[4])), xmul(d[5], d[5]));
  return xadd(xmul(sr, qr), xmul(st, qt));
}
SMCL_HD double kernel_of_tangent(const double d[6], double sr, double st) { return exp(-kernel_q(d, sr, st)); }

// svgd.hpp:45-47
SMCL_HD bool kernel_underflows(const Pose& a, const Pose& b, double st) {
  const double d0 = xsub(b.t[0], a.t[0]), d1 = xsub(b.t[1], a.t[1]), d2 = xsub(b.t[2], a.t[2]);
  return xmul(st, xadd(xadd(xmul(d0, d0), xmul(d1, d1)), xmul(d2, d2))) > 110.0;
}

// ---------------------------------------------------------------- RNG (rng.hpp)
struct SplitMix64 {
  uint64_t state;
  SMCL_HD explicit SplitMix64(uint64_t s) : state(s) {}
  SMCL_HD uint64_t next() {
    uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  SMCL_HD double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  SMCL_HD double uniform_range(double lo, double hi) { return xadd(lo, xmul(xsub(hi, lo), uniform01())); }
  SMCL_HD void normal_pair(double& z0, double& z1) {
    const double u1 = xsub(1.0, uniform01());
    const double u2 = uniform01();
    const double r = sqrt(xmul(-2.0, log(u1)));
    const double a = xmul(2.0 * kPi, u2);
    z0 = xmul(r, cos(a));
    z1 = xmul(r, sin(a));
  }
  SMCL_HD void normal6(double z[6]) {
    normal_pair(z[0], z[1]);
    normal_pair(z[2], z[3]);
    normal_pair(z[4], z[5]);
  }
};

SMCL_HD uint64_t mix_seed(uint64_t a, uint64_t b) {
  SplitMix64 g(a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2)));
  return g.next();
}
SMCL_HD uint64_t mix_seed(uint64_t a, uint64_t b, uint64_t c) { return mix_seed(mix_seed(a, b), c); }

// Eigen toRotationMatrix of q = (x, y, z, w).
SMCL_HD void quat_to_matrix(double x, double y, double z, double w, double R[9]) {
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twx = xmul(tx, w), twy = xmul(ty, w), twz = xmul(tz, w);
  const double txx = xmul(tx, x), txy = xmul(ty, x), txz = xmul(tz, x);
  const double tyy = xmul(ty, y), tyz = xmul(tz, y), tzz = xmul(tz, z);
  R[0] = xsub(1.0, xadd(tyy, tzz));
  R[1] = xsub(txy, twz);
  R[2] = xadd(txz, twy);
  R[3] = xadd(txy, twz);
  R[4] = xsub(1.0, xadd(txx, tzz));
  R[5] = xsub(tyz, twx);
  R[6] = xsub(txz, twy);
  R[7] = xadd(tyz, twx);
  R[8] = xsub(1.0, xadd(txx, tyy));
}

// rng.hpp:76-87 (Shoemake).
SMCL_HD void random_rotation(SplitMix64& rng, double R[9]) {
  const double u1 = rng.uniform01(), u2 = rng.uniform01(), u3 = rng.uniform01();
  const double a = sqrt(xsub(1.0, u1)), b = sqrt(u1);
  const double w = xmul(b, cos(xmul(2.0 * kPi, u3)));
  const double x = xmul(a, sin(xmul(2.0 * kPi, u2)));
  const double y = xmul(a, cos(xmul(2.0 * kPi, u2)));
  const double z = xmul(b, sin(xmul(2.0 * kPi, u3)));
  quat_to_matrix(x, y, z, w, R);
}

// rng.hpp:89-92 (Eigen AngleAxis(yaw, UnitZ).toRotationMatrix()).
SMCL_HD void random_yaw(SplitMix64& rng, double R[9]) {
  const double yaw = rng.uniform_range(-kPi, kPi);
  const double s = sin(yaw), c = cos(yaw);
  const double omc = xsub(1.0, c);
  // axis (0,0,1): sin_axis = (0,0,s), cos1_axis = (0,0,1-c)
  const double tmp01 = xmul(xmul(omc, 0.0), 0.0);
  R[1] = xsub(tmp01, s);
  R[3] = xadd(tmp01, s);
  const double tmp02 = xmul(xmul(omc, 0.0), 1.0);
  R[2] = xadd(tmp02, xmul(s, 0.0));
  R[6] = xsub(tmp02, xmul(s, 0.0));
  const double tmp12 = xmul(xmul(omc, 0.0), 1.0);
  R[5] = xsub(tmp12, xmul(s, 0.0));
  R[7] = xadd(tmp12, xmul(s, 0.0));
  R[0] = xadd(xmul(xmul(omc, 0.0), 0.0), c);
  R[4] = xadd(xmul(xmul(omc, 0.0), 0.0), c);
  R[8] = xadd(xmul(omc, 1.0), c);
}

}  // namespace smcl
