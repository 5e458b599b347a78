// ORACLE — test infrastructure only. CPU restatement of the steinmcl reference
// (MegaParticles, arXiv 2404.16370) hot path. Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load this code; the
// product (paper_2404_16370_b200/) never links it.
//
// Fixed-size linear algebra, SE3, RNG and deterministic reductions without
// Eigen. Every expression follows the reference's formula with a canonical
// left-to-right evaluation order ((x0 + x1) + x2 ...), and the library is built
// with -ffp-contract=off so that no multiply-add is fused. The CUDA "exact"
// paths mirror this order with __dmul_rn/__dadd_rn, which is what makes
// bit-for-bit GPU==oracle comparisons possible for +,-,*,/,sqrt-only math.
//
// Ulp-level agreement with an Eigen build of the reference is unpinned (Eigen's
// vectorised reduction order is not documented); see DESIGN.md §Oracle.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- vectors
struct V3 {
  double x[3] = {0.0, 0.0, 0.0};
  double& operator[](int i) { return x[i]; }
  double operator[](int i) const { return x[i]; }
};
struct V6 {
  double x[6] = {0, 0, 0, 0, 0, 0};
  double& operator[](int i) { return x[i]; }
  double operator[](int i) const { return x[i]; }
};
// Row-major 3x3: m[r*3+c].
struct M3 {
  double m[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  double& operator()(int r, int c) { return m[r * 3 + c]; }
  double operator()(int r, int c) const { return m[r * 3 + c]; }
  static M3 identity() {
    M3 a;
    a.m[0] = a.m[4] = a.m[8] = 1.0;
    return a;
  }
};
// Row-major 6x6.
struct M6 {
  double m[36] = {};
  double& operator()(int r, int c) { return m[r * 6 + c]; }
  double operator()(int r, int c) const { return m[r * 6 + c]; }
};

inline V3 v3(double a, double b, double c) {
  V3 v;
  v.x[0] = a;
  v.x[1] = b;
  v.x[2] = c;
  return v;
}
inline V3 operator+(const V3& a, const V3& b) { return v3(a[0] + b[0], a[1] + b[1], a[2] + b[2]); }
inline V3 operator-(const V3& a, const V3& b) { return v3(a[0] - b[0], a[1] - b[1], a[2] - b[2]); }
inline V3 operator*(double s, const V3& a) { return v3(s * a[0], s * a[1], s * a[2]); }
inline double dot(const V3& a, const V3& b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }
inline double sqnorm(const V3& a) { return dot(a, a); }
inline double norm(const V3& a) { return std::sqrt(sqnorm(a)); }

// se3.hpp:19-25
inline M3 skew(const V3& a) {
  M3 s;
  s(0, 0) = 0.0;   s(0, 1) = -a[2]; s(0, 2) = a[1];
  s(1, 0) = a[2];  s(1, 1) = 0.0;   s(1, 2) = -a[0];
  s(2, 0) = -a[1]; s(2, 1) = a[0];  s(2, 2) = 0.0;
  return s;
}
inline M3 mul(const M3& a, const M3& b) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r(i, j) = (a(i, 0) * b(0, j) + a(i, 1) * b(1, j)) + a(i, 2) * b(2, j);
  return r;
}
inline V3 mul(const M3& a, const V3& v) {
  V3 r;
  for (int i = 0; i < 3; ++i) r[i] = (a(i, 0) * v[0] + a(i, 1) * v[1]) + a(i, 2) * v[2];
  return r;
}
inline M3 transpose(const M3& a) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = a(j, i);
  return r;
}
inline M3 add(const M3& a, const M3& b) {
  M3 r;
  for (int i = 0; i < 9; ++i) r.m[i] = a.m[i] + b.m[i];
  return r;
}
inline M3 scale(double s, const M3& a) {
  M3 r;
  for (int i = 0; i < 9; ++i) r.m[i] = s * a.m[i];
  return r;
}
inline double trace(const M3& a) { return (a(0, 0) + a(1, 1)) + a(2, 2); }

// Eigen's 3x3 inverse (InverseImpl.h compute_inverse<...,3>): cofactors of
// column 0, det = sum(cof0 .* col0), invdet = 1/det, result(i,j) = cof(j,i)*invdet.
inline double cofactor3(const M3& m, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return m(i1, j1) * m(i2, j2) - m(i1, j2) * m(i2, j1);
}
inline M3 inverse3(const M3& m) {
  const double c00 = cofactor3(m, 0, 0), c10 = cofactor3(m, 1, 0), c20 = cofactor3(m, 2, 0);
  const double det = (c00 * m(0, 0) + c10 * m(1, 0)) + c20 * m(2, 0);
  const double invdet = 1.0 / det;
  M3 r;
  r(0, 0) = c00 * invdet;
  r(0, 1) = c10 * invdet;
  r(0, 2) = c20 * invdet;
  r(1, 0) = cofactor3(m, 0, 1) * invdet;
  r(1, 1) = cofactor3(m, 1, 1) * invdet;
  r(1, 2) = cofactor3(m, 2, 1) * invdet;
  r(2, 0) = cofactor3(m, 0, 2) * invdet;
  r(2, 1) = cofactor3(m, 1, 2) * invdet;
  r(2, 2) = cofactor3(m, 2, 2) * invdet;
  return r;
}

// ---------------------------------------------------------------- SE3
// se3.hpp:30-59. Rotation matrix + translation; right perturbations.
struct Pose {
  M3 R = M3::identity();
  V3 t;
};

inline Pose compose(const Pose& a, const Pose& b) {  // se3.hpp:61-63
  Pose p;
  p.R = mul(a.R, b.R);
  p.t = mul(a.R, b.t) + a.t;
  return p;
}
inline V3 transform(const Pose& a, const V3& p) { return mul(a.R, p) + a.t; }  // se3.hpp:65
inline Pose inverse(const Pose& a) {  // se3.hpp:36-41
  Pose p;
  p.R = transpose(a.R);
  const V3 rt = mul(p.R, a.t);
  p.t = v3(-rt[0], -rt[1], -rt[2]);
  return p;
}
// se3.hpp:44-46: max |R^T R - I|
inline double rotation_drift(const Pose& p) {
  const M3 rtr = mul(transpose(p.R), p.R);
  double mx = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const double d = std::fabs(rtr(i, j) - (i == j ? 1.0 : 0.0));
      if (d > mx) mx = d;
    }
  return mx;
}

// Eigen Quaternion(Matrix3) (Quaternion.h quaternionbase_assign_impl), q in
// (x,y,z,w) coefficient order.
inline void quat_from_matrix(const M3& mat, double q[4]) {
  double t = trace(mat);
  if (t > 0.0) {
    t = std::sqrt(t + 1.0);
    q[3] = 0.5 * t;
    t = 0.5 / t;
    q[0] = (mat(2, 1) - mat(1, 2)) * t;
    q[1] = (mat(0, 2) - mat(2, 0)) * t;
    q[2] = (mat(1, 0) - mat(0, 1)) * t;
  } else {
    int i = 0;
    if (mat(1, 1) > mat(0, 0)) i = 1;
    if (mat(2, 2) > mat(i, i)) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    t = std::sqrt(((mat(i, i) - mat(j, j)) - mat(k, k)) + 1.0);
    q[i] = 0.5 * t;
    t = 0.5 / t;
    q[3] = (mat(k, j) - mat(j, k)) * t;
    q[j] = (mat(j, i) + mat(i, j)) * t;
    q[k] = (mat(k, i) + mat(i, k)) * t;
  }
}
// Eigen QuaternionBase::toRotationMatrix, q = (x,y,z,w).
inline M3 quat_to_matrix(const double q[4]) {
  const double x = q[0], y = q[1], z = q[2], w = q[3];
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  M3 r;
  r(0, 0) = 1.0 - (tyy + tzz);
  r(0, 1) = txy - twz;
  r(0, 2) = txz + twy;
  r(1, 0) = txy + twz;
  r(1, 1) = 1.0 - (txx + tzz);
  r(1, 2) = tyz - twx;
  r(2, 0) = txz - twy;
  r(2, 1) = tyz + twx;
  r(2, 2) = 1.0 - (txx + tyy);
  return r;
}
// se3.hpp:48-58
inline void orthonormalize(Pose& p) {
  double q[4];
  quat_from_matrix(p.R, q);
  const double n = std::sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
  for (double& c : q) c = c / n;
  p.R = quat_to_matrix(q);
}
inline void renormalize_if_needed(Pose& p, double threshold = 1e-7) {
  if (rotation_drift(p) > threshold) orthonormalize(p);
}

// se3.hpp:73-97
inline Pose se3_exp(const V6& xi) {
  const V3 omega = v3(xi[0], xi[1], xi[2]);
  const V3 v = v3(xi[3], xi[4], xi[5]);
  const double theta2 = sqnorm(omega);
  const double theta = std::sqrt(theta2);
  double a, b, c;
  if (theta < 1e-4) {
    a = (1.0 - theta2 / 6.0) + (theta2 * theta2) / 120.0;
    b = (0.5 - theta2 / 24.0) + (theta2 * theta2) / 720.0;
    c = (1.0 / 6.0 - theta2 / 120.0) + (theta2 * theta2) / 5040.0;
  } else {
    const double s_half = std::sin(0.5 * theta);
    a = std::sin(theta) / theta;
    b = ((2.0 * s_half) * s_half) / theta2;
    c = (1.0 - a) / theta2;
  }
  const M3 s = skew(omega);
  const M3 s2 = mul(s, s);
  Pose p;
  M3 vm;
  for (int i = 0; i < 9; ++i) {
    const double id = (i % 4 == 0) ? 1.0 : 0.0;
    p.R.m[i] = (id + a * s.m[i]) + b * s2.m[i];
    vm.m[i] = (id + b * s.m[i]) + c * s2.m[i];
  }
  p.t = mul(vm, v);
  return p;
}

// se3.hpp:103-149
inline V6 se3_log(const Pose& p) {
  const M3& r = p.R;
  const V3 vee = v3(r(2, 1) - r(1, 2), r(0, 2) - r(2, 0), r(1, 0) - r(0, 1));
  const double s = 0.5 * norm(vee);
  const double cos_theta = std::min(1.0, std::max(-1.0, 0.5 * (trace(r) - 1.0)));
  const double theta = std::atan2(s, cos_theta);
  V3 omega;
  if (theta > M_PI - 1e-6) {
    M3 aat;
    for (int i = 0; i < 9; ++i) aat.m[i] = 0.5 * (r.m[i] + ((i % 4 == 0) ? 1.0 : 0.0));
    int k = 0;
    if (aat(1, 1) > aat(k, k)) k = 1;
    if (aat(2, 2) > aat(k, k)) k = 2;
    V3 axis;
    axis[k] = std::sqrt(std::max(aat(k, k), 0.0));
    const double inv = axis[k] > 0.0 ? 1.0 / axis[k] : 0.0;
    for (int j = 0; j < 3; ++j)
      if (j != k) axis[j] = aat(j, k) * inv;
    const double n = norm(axis);
    if (n > 0.0)
      for (int j = 0; j < 3; ++j) axis[j] = axis[j] / n;
    omega = theta * axis;
  } else if (theta < 1e-8) {
    omega = 0.5 * vee;
  } else {
    omega = (theta / (2.0 * std::sin(theta))) * vee;
  }
  const double theta2 = sqnorm(omega);
  double coef;
  if (theta2 < 1e-8) {
    coef = 1.0 / 12.0 + theta2 / 720.0;
  } else {
    const double th = std::sqrt(theta2);
    const double a = std::sin(th) / th;
    const double s_half = std::sin(0.5 * th);
    const double b = ((2.0 * s_half) * s_half) / theta2;
    coef = (1.0 - (0.5 * a) / b) / theta2;
  }
  const M3 sk = skew(omega);
  const M3 sk2 = mul(sk, sk);
  M3 v_inv;
  for (int i = 0; i < 9; ++i) {
    const double id = (i % 4 == 0) ? 1.0 : 0.0;
    v_inv.m[i] = (id - 0.5 * sk.m[i]) + coef * sk2.m[i];
  }
  const V3 vt = mul(v_inv, p.t);
  V6 xi;
  xi[0] = omega[0]; xi[1] = omega[1]; xi[2] = omega[2];
  xi[3] = vt[0]; xi[4] = vt[1]; xi[5] = vt[2];
  return xi;
}

// ---------------------------------------------------------------- RNG
// rng.hpp:15-31
struct SplitMix64 {
  std::uint64_t state = 0;
  SplitMix64() = default;
  explicit SplitMix64(std::uint64_t s) : state(s) {}
  std::uint64_t operator()() {
    std::uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
};
// rng.hpp:33-40
inline std::uint64_t mix_seed(std::uint64_t a, std::uint64_t b) {
  SplitMix64 g(a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2)));
  return g();
}
inline std::uint64_t mix_seed(std::uint64_t a, std::uint64_t b, std::uint64_t c) {
  return mix_seed(mix_seed(a, b), c);
}
// rng.hpp:43-49
inline double uniform01(SplitMix64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }
inline double uniform_range(SplitMix64& rng, double lo, double hi) {
  return lo + (hi - lo) * uniform01(rng);
}
// rng.hpp:52-59
inline void normal_pair(SplitMix64& rng, double& z0, double& z1) {
  const double u1 = 1.0 - uniform01(rng);
  const double u2 = uniform01(rng);
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double a = (2.0 * M_PI) * u2;
  z0 = r * std::cos(a);
  z1 = r * std::sin(a);
}
inline double normal01(SplitMix64& rng) {
  double z0, z1;
  normal_pair(rng, z0, z1);
  return z0;
}
// rng.hpp:67-73
inline V6 normal6(SplitMix64& rng) {
  V6 z;
  normal_pair(rng, z[0], z[1]);
  normal_pair(rng, z[2], z[3]);
  normal_pair(rng, z[4], z[5]);
  return z;
}
// rng.hpp:76-87 (Shoemake; Quaterniond(w,x,y,z).toRotationMatrix())
inline M3 random_rotation(SplitMix64& rng) {
  const double u1 = uniform01(rng);
  const double u2 = uniform01(rng);
  const double u3 = uniform01(rng);
  const double a = std::sqrt(1.0 - u1);
  const double b = std::sqrt(u1);
  double q[4];
  q[3] = b * std::cos((2.0 * M_PI) * u3);
  q[0] = a * std::sin((2.0 * M_PI) * u2);
  q[1] = a * std::cos((2.0 * M_PI) * u2);
  q[2] = b * std::sin((2.0 * M_PI) * u3);
  return quat_to_matrix(q);
}
// rng.hpp:89-92 (Eigen AngleAxis::toRotationMatrix with axis = UnitZ)
inline M3 random_yaw(SplitMix64& rng) {
  const double yaw = uniform_range(rng, -M_PI, M_PI);
  const double s = std::sin(yaw), c = std::cos(yaw);
  const double ax[3] = {0.0, 0.0, 1.0};
  const double sin_axis[3] = {s * ax[0], s * ax[1], s * ax[2]};
  const double cos1_axis[3] = {(1.0 - c) * ax[0], (1.0 - c) * ax[1], (1.0 - c) * ax[2]};
  M3 r;
  double tmp = cos1_axis[0] * ax[1];
  r(0, 1) = tmp - sin_axis[2];
  r(1, 0) = tmp + sin_axis[2];
  tmp = cos1_axis[0] * ax[2];
  r(0, 2) = tmp + sin_axis[1];
  r(2, 0) = tmp - sin_axis[1];
  tmp = cos1_axis[1] * ax[2];
  r(1, 2) = tmp - sin_axis[0];
  r(2, 1) = tmp + sin_axis[0];
  for (int i = 0; i < 3; ++i) r(i, i) = cos1_axis[i] * ax[i] + c;
  return r;
}

// ---------------------------------------------------------------- reductions
// reduce.hpp:14-69: fixed 4096-element chunks, combined in chunk order.
inline constexpr std::size_t k_reduce_chunk = 4096;

template <class F>
double chunked_sum(std::size_t n, F&& value_at) {
  if (n == 0) return 0.0;
  const std::size_t n_chunks = (n + k_reduce_chunk - 1) / k_reduce_chunk;
  std::vector<double> partial(n_chunks, 0.0);
#pragma omp parallel for schedule(static)
  for (std::int64_t c = 0; c < static_cast<std::int64_t>(n_chunks); ++c) {
    const std::size_t begin = static_cast<std::size_t>(c) * k_reduce_chunk;
    const std::size_t end = std::min(begin + k_reduce_chunk, n);
    double acc = 0.0;
    for (std::size_t i = begin; i < end; ++i) acc += value_at(i);
    partial[static_cast<std::size_t>(c)] = acc;
  }
  double total = 0.0;
  for (double v : partial) total += v;
  return total;
}

struct ArgMax {
  double value = -std::numeric_limits<double>::infinity();
  std::int64_t index = -1;
};

template <class F>
ArgMax chunked_argmax(std::size_t n, F&& value_at) {
  ArgMax out;
  if (n == 0) return out;
  const std::size_t n_chunks = (n + k_reduce_chunk - 1) / k_reduce_chunk;
  std::vector<ArgMax> partial(n_chunks);
#pragma omp parallel for schedule(static)
  for (std::int64_t c = 0; c < static_cast<std::int64_t>(n_chunks); ++c) {
    const std::size_t begin = static_cast<std::size_t>(c) * k_reduce_chunk;
    const std::size_t end = std::min(begin + k_reduce_chunk, n);
    ArgMax best;
    for (std::size_t i = begin; i < end; ++i) {
      const double v = value_at(i);
      if (v > best.value) {
        best.value = v;
        best.index = static_cast<std::int64_t>(i);
      }
    }
    partial[static_cast<std::size_t>(c)] = best;
  }
  for (const ArgMax& p : partial)
    if (p.value > out.value) out = p;
  return out;
}

}  // namespace orc
