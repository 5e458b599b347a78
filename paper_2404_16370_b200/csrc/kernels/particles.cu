// K9 predict / noise injection (reference filter.cpp:67-84), K10 uniform
// initialisation (filter.cpp:39-65), K8 SVGD (svgd.cpp:7-62): one thread per
// particle, fp64, counter-seeded SplitMix64 streams keyed by the GLOBAL
// particle index (so results do not depend on the shard count).
#include <cuda_runtime.h>

#include <cstdlib>

#include "../engine.cuh"
#include "../kernels.cuh"

namespace smcl {

namespace {

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

__global__ void k_predict(Pose* __restrict__ poses, int64_t n, int64_t gbase, PredictParams pp) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Pose p = compose_x(poses[i], pp.delta);
  if (!pp.noiseless) {
    SplitMix64 rng(mix_seed(pp.frame_seed, static_cast<uint64_t>(gbase + i)));
    double z[6], xi[6];
    rng.normal6(z);
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      double acc = xmul(pp.L[r * 6 + 0], z[0]);
#pragma unroll
      for (int c = 1; c < 6; ++c) acc = xadd(acc, xmul(pp.L[r * 6 + c], z[c]));
      xi[r] = acc;
    }
    p = compose_x(p, se3_exp(xi));
  }
  renormalize_if_needed(p);
  poses[i] = p;
}

__global__ void k_init_uniform(Pose* __restrict__ poses, double* __restrict__ log_post, int32_t* __restrict__ id,
                               int32_t* __restrict__ idx, float* __restrict__ kval, int32_t* __restrict__ count,
                               int64_t n, int64_t gbase, int k, InitParams ip) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t gi = gbase + i;
  SplitMix64 rng(mix_seed(ip.stream, static_cast<uint64_t>(gi)));
  Pose p;
  if (ip.full_rotation)
    random_rotation(rng, p.R);
  else
    random_yaw(rng, p.R);
#pragma unroll
  for (int a = 0; a < 3; ++a) p.t[a] = rng.uniform_range(ip.bmin[a], ip.bmax[a]);
  poses[i] = p;
  log_post[i] = ip.log_post0;
  id[i] = static_cast<int32_t>(gi);
  count[i] = 1;
  for (int s = 0; s < k; ++s) {
    idx[i * k + s] = s == 0 ? static_cast<int32_t>(gi) : -1;
    kval[i * k + s] = s == 0 ? 1.0f : 0.0f;
  }
}

// d = log(a^-1 b) (se3.hpp:103-149) for the SVGD sums, without libm sin
// calls and with FMA contraction (svgd results are compared within 1e-12
// relative, not bitwise). With Rrel = Ra^T Rb, vee = (Rrel - Rrel^T)^vee,
// s = |vee|/2, c = (tr Rrel - 1)/2, r = hypot(s, c), theta = atan2(s, c):
//   sin theta = s / r exactly, so the reference's w = theta / (2 sin theta) vee
//   is theta r / (2 s) vee; |w| = th = theta r, and sin/cos of th follow from
//   those of theta and the tiny th - theta (second order). V^-1 u =
//   u - w x u / 2 + coef w x (w x u) with coef = (1 - (th/2) cot(th/2)) / th^2
//   (the reference's (1 - (a/2)/b) / th^2). Near pi the reference branch is used.
__device__ __forceinline__ void se3_log_rel_fast(const Pose& a, const Pose& b, double d[6]) {
  double m[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      m[i * 3 + j] = fma(a.R[0 * 3 + i], b.R[0 * 3 + j], fma(a.R[1 * 3 + i], b.R[1 * 3 + j], a.R[2 * 3 + i] * b.R[2 * 3 + j]));
  const double v0 = m[7] - m[5], v1 = m[2] - m[6], v2 = m[3] - m[1];
  const double vv = fma(v0, v0, fma(v1, v1, v2 * v2));
  const double c = fmin(1.0, fmax(-1.0, 0.5 * ((m[0] + m[4]) + m[8] - 1.0)));
  double s = 0.0, ivs = 0.0;
  if (vv > 0.0) {
    ivs = rsqrt_nr(vv);
    s = 0.5 * (vv * ivs);
  }
  const double theta = atan2_pos(s, c);
  if (theta > kPi - 1e-6) {  // reference pi branch
    se3_log(inv_compose_x(a, b), d);
    return;
  }
  double w0, w1, w2, th;
  if (theta < 1e-8) {
    w0 = 0.5 * v0;
    w1 = 0.5 * v1;
    w2 = 0.5 * v2;
    th = sqrt(fma(w0, w0, fma(w1, w1, w2 * w2)));
  } else {
    const double r2 = fma(s, s, c * c);
    const double inv_r = rsqrt_nr(r2);
    const double r = r2 * inv_r;
    const double f = theta * r * ivs;  // theta r / (2 s) = theta r / |vee|
    w0 = f * v0;
    w1 = f * v1;
    w2 = f * v2;
    th = theta * r;
  }
  const double th2 = th * th;
  double coef;
  if (th2 < 1e-8) {
    coef = 1.0 / 12.0 + th2 / 720.0;
  } else {
    const double S = s / sqrt(fma(s, s, c * c)), C = c / sqrt(fma(s, s, c * c)), dl = th - theta;
    const double sin_th = fma(dl, C, S) - 0.5 * dl * dl * S;
    const double cos_th = fma(-dl, S, C) - 0.5 * dl * dl * C;
    // (th/2) cot(th/2) = (th/2) (1 + cos th) / sin th
    coef = (1.0 - 0.5 * th * (1.0 + cos_th) * rcp_nr(sin_th)) * rcp_nr(th2);
  }
  const double e0 = b.t[0] - a.t[0], e1 = b.t[1] - a.t[1], e2 = b.t[2] - a.t[2];
  double u[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) u[i] = fma(a.R[0 * 3 + i], e0, fma(a.R[1 * 3 + i], e1, a.R[2 * 3 + i] * e2));
  const double x0 = w1 * u[2] - w2 * u[1], x1 = w2 * u[0] - w0 * u[2], x2 = w0 * u[1] - w1 * u[0];  // w x u
  const double y0 = w1 * x2 - w2 * x1, y1 = w2 * x0 - w0 * x2, y2 = w0 * x1 - w1 * x0;              // w x (w x u)
  d[0] = w0;
  d[1] = w1;
  d[2] = w2;
  d[3] = fma(coef, y0, fma(-0.5, x0, u[0]));
  d[4] = fma(coef, y1, fma(-0.5, x1, u[1]));
  d[5] = fma(coef, y2, fma(-0.5, x2, u[2]));
}

// svgd.cpp:7-34 compute_phi, optionally fused with apply_updates (svgd.cpp:51-62)
// writing a second pose buffer so every read sees the frozen snapshot.
template <bool APPLY, int MINB, bool PF = true>
__global__ void __launch_bounds__(128, MINB) k_svgd(const Pose* __restrict__ all_poses, const double* __restrict__ all_steps,
                                              int64_t n, int64_t gbase, const int32_t* __restrict__ idx,
                                              const int32_t* __restrict__ count, int k, SvgdParams sp,
                                              double* __restrict__ phi_out, Pose* __restrict__ poses_out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t gi = gbase + i;
  const Pose pi = ldg_pose(all_poses + gi);
  double numer[6] = {0, 0, 0, 0, 0, 0};
  double denom = 0.0;
  const int cnt = count[i];
  const int32_t* __restrict__ row = idx + i * k;
  // PF: neighbour s + 1's pose and step are loaded while neighbour s is
  // evaluated (the loop is bound by these dependent L2/HBM gathers).
  int32_t jn = 0;
  Pose pn;
  double sn[6];
  auto fetch = [&](int s) {
    jn = row[s];
    pn = ldg_pose(all_poses + jn);
    const double2* sp2 = reinterpret_cast<const double2*>(all_steps + 6 * static_cast<int64_t>(jn));
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double2 v = __ldg(sp2 + c);
      sn[2 * c] = v.x;
      sn[2 * c + 1] = v.y;
    }
  };
  if (PF && cnt > 0) fetch(0);
  for (int s = 0; s < cnt; ++s) {
    int32_t j;
    Pose pj;
    double sj[6];
    if (PF) {
      j = jn;
      pj = pn;
#pragma unroll
      for (int c = 0; c < 6; ++c) sj[c] = sn[c];
      if (s + 1 < cnt) fetch(s + 1);
    } else {
      j = row[s];
#pragma unroll
      for (int c = 0; c < 6; ++c) sj[c] = all_steps[6 * static_cast<int64_t>(j) + c];
    }
    if (j == gi) {
#pragma unroll
      for (int c = 0; c < 6; ++c) numer[c] = numer[c] + sj[c];
      denom = denom + 1.0;
      continue;
    }
    if (!PF) pj = ldg_pose(all_poses + j);
    if (kernel_underflows(pi, pj, sp.sigma_t)) continue;
    double d[6];
    se3_log_rel_fast(pi, pj, d);
    const double q = fma(sp.sigma_r, fma(d[0], d[0], fma(d[1], d[1], d[2] * d[2])),
                         sp.sigma_t * fma(d[3], d[3], fma(d[4], d[4], d[5] * d[5])));
    const double kv = exp(-q);
    const double gr = -2.0 * kv * sp.sigma_r * sp.repulsion_gain, gt = -2.0 * kv * sp.sigma_t * sp.repulsion_gain;
#pragma unroll
    for (int c = 0; c < 6; ++c) numer[c] = fma(kv, sj[c], fma(c < 3 ? gr : gt, d[c], numer[c]));
    denom = denom + kv;
  }
  double phi[6];
  const double inv = 1.0 / denom;
#pragma unroll
  for (int c = 0; c < 6; ++c) phi[c] = numer[c] * inv;
  if (phi_out) {
#pragma unroll
    for (int c = 0; c < 6; ++c) phi_out[6 * i + c] = phi[c];
  }
  if (APPLY) {
    Pose p = compose_x(pi, se3_exp(phi));
    renormalize_if_needed(p);
    poses_out[i] = p;
  }
}

__global__ void k_apply(Pose* __restrict__ poses, const double* __restrict__ phis, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double phi[6];
#pragma unroll
  for (int c = 0; c < 6; ++c) phi[c] = phis[6 * i + c];
  Pose p = compose_x(poses[i], se3_exp(phi));
  renormalize_if_needed(p);
  poses[i] = p;
}

// Batch primitives for parity tests of the device SE3 library.
__global__ void k_exp_batch(const double* xi, int64_t n, Pose* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = se3_exp(xi + 6 * i);
}
__global__ void k_log_batch(const Pose* p, int64_t n, double* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) se3_log(p[i], out + 6 * i);
}
__global__ void k_kernel_batch(const Pose* a, const Pose* b, int64_t n, double sr, double st, double* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d[6];
  se3_log(inv_compose_x(a[i], b[i]), d);
  out[i] = exp(-kernel_q(d, sr, st));
}

}  // namespace

void launch_predict(Pose* poses, int64_t n, int64_t gbase, const PredictParams& pp, cudaStream_t st) {
  count_launch();
  if (n > 0) k_predict<<<blocks_for(n, 128), 128, 0, st>>>(poses, n, gbase, pp);
}
void launch_init_uniform(Pose* poses, double* log_post, int32_t* id, int32_t* idx, float* kval, int32_t* count,
                         int64_t n, int64_t gbase, int k, const InitParams& ip, cudaStream_t st) {
  count_launch();
  if (n > 0) k_init_uniform<<<blocks_for(n, 128), 128, 0, st>>>(poses, log_post, id, idx, kval, count, n, gbase, k, ip);
}
void launch_svgd(const Pose* all_poses, const double* all_steps, int64_t n, int64_t gbase, const int32_t* idx,
                 const int32_t* count, int k, const SvgdParams& sp, double* phi_out, Pose* poses_out,
                 cudaStream_t st) {
  count_launch();
  if (n <= 0) return;
  // The loop is bound by the dependent neighbour gathers (long-scoreboard
  // stalls): with the next neighbour's pose and step prefetched, 3 CTAs x 4
  // warps per SM (160 registers, no spills) measured best on B200 at 1M:
  // 0.58 ms (prefetch at 4 / 5 / 6 CTAs: 0.66 / 1.19 / 1.47 ms, spilling;
  // no prefetch at 7 CTAs, 72 registers: 0.78 ms).
  static const int cfg = [] {  // A/B: SMCL_SVGD_CFG=0 (no prefetch, 7 CTAs) or the CTAs per SM with prefetch
    const char* e = std::getenv("SMCL_SVGD_CFG");
    return e ? std::atoi(e) : 3;
  }();
  const unsigned g = static_cast<unsigned>(blocks_for(n, 128));
#define SVGD_LAUNCH(PF, MB)                                                                                      \
  if (poses_out)                                                                                                 \
    k_svgd<true, MB, PF><<<g, 128, 0, st>>>(all_poses, all_steps, n, gbase, idx, count, k, sp, phi_out, poses_out); \
  else                                                                                                           \
    k_svgd<false, MB, PF><<<g, 128, 0, st>>>(all_poses, all_steps, n, gbase, idx, count, k, sp, phi_out, nullptr);
  if (cfg == 0) {
    SVGD_LAUNCH(false, 7)
  } else if (cfg == 4) {
    SVGD_LAUNCH(true, 4)
  } else {
    SVGD_LAUNCH(true, 3)
  }
#undef SVGD_LAUNCH
}
void launch_apply(Pose* poses, const double* phis, int64_t n, cudaStream_t st) {
  count_launch();
  if (n > 0) k_apply<<<blocks_for(n, 128), 128, 0, st>>>(poses, phis, n);
}
void launch_exp_batch(const double* xi, int64_t n, Pose* out, cudaStream_t st) {
  count_launch();
  if (n > 0) k_exp_batch<<<blocks_for(n, 128), 128, 0, st>>>(xi, n, out);
}
void launch_log_batch(const Pose* p, int64_t n, double* out, cudaStream_t st) {
  count_launch();
  if (n > 0) k_log_batch<<<blocks_for(n, 128), 128, 0, st>>>(p, n, out);
}
void launch_kernel_batch(const Pose* a, const Pose* b, int64_t n, double sr, double st_, double* out, cudaStream_t st) {
  count_launch();
  if (n > 0) k_kernel_batch<<<blocks_for(n, 128), 128, 0, st>>>(a, b, n, sr, st_, out);
}

}  // namespace smcl
