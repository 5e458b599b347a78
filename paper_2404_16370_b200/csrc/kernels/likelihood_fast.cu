// K1 / K2 fast path: per-particle GICP likelihood (+ Gauss-Newton system) for
// plane-model maps and scans (reference gicp.cpp:11-45, 109-137).
//
// Kernels:
//  * k_gicp_fast_q   K1 on L2-resident (plain-layout) record tables: warp per
//    particle, lanes stride the scan points (4 per lane per step); records
//    gathered into registers, candidates enqueued in a per-warp shared ring,
//    phase B on full warps from consecutive ring positions.
//  * k_gicp_fast     the staged-slot form (cp.async of every in-bounds record
//    into the warp's stage, compaction by slot index): K1 and the
//    likelihood-only warp pass on bricked, HBM-sized tables.
//  * k_ll_count      K2a: exact n_matched of every particle from an occupancy
//    bitmap with a proven fp32 margin, and the list of particles the gate keeps.
//  * k_gicp_ll_lanes K2: lane per particle, the likelihood of the gate's list.
//
// Phase A (every point): the point is transformed in fp64 with the pose
// pre-scaled to voxel units (x = Rv mu + tv, 9 DFMA); one round-down add of
// 1.5 * 2^28 splits x into the cell and a 24-bit fraction (cell_frac). x
// differs from the reference's ((R mu + t) - o) * inv_res (nnf.hpp:24-35) by
// < 2.2e-8 voxel (coordinates below 2^26 voxels; beyond, every point
// resolves), so the cell is the reference's unless the fraction is within
// 2^-24 of a face: such points "resolve" in phase B through the
// reference-order fp64 transform.
// Phase B (candidates, full warps): the body-frame structured-covariance
// algebra in fp32:
//   Sigma_M' + Sigma_s = A I - beta m m^T - gamma n n^T,
//   Omega' = (1/A)(I + P m m^T + Q n n^T + T (m n^T + n m^T)),
//   Delta  = A (s_M + s_S) + beta gamma |m x n|^2   (no cancellation),
// accumulating ll, H (21) and b (6) per lane; a shuffle reduction gives the
// per-particle system.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "../engine.cuh"
#include "../kernels.cuh"

namespace smcl {

namespace {

constexpr uint32_t kMetaStage = 1u << 16;    // fq.w: record staged (in bounds, cell proven)
constexpr uint32_t kMetaResolve = 1u << 17;  // fq.w: fraction within 2^-24 of a cell face: reference-order path

// Slots [0, kStep) hold the current step's points; slots [kStep, kStep + 32)
// the carry: candidates left over from earlier steps of the same particle
// (fewer than 32), so phase B runs full warps except on a particle's last step.
template <int kStep>
struct WarpStage {
  float4 m0[kStep + 32];  // staged cell records by point slot (SoA halves: conflict-free LDS.128)
  float4 m1[kStep + 32];
  float4 fq[kStep + 32];  // (fraction.xyz fp32, meta bits: k | kMetaStage | kMetaResolve) by point slot
  uint16_t q[kStep];  // compacted candidate slots
  double pose_v[12];  // Rv (row-major), tv: reloaded by phase A each step (no registers held in phase B)
  float rf[12];       // R in fp32 (row-major, 9 used): reloaded by each phase-B batch (no registers held in phase A)
};

// 128-bit shared-memory store / load at a shared-window address.
__device__ __forceinline__ void sts_f4(unsigned a, const float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float4 lds_f4(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

// Shared-memory loads the compiler may not hoist out of the batch loop (the
// values are re-read where they are used instead of pinning registers).
__device__ __forceinline__ float4 lds_f4_volatile(const float* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
  return v;
}

struct Acc {
  float hbr[6];  // Omega' lower: 00,10,11,20,21,22
  float htr[9];  // [mu]x Omega'
  float htl[6];  // lower of -W [mu]x
  float b[6];
  float cost;    // sum e^T Omega e
};

// 16-byte async copy; when !pred nothing is read and the destination is zero-filled.
// kL1: also allocate in L1 (.ca) — pays for bricked HBM-sized tables, where
// neighbouring particles re-read the same records; L2-resident tables use .cg.
// The zero fill uses the ignore-src predicate form (no src-size register).
template <bool kL1>
__device__ __forceinline__ void cp_async16_pred(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if (kL1)
    asm volatile("{\n .reg .pred q;\n setp.eq.u32 q, %2, 0;\n cp.async.ca.shared.global [%0], [%1], 16, q;\n}\n" ::"r"(s),
                 "l"(gmem), "r"(static_cast<unsigned>(pred))
                 : "memory");
  else
    asm volatile("{\n .reg .pred q;\n setp.eq.u32 q, %2, 0;\n cp.async.cg.shared.global [%0], [%1], 16, q;\n}\n" ::"r"(s),
                 "l"(gmem), "r"(static_cast<unsigned>(pred))
                 : "memory");
}
// One 32-byte record as a single 256-bit load (sm_100 LDG.256), predicated:
// when !pred nothing is read and the record reads as empty (beta = -1).
// One L1TEX request per record instead of two: random record gathers from
// the L2-resident table reach 8.1 TB/s this way against 3.2 (two 16-byte
// loads) or 4.6 (two 16-byte cp.async) — build/tools/micro_peaks.
__device__ __forceinline__ void ldg_rec_pred(const float4* src, bool pred, float4& m0, float4& m1) {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = -1.f, b0 = 0.f, b1 = 0.f, b2 = 0.f, b3 = 0.f;
  asm("{\n .reg .pred p;\n setp.ne.u32 p, %9, 0;\n"
      " @p ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n}"
      : "+f"(a0), "+f"(a1), "+f"(a2), "+f"(a3), "+f"(b0), "+f"(b1), "+f"(b2), "+f"(b3)
      : "l"(src), "r"(static_cast<unsigned>(pred)));
  m0 = make_float4(a0, a1, a2, a3);
  m1 = make_float4(b0, b1, b2, b3);
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// MUFU reciprocal (~1 ulp): A in [1e-8, 1e3], Delta in [1e-16, 1e6] for any
// physical covariance, far from the flush-to-zero range.
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Likelihood only: e^T Omega e is basis independent, and with n_w = R n the
// scalars the cost needs are world-frame dot/cross products (u.e = m'.e',
// n_w.e = n.e', u.n_w = m'.n, |u x n_w| = |m' x n|): one rotation (n) per
// point instead of two (e, u).
__device__ __forceinline__ float fast_cost(const float Rf[9], const float fr[3], float res, const float4 m0,
                                           const float4 m1, const float4 s0, const float4 s1) {
  const float ex = fmaf(-fr[0], res, m0.x), ey = fmaf(-fr[1], res, m0.y), ez = fmaf(-fr[2], res, m0.z);
  const float mx = m1.x, my = m1.y, mz = m1.z;  // map plane direction u (world)
  const float nx = Rf[0] * s1.x + Rf[1] * s1.y + Rf[2] * s1.z;  // R n (row-major R)
  const float ny = Rf[3] * s1.x + Rf[4] * s1.y + Rf[5] * s1.z;
  const float nz = Rf[6] * s1.x + Rf[7] * s1.y + Rf[8] * s1.z;
  const float beta = m0.w, sM = m1.w, gam = s0.w, sS = s1.w;
  const float Ssum = sM + sS;
  const float AmB = Ssum + gam;   // A - beta
  const float AmG = Ssum + beta;  // A - gamma
  const float A = AmG + gam;      // beta + gamma + s_M + s_S (4 adds instead of 8)
  const float c = mx * nx + my * ny + mz * nz;
  const float cx = my * nz - mz * ny, cy = mz * nx - mx * nz, cz = mx * ny - my * nx;
  const float w = cx * cx + cy * cy + cz * cz;
  const float bg = beta * gam;
  const float invD = rcp_approx(fmaf(A, Ssum, bg * w));
  const float invA = rcp_approx(A);
  const float x = mx * ex + my * ey + mz * ez;
  const float y = nx * ex + ny * ey + nz * ez;
  // e^T Omega e = |e|^2 / A + (beta AmG x^2 + gamma AmB y^2 + 2 c beta gamma x y) / (A Delta)
  const float bx = beta * x, gy = gam * y;
  const float inner = fmaf(AmG * bx, x, fmaf(AmB * gy, y, (c + c) * bx * gy));
  return fmaf(ex * ex + ey * ey + ez * ez, invA, inner * (invD * invA));
}

template <bool GN, bool kCost = true>
__device__ __forceinline__ void fast_item(Acc& acc, const float Rf[9], const float fr[3], float res, const float4 m0,
                                          const float4 m1, const float4 s0, const float4 s1) {
  if (!GN) {
    acc.cost += fast_cost(Rf, fr, res, m0, m1, s0, s1);
    return;
  }
  // World residual e = mu_M - p = (mu_M - corner) - frac*res.
  const float ewx = fmaf(-fr[0], res, m0.x), ewy = fmaf(-fr[1], res, m0.y), ewz = fmaf(-fr[2], res, m0.z);
  // Body frame: e' = R^T e_w, m' = R^T u_M, n' = u_s, mu = scan mean.
  const float ex = Rf[0] * ewx + Rf[3] * ewy + Rf[6] * ewz;
  const float ey = Rf[1] * ewx + Rf[4] * ewy + Rf[7] * ewz;
  const float ez = Rf[2] * ewx + Rf[5] * ewy + Rf[8] * ewz;
  const float mx = Rf[0] * m1.x + Rf[3] * m1.y + Rf[6] * m1.z;
  const float my = Rf[1] * m1.x + Rf[4] * m1.y + Rf[7] * m1.z;
  const float mz = Rf[2] * m1.x + Rf[5] * m1.y + Rf[8] * m1.z;
  const float nx = s1.x, ny = s1.y, nz = s1.z;
  const float beta = m0.w, sM = m1.w, gam = s0.w, sS = s1.w;
  const float Ssum = sM + sS;
  const float AmB = Ssum + gam;   // A - beta
  const float AmG = Ssum + beta;  // A - gamma
  const float A = AmG + gam;      // beta + gamma + s_M + s_S (4 adds instead of 8)
  const float c = mx * nx + my * ny + mz * nz;
  const float cx = my * nz - mz * ny, cy = mz * nx - mx * nz, cz = mx * ny - my * nx;
  const float w = cx * cx + cy * cy + cz * cz;
  const float bg = beta * gam;
  // MUFU reciprocals (2 ulp): A in [1e-8, 1e3], Delta in [1e-16, 1e6] for any
  // physical covariance, well inside __fdividef's range.
  const float invD = rcp_approx(fmaf(A, Ssum, bg * w));
  const float invA = rcp_approx(A);
  // P, Q, T pre-scaled by 1/A: Omega' = invA I + Pa m m^T + Qa n n^T + Ta (m n^T + n m^T)
  const float invDA = invD * invA;
  const float bI = beta * invDA;
  const float Pa = bI * AmG, Qa = gam * AmB * invDA, Ta = c * (bI * gam);
  const float x = mx * ex + my * ey + mz * ez;
  const float y = nx * ex + ny * ey + nz * ez;
  const float am = fmaf(Pa, x, Ta * y), an = fmaf(Qa, y, Ta * x);  // (Omega' - invA I) e = am m + an n
  if (kCost) acc.cost += fmaf(ex * ex + ey * ey + ez * ez, invA, fmaf(am, x, an * y));
  if (GN) {
    const float gx = fmaf(ex, invA, fmaf(am, mx, an * nx));  // g = Omega' e
    const float gy = fmaf(ey, invA, fmaf(am, my, an * ny));
    const float gz = fmaf(ez, invA, fmaf(am, mz, an * nz));
    const float ux = s0.x, uy = s0.y, uz = s0.z;  // scan mean (body frame)
    acc.b[0] += gy * uz - gz * uy;  // b_top += g x mu
    acc.b[1] += gz * ux - gx * uz;
    acc.b[2] += gx * uy - gy * ux;
    acc.b[3] -= gx;  // b_bot -= g
    acc.b[4] -= gy;
    acc.b[5] -= gz;
    // Omega' = invA I + alpha m^T + beta_ n^T,  alpha = Pa m + Ta n, beta_ = Qa n + Ta m
    // (symmetric: alpha_r m_q + beta_r n_q = invA (P m_r m_q + Q n_r n_q + T (n_r m_q + m_r n_q))).
    const float mv[3] = {mx, my, mz}, nv[3] = {nx, ny, nz};
    float al[3], be[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      al[r] = fmaf(Pa, mv[r], Ta * nv[r]);
      be[r] = fmaf(Qa, nv[r], Ta * mv[r]);
    }
    float O[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int q = 0; q <= r; ++q) {
        const float v = fmaf(al[r], mv[q], fmaf(be[r], nv[q], r == q ? invA : 0.f));
        O[r][q] = O[q][r] = v;
      }
    acc.hbr[0] += O[0][0];
    acc.hbr[1] += O[1][0];
    acc.hbr[2] += O[1][1];
    acc.hbr[3] += O[2][0];
    acc.hbr[4] += O[2][1];
    acc.hbr[5] += O[2][2];
    float W[3][3];  // W = [mu]x Omega'
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      W[0][j] = uy * O[2][j] - uz * O[1][j];
      W[1][j] = uz * O[0][j] - ux * O[2][j];
      W[2][j] = ux * O[1][j] - uy * O[0][j];
    }
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int q = 0; q < 3; ++q) acc.htr[r * 3 + q] += W[r][q];
    // H_tl -= W [mu]x (lower triangle), two FMAs per entry
    acc.htl[0] = fmaf(W[0][2], uy, fmaf(-W[0][1], uz, acc.htl[0]));
    acc.htl[1] = fmaf(W[1][2], uy, fmaf(-W[1][1], uz, acc.htl[1]));
    acc.htl[2] = fmaf(W[1][0], uz, fmaf(-W[1][2], ux, acc.htl[2]));
    acc.htl[3] = fmaf(W[2][2], uy, fmaf(-W[2][1], uz, acc.htl[3]));
    acc.htl[4] = fmaf(W[2][0], uz, fmaf(-W[2][2], ux, acc.htl[4]));
    acc.htl[5] = fmaf(W[2][1], ux, fmaf(-W[2][0], uy, acc.htl[5]));
  }
}

// Cell and fraction of a voxel coordinate x (|x| < 2^27) from ONE fp64 add:
// y = RD(x + 1.5 * 2^28) has ulp 2^-24, so its 52-bit mantissa holds the
// fixed-point value (2^27 + x) * 2^24 rounded down: the integer part
// (2^27 + floor(x), 28 bits) straddles the two words and the low 24 bits are
// f24 = floor(frac(x) * 2^24). With exponent 1051 (0x41B) in the high word,
//   ic  = funnelshift_l(lo, hi, 8) - 0xB8000000 = floor(x)  (negative: huge unsigned)
//   fr  = (f24 >> 1) * 2^-23 + 2^-24  (midpoint of the 2^-23 interval holding
//         frac(x): |fr - frac(x)| <= 2^-24 ~ 6e-8 voxel, the fp32 fraction's own
//         rounding), built from the bits with one FADD
//   clear of both faces by more than the 2.2e-8-voxel transform bound iff
//         1 <= f24 <= 2^24 - 2 (frac(x) in [2^-24, 1 - 2^-24)).
// 4 fp64 operations per axis instead of 6 plus a conversion (no F2F: the
// short-scoreboard stall of phase A). NaN x gives garbage bits: callers stage
// only real scan points of finite-pose particles (huge covers non-finite poses).
struct CellFrac {
  unsigned ic;
  float fr;
  unsigned f24;  // the fraction's raw bits (frac_of_f24 builds fr from them)
  bool clear;
};
__device__ __forceinline__ float frac_of_f24(unsigned f24) {
  return __uint_as_float(0x3F800000u | (f24 >> 1)) - (1.0f - 0x1p-24f);
}
__device__ __forceinline__ CellFrac cell_frac(double x) {
  constexpr double kMagic28 = 402653184.0;  // 1.5 * 2^28
  const double y = __dadd_rd(x, kMagic28);
  const unsigned lo = static_cast<unsigned>(__double2loint(y)), hi = static_cast<unsigned>(__double2hiint(y));
  CellFrac c;
  c.ic = __funnelshift_l(lo, hi, 8) - 0xB8000000u;
  const unsigned f24 = lo & 0xFFFFFFu;
  c.f24 = f24;
  c.fr = frac_of_f24(f24);
  c.clear = f24 - 1u < 0xFFFFFEu;
  return c;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Record slot of cell (ix, iy, iz) for the table layout fixed at compile time.
template <int kBrick>
__device__ __forceinline__ uint32_t rec_index(const MapFast& m, uint32_t ix, uint32_t iy, uint32_t iz) {
  const uint32_t nx = static_cast<uint32_t>(m.g.dims[0]), ny = static_cast<uint32_t>(m.g.dims[1]);
  if (!kBrick) return (iz * ny + iy) * nx + ix;
  const uint32_t b = ((iz >> 2) * ((ny + 3u) >> 2) + (iy >> 2)) * ((nx + 3u) >> 2) + (ix >> 2);
  return (b << 6) | ((iz & 3u) << 4) | ((iy & 3u) << 2) | (ix & 3u);
}

// Pose reload the compiler cannot merge with an earlier load of the same
// address: the rare resolve paths re-read the pose instead of keeping its
// 24 fp64 registers live across the whole scan loop.
__device__ __forceinline__ Pose reload_pose(const Pose* p) {
  Pose P;
  double* w = reinterpret_cast<double*>(&P);
  const double* s = reinterpret_cast<const double*>(p);
#pragma unroll
  for (int q = 0; q < 12; q += 2)
    asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(w[q]), "=d"(w[q + 1]) : "l"(s + q));
  return P;
}

__device__ __forceinline__ void transform_x(const double* R, const double* t, const double mu[3], double p[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
    p[i] = xadd(xadd(xadd(xmul(R[i * 3 + 0], mu[0]), xmul(R[i * 3 + 1], mu[1])), xmul(R[i * 3 + 2], mu[2])), t[i]);
}

template <bool GN, int kFastUnroll, int kWarps, int kBrick, bool kLdg = false, bool kCost = true>
__global__ void __launch_bounds__(kWarps * 32, 1)
    k_gicp_fast(const Pose* __restrict__ poses, int64_t n, ScanView scan, MapFast map, float* __restrict__ sysf,
                double* __restrict__ raw_ll, int32_t* __restrict__ nm_out, const int32_t* __restrict__ list,
                const unsigned* __restrict__ list_count) {
  constexpr int kStep = 32 * kFastUnroll;
  using Stage = WarpStage<kStep>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Stage* stages = reinterpret_cast<Stage*>(smem_raw);
  // Scan in shared memory, padded with NaN points to a multiple of kStep:
  // fp64 means (phase A transform), fp32 records split in two conflict-free halves.
  const int S = scan.n;
  const int Sp = (S + kStep - 1) / kStep * kStep;
  float4* s_r0 = reinterpret_cast<float4*>(smem_raw + sizeof(Stage) * kWarps);  // Sp: mu.xyz, gamma
  float4* s_r1 = s_r0 + Sp;                                                    // Sp: u.xyz, s
  double* s_mu = reinterpret_cast<double*>(s_r1 + Sp);                         // Sp*3
  for (int q = threadIdx.x; q < Sp; q += blockDim.x) {
    s_r0[q] = q < S ? scan.rec[2 * q] : make_float4(0.f, 0.f, 0.f, 0.f);
    s_r1[q] = q < S ? scan.rec[2 * q + 1] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int q = threadIdx.x; q < 3 * Sp; q += blockDim.x)
    s_mu[q] = q < 3 * S ? scan.mu[q] : __longlong_as_double(0x7ff8000000000000ll);
  __syncthreads();

  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t gwarp = static_cast<int64_t>(blockIdx.x) * kWarps + wid;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kWarps;
  const NnfGeom g = map.g;
  float res;  // kept in a register (not re-converted from the parameter in every batch)
  asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(res) : "d"(g.res));
  const int nx = g.dims[0], ny = g.dims[1];
  const unsigned dx = static_cast<unsigned>(g.dims[0]), dy = static_cast<unsigned>(g.dims[1]),
                 dz = static_cast<unsigned>(g.dims[2]);
  Stage& ws = stages[wid];

  const int64_t n_eff = list ? static_cast<int64_t>(*list_count) : n;  // list: the gate's live particles
  for (int64_t it = gwarp; it < n_eff; it += nwarps) {
    const int64_t i = list ? static_cast<int64_t>(list[it]) : it;
    // Pose in voxel units x = Rv mu + tv (Rv = R/res, tv = (t - o)/res) in
    // fp64 registers; Rf = R (fp32) for the body-frame algebra.
    bool huge;
    {
      // Lane q < 12 loads pose word q (R row-major, then t) and writes its
      // voxel-unit value and (q < 9) its fp32 rotation entry; the |x| bound is
      // shared by shuffles.
      const double pv = __ldg(reinterpret_cast<const double*>(poses + i) + (lane < 12 ? lane : 0));
      const bool isR = lane < 9, isT = lane >= 9 && lane < 12;
      const double o = lane == 9 ? g.origin[0] : (lane == 10 ? g.origin[1] : (lane == 11 ? g.origin[2] : 0.0));
      const double centered = pv - o;
      if (lane < 12) ws.pose_v[lane] = centered * g.inv_res;
      const float rf = static_cast<float>(pv);
      if (lane < 12) ws.rf[lane] = rf;
      // Resolve every point (NaN too) unless (max|R| |mu|_1 + max(|t| + |o|))
      // / res < 2^26: the reference forms p = R mu + t in world coordinates,
      // whose rounding (~3 ulp of |t| + |R mu|, plus p - o) stays below 2.2e-8
      // voxel there, inside the 2^-24 face margin; the fixed-point split
      // (cell_frac) needs |x| < 2^27 (implied).
      float mr = isR ? fabsf(rf) : 0.f,
            mt = isT ? fabsf(static_cast<float>(pv)) + fabsf(static_cast<float>(o)) : 0.f;
#pragma unroll
      for (int m = 8; m > 0; m >>= 1) {
        mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, m));
        mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, m));
      }
      mr = __shfl_sync(0xffffffffu, mr, 0);
      mt = __shfl_sync(0xffffffffu, mt, 0);
      huge = !((static_cast<double>(mr) * scan.mu_l1_max + static_cast<double>(mt)) * g.inv_res < 6.7e7) ||
             !(pv == pv);
      huge = __any_sync(0xffffffffu, huge);
    }
    __syncwarp();
    Acc acc;
#pragma unroll
    for (int q = 0; q < 6; ++q) acc.hbr[q] = acc.htl[q] = acc.b[q] = 0.f;
#pragma unroll
    for (int q = 0; q < 9; ++q) acc.htr[q] = 0.f;
    acc.cost = 0.f;
    int nmatch = 0;
    int n_carry = 0;  // candidates waiting in the carry slots (< 32)

    for (int base = 0; base < S; base += kStep) {
      // ---- phase A: fp64 cell + exact fraction, predicated async gather
      double Rv[9], tv[3];
      float4 rm0[kLdg ? kFastUnroll : 1], rm1[kLdg ? kFastUnroll : 1];  // kLdg: records in flight
      unsigned sflags = 0;  // per point slot u: bit 2u staged, bit 2u+1 resolve (compaction reads no meta back)
#pragma unroll
      for (int q = 0; q < 9; ++q) Rv[q] = ws.pose_v[q];
#pragma unroll
      for (int a = 0; a < 3; ++a) tv[a] = ws.pose_v[9 + a];
#pragma unroll
      for (int u = 0; u < kFastUnroll; ++u) {
        const int slot = u * 32 + lane, k = base + slot;
        const double m0 = s_mu[3 * k], m1 = s_mu[3 * k + 1], m2 = s_mu[3 * k + 2];
        float fr[3];
        int ic[3];
        bool safe = !huge, inb = true;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          const double x = fma(Rv[ax * 3 + 2], m2, fma(Rv[ax * 3 + 1], m1, fma(Rv[ax * 3 + 0], m0, tv[ax])));
          const CellFrac cf = cell_frac(x);
          ic[ax] = static_cast<int>(cf.ic);
          inb = inb & (cf.ic < (ax == 0 ? dx : (ax == 1 ? dy : dz)));
          fr[ax] = cf.fr;
          safe = safe & cf.clear;
        }
        const bool real = k < S;  // padded points (NaN) are neither staged nor resolved
        const bool amb = !safe;
        const bool resolve = amb && real;
        const bool stage = !amb && inb && real;
        // Unstaged points form an address that is never read (predicated
        // load / ignore-src copy), so the cell needs no select.
        const float4* src = map.rec + 2 * static_cast<uint64_t>(rec_index<kBrick>(map, ic[0], ic[1], ic[2]));
        if (kLdg) {
          ldg_rec_pred(src, stage, rm0[kLdg ? u : 0], rm1[kLdg ? u : 0]);
        } else {
          cp_async16_pred<kBrick != 0>(&ws.m0[slot], src, stage);
          cp_async16_pred<kBrick != 0>(&ws.m1[slot], src + 1, stage);
        }
        const uint32_t meta = static_cast<uint32_t>(k) | (stage ? kMetaStage : 0u) | (resolve ? kMetaResolve : 0u);
        ws.fq[slot] = make_float4(fr[0], fr[1], fr[2], __uint_as_float(meta));
        sflags |= (stage ? 1u : 0u) << (2 * u);
        sflags |= (resolve ? 2u : 0u) << (2 * u);
      }
      if (kLdg) {
#pragma unroll
        for (int u = 0; u < kFastUnroll; ++u) {
          ws.m0[u * 32 + lane] = rm0[kLdg ? u : 0];
          ws.m1[u * 32 + lane] = rm1[kLdg ? u : 0];
        }
      } else {
        cp_async_wait_all();
      }
      __syncwarp();
      // ---- compaction of the candidate slots (records stay in place)
      int n_cand = 0;
#pragma unroll
      for (int u = 0; u < kFastUnroll; ++u) {
        const int slot = u * 32 + lane;
        const bool staged = (sflags >> (2 * u)) & 1u, resolving = (sflags >> (2 * u + 1)) & 1u;
        // the record's occupancy is read only where one was staged (strided 4-byte reads conflict 4 ways)
        const bool keep = resolving || (staged && ws.m0[slot].w >= 0.f);
        const unsigned mask = __ballot_sync(0xffffffffu, keep);
        if (keep) ws.q[n_cand + __popc(mask & ((1u << lane) - 1u))] = static_cast<uint16_t>(slot);
        n_cand += __popc(mask);
      }
      __syncwarp();
      // ---- phase B: structured algebra on full warps; carried candidates
      // first, then this step's. Only the particle's last step runs a partial
      // warp; otherwise the remainder (< 32) moves to the carry slots.
      const int total = n_carry + n_cand;
      const bool last_step = base + kStep >= S;
      const int n_run = last_step ? total : (total & ~31);
      for (int b0 = 0; b0 < n_run; b0 += 32) {
        const int e = b0 + lane;
        bool valid = false;
        float Rf[9];
        {
          const float4 r0 = lds_f4_volatile(ws.rf), r1 = lds_f4_volatile(ws.rf + 4), r2 = lds_f4_volatile(ws.rf + 8);
          Rf[0] = r0.x, Rf[1] = r0.y, Rf[2] = r0.z, Rf[3] = r0.w, Rf[4] = r1.x, Rf[5] = r1.y, Rf[6] = r1.z,
          Rf[7] = r1.w, Rf[8] = r2.x;
        }
        if (e < n_run) {
          const int slot = e < n_carry ? kStep + e : ws.q[e - n_carry];
          const float4 fq = lds_f4_volatile(reinterpret_cast<const float*>(&ws.fq[slot]));  // one 128-bit read (meta included)
          const uint32_t meta = __float_as_uint(fq.w);
          const int k = static_cast<int>(meta & 0xFFFFu);
          float fr[3] = {fq.x, fq.y, fq.z};
          float4 m0, m1;
          valid = true;
          if (meta & kMetaResolve) {  // exact transform, floor and bounds (nnf.hpp:24-35), direct gather
            const Pose P = poses[i];
            const double mu[3] = {scan.mu[3 * k], scan.mu[3 * k + 1], scan.mu[3 * k + 2]};
            double p[3];
            transform_x(P.R, P.t, mu, p);
            int c3[3];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
              const double x = xmul(xsub(p[ax], g.origin[ax]), g.inv_res);
              const double fl = floor(x);
              valid = valid && (fl >= 0.0 && fl < static_cast<double>(g.dims[ax]));
              c3[ax] = valid ? static_cast<int>(fl) : 0;
              fr[ax] = __double2float_rn(xsub(x, fl));
            }
            const uint64_t c = rec_index<kBrick>(map, c3[0], c3[1], c3[2]);
            m0 = valid ? __ldg(map.rec + 2 * c) : make_float4(0.f, 0.f, 0.f, -1.f);
            m1 = valid ? __ldg(map.rec + 2 * c + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
            m0 = ws.m0[slot];
            m1 = ws.m1[slot];
          }
          valid = valid && m0.w >= 0.f;
          if (valid) fast_item<GN, kCost>(acc, Rf, fr, res, m0, m1, s_r0[k], s_r1[k]);
        }
        nmatch += __popc(__ballot_sync(0xffffffffu, valid));
      }
      __syncwarp();
      if (!last_step) {  // remainder elements [n_run, total) -> carry slots [0, total - n_run)
        const int e = n_run + lane;
        if (e < total && e >= n_carry) {  // e < n_carry (n_run == 0): already in carry slot e
          const int src = ws.q[e - n_carry], dst = kStep + e - n_run;
          ws.m0[dst] = ws.m0[src];
          ws.m1[dst] = ws.m1[src];
          ws.fq[dst] = ws.fq[src];
        }
        n_carry = total - n_run;
        __syncwarp();
      }
    }

    // ---- epilogue: lane q ends up with the warp total of accumulator q
    if (GN) {
      float v[32];
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        v[q] = acc.htl[q];
        v[15 + q] = acc.hbr[q];
        v[21 + q] = acc.b[q];
      }
#pragma unroll
      for (int q = 0; q < 9; ++q) v[6 + q] = acc.htr[q];
      v[27] = acc.cost;
      v[28] = v[29] = v[30] = v[31] = 0.f;
      // Butterfly reduce-scatter: after the step with offset s each lane keeps
      // the half selected by (lane & s); 31 shuffles instead of 140.
#pragma unroll
      for (int s = 16; s >= 1; s >>= 1) {
        const bool up = (lane & s) != 0;
#pragma unroll
        for (int j = 0; j < s; ++j) {
          const float send = up ? v[j] : v[j + s];
          const float keep = up ? v[j + s] : v[j];
          v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
        }
      }
      // One 128-byte line per particle (lanes 28-31 hold zeros), widened to
      // fp64 by the solve (SMCL_FAST_SYS_OFF).
      sysf[i * kSysF + lane] = v[0];
      if (kCost && lane == 27) raw_ll[i] = nmatch == 0 ? -1e30 : -static_cast<double>(v[0]);
    } else {
      const float cost = warp_sum(acc.cost);
      if (lane == 0) raw_ll[i] = nmatch == 0 ? -1e30 : -static_cast<double>(cost);
    }
    if (lane == 0) nm_out[i] = nmatch;  // also under the gate (predicted-live particles skip K2a)
    __syncwarp();
  }
}

// K1 variant with a per-warp candidate queue (L2-resident, plain-layout
// tables). Phase A gathers each point's 32-byte record straight into
// registers (one predicated 256-bit load), so the cell's occupancy is known
// before anything touches shared memory: only the candidates (occupied cells
// and resolving points, ~45 %) are written, at consecutive queue positions
// (ballot prefix), as (record, fraction + meta) = 48 B. Phase B consumes the
// queue 32 entries at a time from consecutive positions: conflict-free reads,
// no slot indirection, and the < 32 leftovers simply stay queued for the
// next step (ring of kQ = 32 U + 32 entries). Against k_gicp_fast this
// removes the all-point cp.async and fraction stores, the compaction
// read-back and the bank conflicts of the compacted-slot reads.
template <int kStepPts>
struct WarpQueue {
  static constexpr int kQ = kStepPts + 32;
  float4 m0[kQ];
  float4 m1[kQ];
  float4 fq[kQ];      // (raw fraction bits f24.xyz, meta: k | kMetaResolve)
  double pose_v[12];  // Rv (row-major), tv
  float rf[12];       // R in fp32 (row-major, 9 used)
};

template <bool GN, int U, int kWarps, bool kCost, int kBrick, bool kSmemRed = true>
__global__ void __launch_bounds__(kWarps * 32, 1)
    k_gicp_fast_q(const Pose* __restrict__ poses, int64_t n, ScanView scan, MapFast map, float* __restrict__ sysf,
                  double* __restrict__ raw_ll, int32_t* __restrict__ nm_out, const int32_t* __restrict__ list,
                  const unsigned* __restrict__ list_count) {
  constexpr int kStep = 32 * U;
  using Q = WarpQueue<kStep>;
  constexpr int kQ = Q::kQ;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Q* queues = reinterpret_cast<Q*>(smem_raw);
  const int S = scan.n;
  const int Sp = (S + kStep - 1) / kStep * kStep;
  float4* s_r0 = reinterpret_cast<float4*>(smem_raw + sizeof(Q) * kWarps);  // Sp: mu.xyz, gamma
  float4* s_r1 = s_r0 + Sp;                                                 // Sp: u.xyz, s
  double* s_mu = reinterpret_cast<double*>(s_r1 + Sp);                      // Sp*3
  for (int q = threadIdx.x; q < Sp; q += blockDim.x) {
    s_r0[q] = q < S ? scan.rec[2 * q] : make_float4(0.f, 0.f, 0.f, 0.f);
    s_r1[q] = q < S ? scan.rec[2 * q + 1] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int q = threadIdx.x; q < 3 * Sp; q += blockDim.x)
    s_mu[q] = q < 3 * S ? scan.mu[q] : __longlong_as_double(0x7ff8000000000000ll);
  __syncthreads();

  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t gwarp = static_cast<int64_t>(blockIdx.x) * kWarps + wid;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kWarps;
  const NnfGeom g = map.g;
  float res;
  asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(res) : "d"(g.res));
  const unsigned dx = static_cast<unsigned>(g.dims[0]), dy = static_cast<unsigned>(g.dims[1]),
                 dz = static_cast<unsigned>(g.dims[2]);
  Q& ws = queues[wid];
  unsigned lt_mask;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt_mask));
  // The ring's shared-memory address, opaque to the compiler (otherwise it is
  // rematerialised from the CTA id, thread id and struct size at every use).
  unsigned qaddr;
  asm volatile("mov.u32 %0, %1;" : "=r"(qaddr) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(ws.m0))));

  const int64_t n_eff = list ? static_cast<int64_t>(*list_count) : n;
  for (int64_t it = gwarp; it < n_eff; it += nwarps) {
    const int64_t i = list ? static_cast<int64_t>(list[it]) : it;
    bool huge;
    {  // as k_gicp_fast: lane q < 12 sets up pose word q
      const double pv = __ldg(reinterpret_cast<const double*>(poses + i) + (lane < 12 ? lane : 0));
      const bool isR = lane < 9, isT = lane >= 9 && lane < 12;
      const double o = lane == 9 ? g.origin[0] : (lane == 10 ? g.origin[1] : (lane == 11 ? g.origin[2] : 0.0));
      if (lane < 12) ws.pose_v[lane] = (pv - o) * g.inv_res;
      const float rf = static_cast<float>(pv);
      if (lane < 12) ws.rf[lane] = rf;
      float mr = isR ? fabsf(rf) : 0.f,
            mt = isT ? fabsf(static_cast<float>(pv)) + fabsf(static_cast<float>(o)) : 0.f;
#pragma unroll
      for (int m = 8; m > 0; m >>= 1) {
        mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, m));
        mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, m));
      }
      mr = __shfl_sync(0xffffffffu, mr, 0);
      mt = __shfl_sync(0xffffffffu, mt, 0);
      huge = !((static_cast<double>(mr) * scan.mu_l1_max + static_cast<double>(mt)) * g.inv_res < 6.7e7) ||
             !(pv == pv);
      huge = __any_sync(0xffffffffu, huge);
    }
    __syncwarp();
    Acc acc;
#pragma unroll
    for (int q = 0; q < 6; ++q) acc.hbr[q] = acc.htl[q] = acc.b[q] = 0.f;
#pragma unroll
    for (int q = 0; q < 9; ++q) acc.htr[q] = 0.f;
    acc.cost = 0.f;
    int nmatch = 0;
    int head = 0, pending = 0;  // queue: entries [head, head + pending) mod kQ

    for (int base = 0; base < S; base += kStep) {
      // ---- phase A: fp64 cell + fraction, predicated 256-bit record loads into registers
      float4 rm0[U], rm1[U];
      float fr[U][3];
      bool rsv[U];  // resolving point (reference-order path in phase B)
      {
        double Rv[9], tv[3];
#pragma unroll
        for (int q = 0; q < 9; ++q) Rv[q] = ws.pose_v[q];
#pragma unroll
        for (int a = 0; a < 3; ++a) tv[a] = ws.pose_v[9 + a];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int k = base + u * 32 + lane;
          const double m0 = s_mu[3 * k], m1 = s_mu[3 * k + 1], m2 = s_mu[3 * k + 2];
          unsigned ic[3];
          bool safe = !huge, inb = true;
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) {
            const double x = fma(Rv[ax * 3 + 2], m2, fma(Rv[ax * 3 + 1], m1, fma(Rv[ax * 3 + 0], m0, tv[ax])));
            const CellFrac cf = cell_frac(x);
            ic[ax] = cf.ic;
            inb = inb & (cf.ic < (ax == 0 ? dx : (ax == 1 ? dy : dz)));
            // raw fraction bits: the float is built in phase B, for candidates only
            fr[u][ax] = __uint_as_float(cf.f24);
            safe = safe & cf.clear;
          }
          const bool real = k < S;
          const bool resolve = !safe && real;
          const bool stage = safe && inb && real;
          const float4* src = map.rec + 2 * static_cast<uint64_t>(rec_index<kBrick>(map, ic[0], ic[1], ic[2]));
          ldg_rec_pred(src, stage, rm0[u], rm1[u]);  // unstaged: reads as empty (m0.w = -1)
          rsv[u] = resolve;
        }
      }
      // ---- enqueue the candidates at consecutive positions
      int wpos = head + pending;  // warp-uniform write cursor (mod kQ)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool keep = rsv[u] || rm0[u].w >= 0.f;
        const unsigned mask = __ballot_sync(0xffffffffu, keep);
        int pos = wpos + __popc(mask & lt_mask);
        pos = pos >= kQ ? pos - kQ : pos;
        if (keep) {  // m1, fq at fixed offsets kQ, 2 kQ from m0
          const unsigned a = qaddr + 16u * static_cast<unsigned>(pos);
          const uint32_t meta = static_cast<uint32_t>(base + u * 32 + lane) | (rsv[u] ? kMetaResolve : 0u);
          sts_f4(a, rm0[u]);
          sts_f4(a + 16u * kQ, rm1[u]);
          sts_f4(a + 32u * kQ, make_float4(fr[u][0], fr[u][1], fr[u][2], __uint_as_float(meta)));
        }
        wpos += __popc(mask);
      }
      pending = wpos - head;
      __syncwarp();
      // ---- phase B: full warps; a partial one only at the particle's last step
      const bool last_step = base + kStep >= S;
      const int n_run = last_step ? pending : (pending & ~31);
      float Rf[9];  // per step (registers held through phase B only)
      {
        const float4 r0 = lds_f4_volatile(ws.rf), r1 = lds_f4_volatile(ws.rf + 4), r2 = lds_f4_volatile(ws.rf + 8);
        Rf[0] = r0.x, Rf[1] = r0.y, Rf[2] = r0.z, Rf[3] = r0.w, Rf[4] = r1.x, Rf[5] = r1.y, Rf[6] = r1.z,
        Rf[7] = r1.w, Rf[8] = r2.x;
      }
      for (int b0 = 0; b0 < n_run; b0 += 32) {
        const int e = b0 + lane;
        bool valid = false;
        if (e < n_run) {
          int slot = head + e;
          slot = slot >= kQ ? slot - kQ : slot;
          const unsigned a = qaddr + 16u * static_cast<unsigned>(slot);
          const float4 fq = lds_f4(a + 32u * kQ);
          const uint32_t mt = __float_as_uint(fq.w);
          const int k = static_cast<int>(mt & 0xFFFFu);
          float f3[3] = {frac_of_f24(__float_as_uint(fq.x)), frac_of_f24(__float_as_uint(fq.y)),
                         frac_of_f24(__float_as_uint(fq.z))};
          float4 m0, m1;
          valid = true;
          if (mt & kMetaResolve) {  // exact transform, floor and bounds (nnf.hpp:24-35), direct gather
            const Pose P = poses[i];
            const double mu[3] = {scan.mu[3 * k], scan.mu[3 * k + 1], scan.mu[3 * k + 2]};
            double p[3];
            transform_x(P.R, P.t, mu, p);
            int c3[3];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
              const double x = xmul(xsub(p[ax], g.origin[ax]), g.inv_res);
              const double fl = floor(x);
              valid = valid && (fl >= 0.0 && fl < static_cast<double>(g.dims[ax]));
              c3[ax] = valid ? static_cast<int>(fl) : 0;
              f3[ax] = __double2float_rn(xsub(x, fl));
            }
            const uint64_t c = rec_index<kBrick>(map, c3[0], c3[1], c3[2]);
            m0 = valid ? __ldg(map.rec + 2 * c) : make_float4(0.f, 0.f, 0.f, -1.f);
            m1 = valid ? __ldg(map.rec + 2 * c + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
            m0 = lds_f4(a);
            m1 = lds_f4(a + 16u * kQ);
          }
          valid = valid && m0.w >= 0.f;
          if (valid) fast_item<GN, kCost>(acc, Rf, f3, res, m0, m1, s_r0[k], s_r1[k]);
        }
        nmatch += __popc(__ballot_sync(0xffffffffu, valid));
      }
      head += n_run;
      head = head >= kQ ? head - kQ : head;
      pending -= n_run;
      __syncwarp();
    }

    // ---- epilogue: lane q ends up with the warp total of accumulator q
    if (GN && kSmemRed) {
      // Reduce-scatter through the drained queue (phase B left it empty and
      // ended with __syncwarp): lane l writes its 28 partial sums down column
      // l of a [28][36] table, lane q < 28 sums row q with eight 128-bit
      // loads. 28 stores + 8 loads + 31 adds instead of the butterfly's 31
      // shuffles, 62 selects and 31 adds; both access patterns are
      // bank-conflict free (row stride 36 words).
      constexpr unsigned kRow = 36u * 4u;
      static_assert(28 * 36 * 4 <= 3 * kQ * 16, "reduction table must fit the queue");
      const float v28[28] = {acc.htl[0], acc.htl[1], acc.htl[2], acc.htl[3], acc.htl[4], acc.htl[5],
                             acc.htr[0], acc.htr[1], acc.htr[2], acc.htr[3], acc.htr[4], acc.htr[5],
                             acc.htr[6], acc.htr[7], acc.htr[8], acc.hbr[0], acc.hbr[1], acc.hbr[2],
                             acc.hbr[3], acc.hbr[4], acc.hbr[5], acc.b[0],   acc.b[1],   acc.b[2],
                             acc.b[3],   acc.b[4],   acc.b[5],   acc.cost};
#pragma unroll
      for (int q = 0; q < 28; ++q)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(qaddr + kRow * q + 4u * lane), "f"(v28[q]) : "memory");
      __syncwarp();
      float tot = 0.f;
      if (lane < 28) {
        float4 r[8];
#pragma unroll
        for (int c = 0; c < 8; ++c)
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(r[c].x), "=f"(r[c].y), "=f"(r[c].z), "=f"(r[c].w)
                       : "r"(qaddr + kRow * lane + 16u * c)
                       : "memory");
        float h[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) h[c] = (r[c].x + r[c].y) + (r[c].z + r[c].w);
        tot = ((h[0] + h[1]) + (h[2] + h[3])) + ((h[4] + h[5]) + (h[6] + h[7]));
      }
      sysf[i * kSysF + lane] = tot;
      if (kCost && lane == 27) raw_ll[i] = nmatch == 0 ? -1e30 : -static_cast<double>(tot);
    } else if (GN) {
      float v[32];
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        v[q] = acc.htl[q];
        v[15 + q] = acc.hbr[q];
        v[21 + q] = acc.b[q];
      }
#pragma unroll
      for (int q = 0; q < 9; ++q) v[6 + q] = acc.htr[q];
      v[27] = acc.cost;
      v[28] = v[29] = v[30] = v[31] = 0.f;
#pragma unroll
      for (int s = 16; s >= 1; s >>= 1) {
        const bool up = (lane & s) != 0;
#pragma unroll
        for (int j = 0; j < s; ++j) {
          const float send = up ? v[j] : v[j + s];
          const float keep = up ? v[j + s] : v[j];
          v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
        }
      }
      sysf[i * kSysF + lane] = v[0];
      if (kCost && lane == 27) raw_ll[i] = nmatch == 0 ? -1e30 : -static_cast<double>(v[0]);
    } else {
      const float cost = warp_sum(acc.cost);
      if (lane == 0) raw_ll[i] = nmatch == 0 ? -1e30 : -static_cast<double>(cost);
    }
    if (lane == 0) nm_out[i] = nmatch;  // also under the gate (predicted-live particles skip K2a)
    __syncwarp();
  }
}

// K2 with one lane per particle (likelihood only). The likelihood algebra is
// short (~45 instructions), so running it on every lane for every point that
// matches on ANY lane costs less than compaction and queue traffic; the scan
// point is warp-uniform (broadcast shared-memory reads), each lane gathers its
// own particle's cell record (U points per lane in flight through cp.async).
// Costs are accumulated in fp64 per lane (~S terms, no warp reduction).
// kLdg: records gathered straight into registers with one predicated 256-bit
// load each (no shared-memory stage); else two 16-byte cp.async per record.
template <int U, int kWarps, int kBrick, bool kLdg, int kMinB = 1>
__global__ void __launch_bounds__(kWarps * 32, kMinB) k_gicp_ll_lanes(const Pose* __restrict__ poses, int64_t n,
                                                             ScanView scan, MapFast map,
                                                             double* __restrict__ raw_ll,
                                                             int32_t* __restrict__ nm_out,
                                                             const int32_t* __restrict__ list,
                                                             const unsigned* __restrict__ list_count) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t n_eff = list ? static_cast<int64_t>(*list_count) : n;  // list: the gate's live particles
  if (static_cast<int64_t>(blockIdx.x) * (kWarps * 32) >= n_eff) return;  // block-uniform
  float4* stage = reinterpret_cast<float4*>(smem_raw);  // [kWarps][U][2][32] (cp.async variant)
  const int S = scan.n;
  float4* s_r0 = stage + (kLdg ? 0 : kWarps * U * 2 * 32);  // S: mu.xyz, gamma
  float4* s_r1 = s_r0 + S;                     // S: u.xyz, s
  double* s_mu = reinterpret_cast<double*>(s_r1 + S);
  for (int q = threadIdx.x; q < S; q += blockDim.x) {
    s_r0[q] = scan.rec[2 * q];
    s_r1[q] = scan.rec[2 * q + 1];
  }
  for (int q = threadIdx.x; q < 3 * S; q += blockDim.x) s_mu[q] = scan.mu[q];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * (kWarps * 32) + threadIdx.x;
  const bool active = r < n_eff;
  const int64_t i = active ? (list ? static_cast<int64_t>(list[r]) : r) : 0;
  float4* ws = stage + wid * U * 2 * 32;
  const NnfGeom g = map.g;
  float res;  // kept in a register (otherwise re-converted from the parameter at every matched point)
  asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(res) : "d"(g.res));
  const int nx = g.dims[0], ny = g.dims[1];
  const unsigned dx = static_cast<unsigned>(g.dims[0]), dy = static_cast<unsigned>(g.dims[1]),
                 dz = static_cast<unsigned>(g.dims[2]);
  double Rv[9], tv[3];
  float Rf[9];
  bool huge;
  {  // the pose itself is not kept: the resolve path reloads it
    const Pose P = poses[active ? i : 0];
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      Rv[q] = P.R[q] * g.inv_res;
      Rf[q] = static_cast<float>(P.R[q]);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) tv[a] = (P.t[a] - g.origin[a]) * g.inv_res;
    double mr = 0.0, mt = 0.0;  // resolve bound, as in k_gicp_fast
#pragma unroll
    for (int q = 0; q < 9; ++q) mr = fmax(mr, fabs(P.R[q]));
#pragma unroll
    for (int a = 0; a < 3; ++a) mt = fmax(mt, fabs(P.t[a]) + fabs(g.origin[a]));
    double sum = 0.0;  // NaN-propagating (fmax drops NaN): non-finite poses resolve every point
#pragma unroll
    for (int q = 0; q < 12; ++q) sum += q < 9 ? P.R[q] : P.t[q - 9];
    huge = !((mr * scan.mu_l1_max + mt) * g.inv_res < 6.7e7) || !(sum == sum);
  }
  double cost = 0.0;
  float cpart = 0.f;  // fp32 partial over <= 16 points, folded into the fp64 total (one conversion per 16 points)
  int nmatch = 0;
  for (int base = 0; base < S; base += U) {
    float fr[U][3];
    uint32_t st[U];  // bit 0 staged, bit 1 resolve
    float4 rm0[kLdg ? U : 1], rm1[kLdg ? U : 1];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = base + u;
      const bool real = k < S && active;
      const double m0 = s_mu[3 * (k < S ? k : 0)], m1 = s_mu[3 * (k < S ? k : 0) + 1],
                   m2 = s_mu[3 * (k < S ? k : 0) + 2];
      int ic[3];
      bool safe = !huge, inb = true;
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        const double x = fma(Rv[ax * 3 + 2], m2, fma(Rv[ax * 3 + 1], m1, fma(Rv[ax * 3 + 0], m0, tv[ax])));
        const CellFrac cf = cell_frac(x);
        ic[ax] = static_cast<int>(cf.ic);
        inb = inb & (cf.ic < (ax == 0 ? dx : (ax == 1 ? dy : dz)));
        fr[u][ax] = cf.fr;
        safe = safe & cf.clear;
      }
      const bool amb = !safe;
      const bool stg = real && !amb && inb;
      st[u] = (stg ? 1u : 0u) | (real && amb ? 2u : 0u);
      const uint64_t cell = stg ? rec_index<kBrick>(map, ic[0], ic[1], ic[2]) : 0u;
      const float4* src = map.rec + 2 * cell;
      if (kLdg) {
        ldg_rec_pred(src, stg, rm0[kLdg ? u : 0], rm1[kLdg ? u : 0]);
      } else {
        cp_async16_pred<kBrick != 0>(&ws[(u * 2) * 32 + lane], src, stg);
        cp_async16_pred<kBrick != 0>(&ws[(u * 2 + 1) * 32 + lane], src + 1, stg);
      }
    }
    if (!kLdg) cp_async_wait_all();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = base + u;
      float4 m0 = kLdg ? rm0[kLdg ? u : 0] : ws[(u * 2) * 32 + lane];
      float4 m1 = kLdg ? rm1[kLdg ? u : 0] : ws[(u * 2 + 1) * 32 + lane];
      bool valid = (st[u] & 1u) != 0;
      if (st[u] & 2u) {  // reference-order transform, floor and bounds (nnf.hpp:24-35)
        const Pose P = reload_pose(poses + i);
        const double mu[3] = {s_mu[3 * k], s_mu[3 * k + 1], s_mu[3 * k + 2]};
        double p[3];
        transform_x(P.R, P.t, mu, p);
        int c3[3];
        valid = true;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          const double x = xmul(xsub(p[ax], g.origin[ax]), g.inv_res);
          const double fl = floor(x);
          valid = valid && (fl >= 0.0 && fl < static_cast<double>(g.dims[ax]));
          c3[ax] = valid ? static_cast<int>(fl) : 0;
          fr[u][ax] = __double2float_rn(xsub(x, fl));
        }
        const uint64_t c = rec_index<kBrick>(map, c3[0], c3[1], c3[2]);
        m0 = valid ? __ldg(map.rec + 2 * c) : make_float4(0.f, 0.f, 0.f, -1.f);
        m1 = valid ? __ldg(map.rec + 2 * c + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      valid = valid && m0.w >= 0.f;
      if (valid) {
        Acc a;
        a.cost = 0.f;
        fast_item<false>(a, Rf, fr[u], res, m0, m1, s_r0[k], s_r1[k]);
        cpart += a.cost;
        ++nmatch;
      }
    }
    if (((base / U) & (16 / U - 1)) == 16 / U - 1 || base + U >= S) {  // warp-uniform
      cost += static_cast<double>(cpart);
      cpart = 0.f;
    }
    __syncwarp();
  }
  if (active) {
    raw_ll[i] = nmatch == 0 ? -1e30 : -cost;
    nm_out[i] = nmatch;  // also under the gate (predicted-live particles skip K2a)
  }
}

// max that propagates NaN (fmaxf returns the other operand).
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

__device__ __forceinline__ bool occupied(const MapFast& m, uint32_t r) {
  return (__ldg(m.occ + (r >> 5)) >> (r & 31u)) & 1u;
}

// K2a: n_matched of every particle (lane per particle, occupancy bitmap
// instead of the 32-byte records) and the list of particles the gate keeps.
// The cell decision runs in fp32 with a proven margin and falls back to the
// reference-order fp64 transform (nnf.hpp:24-35) near a face, so n_matched is
// exactly the reference's:
//   x32 = fma(Rv2, mu2, fma(Rv1, mu1, fma(Rv0, mu0, tv))) in fp32, Rv = R / res,
//   tv = (t - o) / res and mu rounded once to fp32 (u = 2^-24 each), differs
//   from the exact x by <= u (5 sum_j |Rv_j| |mu_j| + 4 |tv|) (two input
//   roundings per product, three FMA roundings of partial sums), and the
//   reference's fp64 x differs from the exact one by < 2.2e-8 voxel (k_gicp_fast);
//   a point whose fp32 fraction is farther than that from both faces has the
//   reference's cell. Per particle the margin uses max|Rv| |mu|_1 <= |mu|_1max / res.
// ~1 point in 1000 takes the fp64 path (corridor map, 0.1 m voxels).
template <int kBrick>
__global__ void __launch_bounds__(256, 4) k_ll_count(const Pose* __restrict__ poses, int64_t n, ScanView scan,
                                                     MapFast map, int min_matched, int32_t* __restrict__ nm_out,
                                                     int32_t* __restrict__ live, unsigned* __restrict__ live_count,
                                                     const int32_t* __restrict__ sub,
                                                     const unsigned* __restrict__ sub_count) {
  constexpr int U = 4;  // points in flight per lane
  // sub: count only these particles (the split's predicted-dead ones)
  const int64_t n_eff = sub ? static_cast<int64_t>(*sub_count) : n;
  if (static_cast<int64_t>(blockIdx.x) * blockDim.x >= n_eff) return;  // block-uniform
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float4* s_m = reinterpret_cast<float4*>(smem_raw);  // fp32 mu (scan record .xyz), padded with NaN
  const int S = scan.n;
  const int Sp = (S + U - 1) / U * U;
  for (int q = threadIdx.x; q < Sp; q += blockDim.x) {
    const float nan = __int_as_float(0x7fc00000);
    s_m[q] = q < S ? scan.rec[2 * q] : make_float4(nan, nan, nan, nan);
  }
  __syncthreads();
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = r < n_eff;
  const int64_t i = active ? (sub ? static_cast<int64_t>(sub[r]) : r) : 0;
  const NnfGeom g = map.g;
  const unsigned dx = static_cast<unsigned>(g.dims[0]), dy = static_cast<unsigned>(g.dims[1]),
                 dz = static_cast<unsigned>(g.dims[2]);
  float Rv[9], tv[3];
  int coff[3];  // per-axis cell offset: the particle's own cell coordinate, minus the magic's bits
  float margin;
  {  // the pose itself is not kept: the resolve path reloads it
    const Pose P = poses[active ? i : 0];
    double tmax = 0.0;
    bool fin = true;
#pragma unroll
    for (int q = 0; q < 9; ++q) Rv[q] = static_cast<float>(P.R[q] * g.inv_res);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      // x - 1/2 (its nearest integer is floor(x) away from faces), centred on
      // the integer c = rint((t - o)/res - 1/2): |tv| <= 1/2, so the fp32
      // rounding of the translation term is ~800x smaller than uncentred
      // (corridor map) and fewer points fall inside the margin.
      const double t = (P.t[a] - g.origin[a]) * g.inv_res - 0.5;
      const double c = rint(t);
      fin = fin && fabs(c) < 1.0e9;
      tv[a] = static_cast<float>(t - c);
      coff[a] = (fin ? static_cast<int>(c) : 0) - 0x4B400000;
      tmax = fmax(tmax, fabs(t - c));
    }
    // u (5 |mu|_1max / res + 4 |tv|) + 2.2e-8, x1.25 for the fp64 set-up roundings; |x - c| < 2^21 for the
    // round-to-nearest split below, else (and for non-finite poses) every point takes the fp64 path.
    const double e = 0x1p-24 * (5.0 * scan.mu_l1_max * g.inv_res + 4.0 * tmax) * 1.25 + 2.5e-8;
    margin = (fin && e < 0.01 && tmax + scan.mu_l1_max * g.inv_res < 2097152.0) ? static_cast<float>(e) : 2.0f;
  }
  // 1.5 * 2^23: a round-to-nearest add of x - 1/2 leaves round(x - 1/2) =
  // floor(x) in the low mantissa bits (|x| < 2^21); g = (x - 1/2) - floor(x)
  // = frac(x) - 1/2, so the fraction clears both faces by margin iff
  // max |g| <= 1/2 - margin (NaN fails).
  constexpr float kMagic32 = 12582912.0f;
  const float gmax = 0.5f - margin;
  int nmatch = 0;
  for (int k0 = 0; k0 < Sp; k0 += U) {
    uint32_t rec[U];
    bool ok[U];
    unsigned amb = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float4 m = s_m[k0 + u];
      unsigned ic[3];
      float gabs = 0.0f;
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        const float x = fmaf(Rv[ax * 3 + 2], m.z, fmaf(Rv[ax * 3 + 1], m.y, fmaf(Rv[ax * 3 + 0], m.x, tv[ax])));
        const float y = __fadd_rn(x, kMagic32);
        const float gc = x - (y - kMagic32);
        ic[ax] = __float_as_uint(y) + static_cast<unsigned>(coff[ax]);
        gabs = fmax_nan(gabs, fabsf(gc));
      }
      const bool safe = gabs <= gmax;  // NaN (padded points, non-finite poses) fails
      const bool inb = ic[0] < dx && ic[1] < dy && ic[2] < dz;
      ok[u] = safe && inb;
      rec[u] = ok[u] ? rec_index<kBrick>(map, ic[0], ic[1], ic[2]) : 0u;
      if (!safe && k0 + u < S) amb |= 1u << u;  // padded points (NaN) are never counted
    }
    uint32_t w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) w[u] = ok[u] ? __ldg(map.occ + (rec[u] >> 5)) : 0u;
#pragma unroll
    for (int u = 0; u < U; ++u) nmatch += static_cast<int>((w[u] >> (rec[u] & 31u)) & 1u);
    if (amb) {  // reference-order transform, floor and bounds (nnf.hpp:24-35)
#pragma unroll 1
      for (int u = 0; u < U; ++u) {
        if (!((amb >> u) & 1u)) continue;
        const int k = k0 + u;
        const double mu[3] = {scan.mu[3 * k], scan.mu[3 * k + 1], scan.mu[3 * k + 2]};
        const Pose Pr = reload_pose(poses + (active ? i : 0));
        double p[3];
        transform_x(Pr.R, Pr.t, mu, p);
        bool valid = true;
        unsigned ic[3];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          const double x = xmul(xsub(p[ax], g.origin[ax]), g.inv_res);
          const double fl = floor(x);
          valid = valid && (fl >= 0.0 && fl < static_cast<double>(g.dims[ax]));
          ic[ax] = valid ? static_cast<unsigned>(fl) : 0u;
        }
        nmatch += (valid && occupied(map, rec_index<kBrick>(map, ic[0], ic[1], ic[2]))) ? 1 : 0;
      }
    }
  }
  if (active) nm_out[i] = nmatch;
  const bool keep = active && nmatch >= min_matched;
  const unsigned mask = __ballot_sync(0xffffffffu, keep);
  const int lane = threadIdx.x & 31;
  unsigned base = 0;
  if (lane == 0 && mask) base = atomicAdd(live_count, static_cast<unsigned>(__popc(mask)));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (keep) live[base + __popc(mask & ((1u << lane) - 1u))] = static_cast<int32_t>(i);
}

// Speculative gate split (step only): the GN pass just counted n_matched of
// every particle at its pre-update pose; particles whose count already passes
// the GN pass's gate go straight to the live list (K2 counts them exactly and
// its n_matched and gating decide), the others to K2a. A misprediction only
// costs time: K2 gates exactly on its own count.
// 1024 particles per 256-thread block, one atomic per list per block (a
// same-address atomic per warp had serialised 64 k atomics: 44 us at 1M).
// List order is irrelevant: K2a / K2 write per-particle results.
constexpr int kSplitPer = 4;
__global__ void __launch_bounds__(256) k_ll_split(const int32_t* __restrict__ nm_pred, int64_t n, int thr,
                                                  int32_t* __restrict__ live, unsigned* __restrict__ live_count,
                                                  int32_t* __restrict__ sub, unsigned* __restrict__ sub_count) {
  __shared__ unsigned s_w[8], s_base[2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * 256 * kSplitPer + threadIdx.x;
  bool L[kSplitPer], A[kSplitPer];
  unsigned v = 0;  // live count | sub count << 16 (<= 1024 each)
#pragma unroll
  for (int u = 0; u < kSplitPer; ++u) {
    const int64_t i = b0 + 256 * u;
    A[u] = i < n;
    L[u] = A[u] && nm_pred[i] >= thr;
    v += L[u] ? 1u : (A[u] ? 0x10000u : 0u);
  }
  unsigned incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_w[wid] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const unsigned x = s_w[w];
      s_w[w] = t;  // exclusive warp offsets
      t += x;
    }
    s_base[0] = (t & 0xFFFFu) ? atomicAdd(live_count, t & 0xFFFFu) : 0u;
    s_base[1] = (t >> 16) ? atomicAdd(sub_count, t >> 16) : 0u;
  }
  __syncthreads();
  const unsigned ex = incl - v + s_w[wid];
  unsigned pl = s_base[0] + (ex & 0xFFFFu), ps = s_base[1] + (ex >> 16);
#pragma unroll
  for (int u = 0; u < kSplitPer; ++u) {
    const int32_t i = static_cast<int32_t>(b0 + 256 * u);
    if (L[u])
      live[pl++] = i;
    else if (A[u])
      sub[ps++] = i;
  }
}

__global__ void k_build_occ(const float4* __restrict__ rec, uint64_t n_records, uint32_t* __restrict__ occ) {
  const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool on = r < n_records && rec[2 * r].w >= 0.f;
  const unsigned m = __ballot_sync(0xffffffffu, on);
  if ((threadIdx.x & 31) == 0 && (r >> 5) < (n_records + 31) / 32) occ[r >> 5] = m;
}

template <int U, int W, bool kLdg = false>
size_t ll_lanes_smem(int S) {
  return sizeof(float4) * ((kLdg ? 0 : static_cast<size_t>(W) * U * 2 * 32) + 2 * static_cast<size_t>(S)) +
         sizeof(double) * 3 * static_cast<size_t>(S);
}

// Launch arguments beyond the kernels' common ones: the live-particle list
// of K2a (null: every particle) and whether K1 accumulates the cost.
struct Extra {
  const int32_t* list = nullptr;
  const unsigned* list_count = nullptr;
  bool cost = true;
};

template <int U, int W, bool kLdg, int kMinB = 1>
void launch_ll_lanes_t(const Pose* poses, int64_t n, const ScanView& scan, const MapFast& map, double* raw_ll,
                       int32_t* nm, const Extra& x, cudaStream_t st) {
  const size_t smem = ll_lanes_smem<U, W, kLdg>(scan.n);
  const unsigned grid = static_cast<unsigned>((n + W * 32 - 1) / (W * 32));
  if (map.brick) {
    cudaFuncSetAttribute(k_gicp_ll_lanes<U, W, 1, kLdg, kMinB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    k_gicp_ll_lanes<U, W, 1, kLdg, kMinB><<<grid, W * 32, smem, st>>>(poses, n, scan, map, raw_ll, nm, x.list,
                                                                      x.list_count);
  } else {
    cudaFuncSetAttribute(k_gicp_ll_lanes<U, W, 0, kLdg, kMinB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    k_gicp_ll_lanes<U, W, 0, kLdg, kMinB><<<grid, W * 32, smem, st>>>(poses, n, scan, map, raw_ll, nm, x.list,
                                                                      x.list_count);
  }
}

template <int U, int W>
size_t fast_smem(int S) {
  const size_t Sp = static_cast<size_t>((S + 32 * U - 1) / (32 * U) * (32 * U));
  return sizeof(WarpStage<32 * U>) * W + sizeof(float4) * 2 * Sp + sizeof(double) * 3 * Sp;
}

template <bool GN, int U, int W, int B, bool L, bool C>
void launch_fast_tblc(const Pose* poses, int64_t n, const ScanView& scan, const MapFast& map, float* sysf,
                      double* raw_ll, int32_t* nm, const Extra& x, cudaStream_t st) {
  const size_t smem = fast_smem<U, W>(scan.n);
  int dev, n_sm, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(k_gicp_fast<GN, U, W, B, L, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gicp_fast<GN, U, W, B, L, C>, W * 32, smem);
  const int64_t want = (n + W - 1) / W;
  const unsigned grid =
      static_cast<unsigned>(std::min<int64_t>(want, static_cast<int64_t>(n_sm) * std::max(per_sm, 1)));
  k_gicp_fast<GN, U, W, B, L, C><<<grid, W * 32, smem, st>>>(poses, n, scan, map, sysf, raw_ll, nm, x.list,
                                                              x.list_count);
}

template <bool GN, int U, int W, int B, bool L>
void launch_fast_tbl(const Pose* poses, int64_t n, const ScanView& scan, const MapFast& map, float* sysf,
                     double* raw_ll, int32_t* nm, const Extra& x, cudaStream_t st) {
  (GN && !x.cost) ? launch_fast_tblc<GN, U, W, B, L, false>(poses, n, scan, map, sysf, raw_ll, nm, x, st)
                  : launch_fast_tblc<GN, U, W, B, L, true>(poses, n, scan, map, sysf, raw_ll, nm, x, st);
}

template <bool GN, int U, int W, int B>
void launch_fast_tb(const Pose* poses, int64_t n, const ScanView& scan, const MapFast& map, float* sysf,
                    double* raw_ll, int32_t* nm, const Extra& x, cudaStream_t st) {
  // Record gathers: the GN pass keeps cp.async (issue bound: 4.57 ms against
  // 5.25 with 256-bit loads + shared stores); the likelihood-only warp variant
  // (bricked HBM-sized tables) gathers with 256-bit loads (outdoor kidnap LL
  // 2.49-2.72 ms against 2.82-2.88; HBM cp.async gathers measure 0.73 TB/s
  // against 1.34 for loads).
  static const bool ldg = GN ? std::getenv("SMCL_K1_LDG") != nullptr : std::getenv("SMCL_K2W_CPASYNC") == nullptr;
  ldg ? launch_fast_tbl<GN, U, W, B, true>(poses, n, scan, map, sysf, raw_ll, nm, x, st)
      : launch_fast_tbl<GN, U, W, B, false>(poses, n, scan, map, sysf, raw_ll, nm, x, st);
}

template <bool GN, int U, int W>
void launch_fast_t(const Pose* poses, int64_t n, const ScanView& scan, const MapFast& map, float* sysf, double* raw_ll,
                   int32_t* nm, const Extra& x, cudaStream_t st) {
  map.brick ? launch_fast_tb<GN, U, W, 1>(poses, n, scan, map, sysf, raw_ll, nm, x, st)
            : launch_fast_tb<GN, U, W, 0>(poses, n, scan, map, sysf, raw_ll, nm, x, st);
}

}  // namespace

template <int U, int W>
size_t fast_q_smem(int S) {
  const size_t Sp = static_cast<size_t>((S + 32 * U - 1) / (32 * U) * (32 * U));
  return sizeof(WarpQueue<32 * U>) * W + sizeof(float4) * 2 * Sp + sizeof(double) * 3 * Sp;
}
template <bool GN, int U, int W>
bool launch_fast_q(const Pose* poses, int64_t n, const ScanView& scan, const MapFast& map, float* sysf,
                   double* raw_ll, int32_t* nm, const Extra& x, cudaStream_t st) {
  const size_t smem = fast_q_smem<U, W>(scan.n);
  if (smem > 227 * 1024) return false;
  int dev, n_sm, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  auto run = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W * 32, smem);
    const int64_t want = (n + W - 1) / W;
    const unsigned grid =
        static_cast<unsigned>(std::min<int64_t>(want, static_cast<int64_t>(n_sm) * std::max(per_sm, 1)));
    kern<<<grid, W * 32, smem, st>>>(poses, n, scan, map, sysf, raw_ll, nm, x.list, x.list_count);
  };
  if (map.brick) return false;  // plain-layout tables only (see launch_gicp_fast)
  static const bool shfl_red = std::getenv("SMCL_K1_SHFL_RED") != nullptr;  // A/B: butterfly epilogue
  if (GN && !x.cost)
    shfl_red ? run(k_gicp_fast_q<GN, U, W, false, 0, false>) : run(k_gicp_fast_q<GN, U, W, false, 0, true>);
  else
    run(k_gicp_fast_q<GN, U, W, true, 0>);
  return true;
}

// A staged-slot configuration requested for the GN pass (SMCL_FAST_CFG_GN /
// SMCL_FAST_CFG): the queue variant stands aside.
static int cfg_gn_override() {
  static const int v = (std::getenv("SMCL_FAST_CFG_GN") || std::getenv("SMCL_FAST_CFG")) ? 1 : 0;
  return v;
}

// U points per lane in flight x W warps per SM (one CTA per SM).
// SMCL_FAST_CFG=UxW overrides the default (tuning sweeps only).
void launch_gicp_fast(bool gn, const Pose* poses, int64_t n, const ScanView& scan, const MapFast& map, float* sysf,
                      double* raw_ll, int32_t* nm, bool need_cost, int min_matched, int32_t* live_list,
                      unsigned* live_count, cudaStream_t st, int pred_thr, int32_t* sub_list, unsigned* sub_count) {
  count_launch();
  if (n <= 0) return;
  Extra x;
  x.cost = need_cost;
  static const bool no_gate = std::getenv("SMCL_NO_LL_GATE") != nullptr;  // experiments: K2 on every particle
  static const bool no_split = std::getenv("SMCL_NO_LL_SPLIT") != nullptr;  // experiments: K2a on every particle
  if (!gn && min_matched > 0 && map.occ && scan.rec && live_list && live_count && !no_gate) {
    // K2a: n_matched of every particle + the list the gate keeps; K2 then
    // evaluates the cost of those particles only. With a prediction (nm holds
    // the GN pass's counts, pred_thr its gate), predicted-live particles skip
    // K2a (k_ll_split) and K2 counts them exactly.
    count_launch();
    const bool split = pred_thr > 0 && sub_list && sub_count && !no_split;

    cudaMemsetAsync(live_count, 0, sizeof(unsigned), st);
    if (split) {
      count_launch();
      cudaMemsetAsync(sub_count, 0, sizeof(unsigned), st);
      k_ll_split<<<static_cast<unsigned>((n + 256 * kSplitPer - 1) / (256 * kSplitPer)), 256, 0, st>>>(
          nm, n, pred_thr, live_list, live_count, sub_list, sub_count);
    }
    const int32_t* sub = split ? sub_list : nullptr;
    const unsigned* sc = split ? sub_count : nullptr;
    const size_t smem = sizeof(float4) * static_cast<size_t>((scan.n + 3) / 4 * 4);
    const unsigned grid = static_cast<unsigned>((n + 255) / 256);
    if (map.brick) {
      cudaFuncSetAttribute(k_ll_count<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      k_ll_count<1><<<grid, 256, smem, st>>>(poses, n, scan, map, min_matched, nm, live_list, live_count, sub, sc);
    } else {
      cudaFuncSetAttribute(k_ll_count<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      k_ll_count<0><<<grid, 256, smem, st>>>(poses, n, scan, map, min_matched, nm, live_list, live_count, sub, sc);
    }
    x.list = live_list;
    x.list_count = live_count;
    static const bool stats = std::getenv("SMCL_LL_SPLIT_STATS") != nullptr;  // diagnostics: list sizes (syncs)
    if (stats) {
      unsigned h[2] = {0, 0};
      cudaMemcpyAsync(&h[0], live_count, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
      if (split) cudaMemcpyAsync(&h[1], sub_count, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      std::fprintf(stderr, "[ll-gate] n %lld live %u counted by K2a %u\n", static_cast<long long>(n), h[0],
                   split ? h[1] : static_cast<unsigned>(n));
    }
  }
  auto parse = [](const char* e) {
    if (!e) return 0;
    int u = 0, w = 0;
    if (std::sscanf(e, "L%dx%d", &u, &w) == 2) return 9000 + u * 100 + w;  // lane-per-particle likelihood
    return std::sscanf(e, "%dx%d", &u, &w) == 2 ? u * 100 + w : 0;
  };
  // GN pass on plain-layout (L2-resident) tables: the queue variant, 4 points
  // per lane x 20 warps per SM (GN 3.74 ms at 1M x 512 against 3.98 for the
  // staged-slot kernel at 4 x 24; queue 2 x 28: 3.74, 2 x 24: 3.90, 4 x 16:
  // 3.96, 4 x 18: 4.06, 4 x 24 spills: 4.78). SMCL_K1_QUEUE=UxW overrides,
  // =0 takes the staged-slot kernel.
  static const int q_cfg = [] {
    const char* e = std::getenv("SMCL_K1_QUEUE");
    int u = 0, w = 0;
    if (!e) return 420;
    return std::sscanf(e, "%dx%d", &u, &w) == 2 ? u * 100 + w : 0;
  }();
  // Bricked (HBM-sized) tables keep the staged-slot kernel: there the pass is
  // bound by HBM gathers and the queue variant measured the same (kidnap GN
  // 6.76 vs 6.77 ms at 16 warps/SM, 7.02 at 20).
  if (gn && q_cfg && cfg_gn_override() == 0 && !map.brick) {
    bool done = false;
    switch (q_cfg) {
      case 420: done = launch_fast_q<true, 4, 20>(poses, n, scan, map, sysf, raw_ll, nm, x, st); break;
      case 416: done = launch_fast_q<true, 4, 16>(poses, n, scan, map, sysf, raw_ll, nm, x, st); break;
      case 224: done = launch_fast_q<true, 2, 24>(poses, n, scan, map, sysf, raw_ll, nm, x, st); break;
      case 228: done = launch_fast_q<true, 2, 28>(poses, n, scan, map, sysf, raw_ll, nm, x, st); break;
      default: break;
    }
    if (done) return;
  }
  static const int cfg_gn = parse(std::getenv("SMCL_FAST_CFG_GN") ? std::getenv("SMCL_FAST_CFG_GN")
                                                                   : std::getenv("SMCL_FAST_CFG"));
  static const int cfg_ll = parse(std::getenv("SMCL_FAST_CFG_LL") ? std::getenv("SMCL_FAST_CFG_LL")
                                                                   : std::getenv("SMCL_FAST_CFG"));
  const int cfg = gn ? cfg_gn : cfg_ll;
  // Measured on B200 at 1M x 512 (profiles/README.md): GN pass 4.77 ms with
  // 16 warps per SM, 4.57 ms with 24 (4x20: 4.63, 4x28 / 4x32 spill).
  // Likelihood pass: lane per particle when the record table is L2-resident;
  // for bricked (HBM-sized) tables a warp walks one particle's scan so its
  // gathers stay inside a few bricks (kidnap outdoor map: 4.8 -> 2.4 ms).
  int c = cfg;
  // The lane kernel needs two resident CTAs per SM (16 warps): scans too large
  // for that (S > ~900 points) take the warp-per-particle kernel as well.
  if (!gn && c == 0) c = (map.brick || 3 * ll_lanes_smem<1, 8, true>(scan.n) > 227 * 1024) ? 416 : 9000;
  // GN pass: 20 warps per SM (96 registers, no spills; 24 warps at 80
  // registers spill: 4.58 ms against 4.42 at 1M x 512) where the scan fits in
  // shared memory next to 20 warp stages (S <= ~1700), else 16. Bricked
  // (HBM-sized) tables keep 16 warps: their L1-allocating gathers need the L1
  // that more warp stages would take (outdoor kidnap GN 2.43 -> 2.31 ms, LL
  // 2.55 -> 2.32).
  if (c == 0 && gn && !map.brick) c = fast_smem<4, 24>(scan.n) <= 227 * 1024 ? 424
                                     : (fast_smem<4, 20>(scan.n) <= 227 * 1024 ? 420 : 416);
  if (c == 0) c = 416;
  if (c >= 9000) {  // SMCL_FAST_CFG=LUxW: lane-per-particle variants (9000 = default)
    static const bool ldg = std::getenv("SMCL_LL_CPASYNC") == nullptr;
    // Default: one record in flight per lane, 8-warp CTAs, 4 CTAs (32 warps)
    // per SM: 2.79 ms at 1M x 512 (cp.async 8 x 8: 3.43; LDG 2 x 8: 2.91;
    // 4 x 8: 3.23; 1 x 8 at 5 / 6 CTAs spills: 3.33 / 3.42).
    if (c == 9000) {  // 3 CTAs per SM when 4 do not fit next to the scan (S > ~1000)
      // The gated pass (x.list) needs the list indirection's registers: 3 CTAs
      // (80 registers) with two records in flight per lane (LL 2.20 -> 2.02 ms
      // at 1M x 512; one record: 2.20, three / four spill: 2.30 / 2.48, two at
      // 2 CTAs / 104 registers: 2.17).
      static const bool minb3 = std::getenv("SMCL_LL_MINB3") != nullptr;
      if (!minb3 && !x.list && 4 * ll_lanes_smem<1, 8, true>(scan.n) <= 227 * 1024)
        launch_ll_lanes_t<1, 8, true, 4>(poses, n, scan, map, raw_ll, nm, x, st);
      else if (x.list)
        launch_ll_lanes_t<2, 8, true, 3>(poses, n, scan, map, raw_ll, nm, x, st);
      else
        launch_ll_lanes_t<1, 8, true, 3>(poses, n, scan, map, raw_ll, nm, x, st);
      return;
    }
    const int u = (c / 100) % 10, w = c % 100;
#define LL_CASE(UU, WW)                                                                         \
    if (!gn && u == UU && w == WW && ll_lanes_smem<UU, WW>(scan.n) <= 227 * 1024) {            \
      ldg ? launch_ll_lanes_t<UU, WW, true>(poses, n, scan, map, raw_ll, nm, x, st)               \
          : launch_ll_lanes_t<UU, WW, false>(poses, n, scan, map, raw_ll, nm, x, st);             \
      return;                                                                                  \
    }
    LL_CASE(8, 8)
    LL_CASE(4, 8)
    LL_CASE(2, 8)
    LL_CASE(2, 16)
    LL_CASE(3, 8)
#undef LL_CASE
    if (!gn && u >= 1 && u <= 4 && w >= 80) {  // SMCL_FAST_CFG_LL=L2x84 / L1x84: 8 warps, >= 4 CTAs per SM
      const int mb = w - 80;
      if (u == 2 && mb == 3) return launch_ll_lanes_t<2, 8, true, 3>(poses, n, scan, map, raw_ll, nm, x, st);
      if (u == 3 && mb == 3) return launch_ll_lanes_t<3, 8, true, 3>(poses, n, scan, map, raw_ll, nm, x, st);
      if (u == 4 && mb == 3) return launch_ll_lanes_t<4, 8, true, 3>(poses, n, scan, map, raw_ll, nm, x, st);
      if (u == 2 && mb == 2) return launch_ll_lanes_t<2, 8, true, 2>(poses, n, scan, map, raw_ll, nm, x, st);
      if (u == 2 && mb == 4) return launch_ll_lanes_t<2, 8, true, 4>(poses, n, scan, map, raw_ll, nm, x, st);
      if (u == 2 && mb == 5) return launch_ll_lanes_t<2, 8, true, 5>(poses, n, scan, map, raw_ll, nm, x, st);
      if (u == 1 && mb == 2) return launch_ll_lanes_t<1, 8, true, 2>(poses, n, scan, map, raw_ll, nm, x, st);
      if (u == 1 && mb == 4) return launch_ll_lanes_t<1, 8, true, 4>(poses, n, scan, map, raw_ll, nm, x, st);
      if (u == 1 && mb == 5) return launch_ll_lanes_t<1, 8, true, 5>(poses, n, scan, map, raw_ll, nm, x, st);
      if (u == 1 && mb == 6) return launch_ll_lanes_t<1, 8, true, 6>(poses, n, scan, map, raw_ll, nm, x, st);
    }
    if (!gn && u == 1 && w >= 40 && w < 80) {  // L1x4M: 4 warps per CTA, >= M CTAs per SM
      const int mb = w - 40;
      if (mb == 8) return launch_ll_lanes_t<1, 4, true, 8>(poses, n, scan, map, raw_ll, nm, x, st);
      if (mb == 10) return launch_ll_lanes_t<1, 4, true, 10>(poses, n, scan, map, raw_ll, nm, x, st);
      if (mb == 12) return launch_ll_lanes_t<1, 4, true, 12>(poses, n, scan, map, raw_ll, nm, x, st);
    }
    c = gn ? 416 : 424;
  }
#define FAST_CASE(U, W)                                                                    \
  case U * 100 + W:                                                                        \
    if (fast_smem<U, W>(scan.n) <= 227 * 1024) {                                           \
      gn ? launch_fast_t<true, U, W>(poses, n, scan, map, sysf, raw_ll, nm, x, st)            \
         : launch_fast_t<false, U, W>(poses, n, scan, map, sysf, raw_ll, nm, x, st);          \
      return;                                                                              \
    }                                                                                      \
    break;
  switch (c) {
    FAST_CASE(8, 14)
    FAST_CASE(4, 16)
    FAST_CASE(4, 20)
    FAST_CASE(4, 24)
    FAST_CASE(4, 32)
    FAST_CASE(2, 32)
    default:
      break;
  }
#undef FAST_CASE
  gn ? launch_fast_t<true, 4, 16>(poses, n, scan, map, sysf, raw_ll, nm, x, st)
     : launch_fast_t<false, 4, 16>(poses, n, scan, map, sysf, raw_ll, nm, x, st);
}

void launch_build_occupancy(const float4* rec, uint64_t n_records, uint32_t* occ, cudaStream_t st) {
  count_launch();
  if (n_records == 0) return;
  k_build_occ<<<static_cast<unsigned>((n_records + 255) / 256), 256, 0, st>>>(rec, n_records, occ);
}

}  // namespace smcl
