// Device-side data layout and kernel entry points of the B200 Stein-particle
// filter. See DESIGN.md §Data layout for the HBM picture.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "smcl_math.cuh"

namespace smcl {

constexpr int kMaxK = 32;          // neighbour-list capacity supported on device
constexpr int kMaxScan = 4096;     // scan points per frame (n_scan_max is 1000 by default)
constexpr int kReduceChunk = 4096; // reduce.hpp:14 k_reduce_chunk

// Nearest-neighbour field geometry (nnf.hpp:13-35).
struct NnfGeom {
  double origin[3];
  double inv_res;  // 1.0 / resolution, exactly as nnf.hpp:25 computes it
  double res;
  int dims[3];
};

// Exact-mode map: NNF index cells + fp64 map Gaussians (reference layout).
struct MapExact {
  NnfGeom g;
  const int32_t* cells;
  const double* mu;     // M*3
  const double* sigma;  // M*9
};

// Fast-mode map: one 32-byte record per NNF cell (denormalised cell -> map
// Gaussian), structured covariance Sigma = beta*(I - u u^T) + s*u u^T... stored as
//   rec[2c+0] = (mu - corner(c)).xyz, beta      (beta < 0: empty cell)
//   rec[2c+1] = u.xyz, s
// with beta = a - s >= 0 (a: double eigenvalue, s: single eigenvalue, u its axis).
struct MapFast {
  NnfGeom g;
  const float4* rec;
};

// Per-frame scan in both precisions. Fast records: (mu.xyz, gamma), (u.xyz, s).
struct ScanView {
  int n;
  const double* mu;     // n*3 fp64 (exact transform input)
  const double* sigma;  // n*9 fp64 (exact mode)
  const float4* rec;    // n*2 (fast mode, may be null)
  double mu_l1_max;     // max_k |mu_k|_1, for the fp32 prefilter error bound
};

// Particle-point GN system accumulators as written by the likelihood kernels:
// 36 (H row-major, lower triangle authoritative) + 6 (b) + ll_raw.
constexpr int kSysStride = 43;

struct GicpParamsDev {
  double damping_scale, omega_max, v_max, miss_cost;
  int min_matched;
  int scan_size;
};

// ---------------------------------------------------------------- launchers
// likelihood.cu
void launch_gicp_exact(bool gn, const Pose* poses, int64_t n, const ScanView& scan, const MapExact& map,
                       double* sys, int32_t* nm, cudaStream_t st);
void launch_gicp_fast(bool gn, const Pose* poses, int64_t n, const ScanView& scan, const MapFast& map, double* sys,
                      int32_t* nm, cudaStream_t st);
void launch_solve(const double* sys, const int32_t* nm, int64_t n, const GicpParamsDev& p, double* steps, double* ll,
                  cudaStream_t st);
void launch_gate_ll(const double* sys, const int32_t* nm, int64_t n, const GicpParamsDev& p, double* ll,
                    cudaStream_t st);
void launch_solve_batch(const double* H, const double* b, const double* lam, int64_t n, double omax, double vmax,
                        double* out, cudaStream_t st);

}  // namespace smcl
