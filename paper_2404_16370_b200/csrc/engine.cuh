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
// Record table layout: x-fastest cells (tables that fit in L2), or 4x4x4-cell
// bricks (64 records = 2 KB contiguous, bricks x-fastest) for tables larger
// than L2: scan points that land close together share bricks, so their
// gathers share L2 lines and DRAM pages (outdoor map: 7 GB table, K1 4.1 ->
// 2.5 ms; for the L2-resident corridor table the extra index math costs more
// than it saves).
struct MapFast {
  NnfGeom g;
  const float4* rec;
  int brick = 0;
  // Occupancy bitmap by record index (bit r: record r is a map Gaussian),
  // the likelihood pass's match-count prepass (K2a): 191 KB for the corridor
  // map, mostly L1-resident.
  const uint32_t* occ = nullptr;
  // One always-empty record (beta = -1): the target of unmatched gathers, so
  // they need no predication.
  const float4* empty = nullptr;
  // Host-side / map-build slot; the likelihood kernels use rec_index<kBrick>.
  // 32-bit index math: the NNF budget (2^30 cells) keeps every table < 2^32 records.
  __host__ __device__ __forceinline__ uint32_t index(uint32_t ix, uint32_t iy, uint32_t iz) const {
    const uint32_t nx = static_cast<uint32_t>(g.dims[0]), ny = static_cast<uint32_t>(g.dims[1]);
    if (!brick) return (iz * ny + iy) * nx + ix;
    const uint32_t b = ((iz >> 2) * ((ny + 3u) >> 2) + (iy >> 2)) * ((nx + 3u) >> 2) + (ix >> 2);
    return (b << 6) | ((iz & 3u) << 4) | ((iy & 3u) << 2) | (ix & 3u);
  }
  static uint64_t n_records(const int dims[3], int brick) {
    if (!brick) return static_cast<uint64_t>(dims[0]) * dims[1] * dims[2];
    return static_cast<uint64_t>((dims[0] + 3) >> 2) * ((dims[1] + 3) >> 2) * ((dims[2] + 3) >> 2) * 64u;
  }
  // Brick layout when the linear table exceeds 64 MB (half the B200 L2).
  static int choose_brick(const int dims[3]) { return n_records(dims, 0) * 32u > (uint64_t(64) << 20) ? 1 : 0; }
};

// Per-frame scan in both precisions. Fast records: (mu.xyz, gamma), (u.xyz, s).
struct ScanView {
  int n;
  const double* mu;     // n*3 fp64 (exact transform input)
  const double* sigma;  // n*9 fp64 (exact mode)
  const float4* rec;    // n*2 (fast mode, may be null)
  double mu_l1_max;     // max_k |mu_k|_1, for the fp32 prefilter error bound
};

// Per-particle GN system as written by the exact likelihood kernel: 36 (H
// row-major) + 6 (b), fp64. The raw log-likelihood goes to its own array.
constexpr int kSysStride = 42;
// The fast kernel's record: its 27 fp32 accumulators (H lower triangle, b) and
// the cost in lane order, padded to one 128-byte line per particle; the solve
// widens them to fp64 exactly as the kernel's own conversion would.
constexpr int kSysF = 32;
// Lane q of the fast record -> offset in the 42-entry (H row-major, b) system.
// htl -> H(r, c), c <= r < 3; htr(r, c) -> H(c+3, r); hbr -> H(r+3, c+3); b.
#define SMCL_FAST_SYS_OFF                                                                                   \
  {0, 6, 7, 12, 13, 14, 18, 24, 30, 19, 25, 31, 20, 26, 32, 21, 27, 28, 33, 34, 35, 36, 37, 38, 39, 40, 41}

struct GicpParamsDev {
  double damping_scale, omega_max, v_max, miss_cost;
  int min_matched;
  int scan_size;
};

// ---------------------------------------------------------------- launchers
// likelihood.cu
void launch_gicp_exact(bool gn, const Pose* poses, int64_t n, const ScanView& scan, const MapExact& map,
                       double* sys, double* raw_ll, int32_t* nm, cudaStream_t st);
// Fast (plane-model) likelihood passes.
// gn: K1, the Gauss-Newton system into sysf (need_cost: also the raw
//     log-likelihood; FilterEngine::step discards the GN pass's likelihood,
//     filter.cpp:166-187, so the step skips it).
// !gn: K2, raw log-likelihood + n_matched. With min_matched > 0 and the map's
//     occupancy bitmap, K2a counts every particle's matches first and the
//     cost is evaluated only for particles the gate keeps (n >= min_matched,
//     gicp.cpp:79-85): the others' likelihood is the sentinel whatever their
//     cost. live_list (n) / live_count (1) are scratch.
// pred_thr > 0 (with sub_list / sub_count): nm holds a prediction of this
// pass's n_matched (the GN pass's counts); particles at or above pred_thr go
// straight to the likelihood kernel, the others through the K2a count.
void launch_gicp_fast(bool gn, const Pose* poses, int64_t n, const ScanView& scan, const MapFast& map, float* sysf,
                      double* raw_ll, int32_t* nm, bool need_cost, int min_matched, int32_t* live_list,
                      unsigned* live_count, cudaStream_t st, int pred_thr = 0, int32_t* sub_list = nullptr,
                      unsigned* sub_count = nullptr);
void launch_build_occupancy(const float4* rec, uint64_t n_records, uint32_t* occ, cudaStream_t st);
// Exactly one of sys (exact record) / sysf (fast record) is non-null.
void launch_solve(const double* sys, const float* sysf, const double* raw_ll, const int32_t* nm, int64_t n,
                  const GicpParamsDev& p, double* steps, double* ll, cudaStream_t st,
                  unsigned long long* nm_sum = nullptr);
void launch_gate_ll(const double* raw_ll, const int32_t* nm, int64_t n, const GicpParamsDev& p, double* ll,
                    cudaStream_t st, unsigned long long* counts = nullptr);
void launch_solve_batch(const double* H, const double* b, const double* lam, int64_t n, double omax, double vmax,
                        double* out, cudaStream_t st);

}  // namespace smcl
