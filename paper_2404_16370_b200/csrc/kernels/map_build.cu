// Device map load: the nearest-neighbour field and the
// denormalised fast-map records built on the GPU instead of the host.
//
// Reference: build_nnf (nnf.cpp:10-96) = occupancy of the point cells, a BFS
// of hop_cap = ceil(max_query_dist / res) + 2 Chebyshev hops around them
// (nnf.cpp:37-80), then PointBucketGrid::nearest_within at every reached cell
// centre (nnf.cpp:82-94, point_grid.cpp:109-141). Here:
//   1. point grid (point_grid.cpp:10-49): cell id per map point, a stable CUB
//      radix sort of (cell, index) -> CSR order with ascending indices inside
//      a cell, counts + exclusive scan -> offsets;
//   2. NNF occupancy, then three separable Chebyshev dilations (the BFS
//      reaches exactly the cells within hop_cap in the max norm);
//   3. one thread per NNF cell: the reference's ring search (same rings, same
//      early exit, ties to the lower index) -> cells[c];
//   4. one thread per NNF cell: the 32-byte fast record (engine.cu setup_map
//      layout) from the per-point plane-model parameters.
// Every arithmetic step follows the host/reference operation order without
// contraction (__dadd_rn/__dmul_rn/__ddiv_rn), so cells are bit-identical to
// the host build (tests/test_gpu_map.py).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>

#include "../engine.cuh"
#include "../kernels.cuh"

namespace smcl {

namespace {

#define MB_CK(x)                  \
  do {                            \
    const cudaError_t e_ = (x);   \
    if (e_ != cudaSuccess) return e_; \
  } while (0)

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// static_cast<int>(std::floor((p - o) / cell)), clamped to [0, dims).
__device__ __forceinline__ int cell_coord(double p, double o, double cell, int dim) {
  return clampi(static_cast<int>(floor(__ddiv_rn(__dsub_rn(p, o), cell))), 0, dim - 1);
}

struct GridDev {
  double org[3];
  double cell;
  int dims[3];
};

// point_grid.cpp:10-49: flat cell id of every map point.
__global__ void k_point_cells(const double* __restrict__ mu, int64_t n, GridDev g, int32_t* __restrict__ cid,
                              int32_t* __restrict__ iota, int32_t* __restrict__ counts) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) c[a] = cell_coord(mu[3 * i + a], g.org[a], g.cell, g.dims[a]);
  const int32_t id = (c[2] * g.dims[1] + c[1]) * g.dims[0] + c[0];
  cid[i] = id;
  iota[i] = static_cast<int32_t>(i);
  atomicAdd(counts + id, 1);
}

// nnf.cpp:40-60: cells holding a map point.
__global__ void k_nnf_occupancy(const double* __restrict__ mu, int64_t n, GridDev g, uint8_t* __restrict__ occ) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) c[a] = cell_coord(mu[3 * i + a], g.org[a], g.cell, g.dims[a]);
  occ[(static_cast<int64_t>(c[2]) * g.dims[1] + c[1]) * g.dims[0] + c[0]] = 1;
}

// One axis of the Chebyshev dilation by `hop` cells.
__global__ void k_dilate(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t n_cells, int nx, int ny,
                         int nz, int axis, int hop) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= n_cells) return;
  const int x = static_cast<int>(c % nx);
  const int y = static_cast<int>((c / nx) % ny);
  const int z = static_cast<int>(c / (static_cast<int64_t>(nx) * ny));
  const int pos = axis == 0 ? x : (axis == 1 ? y : z);
  const int len = axis == 0 ? nx : (axis == 1 ? ny : nz);
  const int64_t stride = axis == 0 ? 1 : (axis == 1 ? nx : static_cast<int64_t>(nx) * ny);
  const int lo = max(pos - hop, 0), hi = min(pos + hop, len - 1);
  uint8_t v = 0;
  for (int q = lo; q <= hi && !v; ++q) v = src[c + static_cast<int64_t>(q - pos) * stride];
  dst[c] = v;
}

// point_grid.cpp:109-141 at the centre of every reached NNF cell (nnf.cpp:82-94).
__global__ void k_nnf_query(const uint8_t* __restrict__ reach, int64_t n_cells, GridDev nnf, double max_dist,
                            GridDev pg, const int32_t* __restrict__ offsets, const int32_t* __restrict__ order,
                            const double* __restrict__ mu, int32_t* __restrict__ cells) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= n_cells) return;
  if (!reach[c]) {
    cells[c] = -1;
    return;
  }
  const int nx = nnf.dims[0], ny = nnf.dims[1];
  const int x = static_cast<int>(c % nx);
  const int y = static_cast<int>((c / nx) % ny);
  const int z = static_cast<int>(c / (static_cast<int64_t>(nx) * ny));
  const double q[3] = {__dadd_rn(nnf.org[0], __dmul_rn(nnf.cell, static_cast<double>(x) + 0.5)),
                       __dadd_rn(nnf.org[1], __dmul_rn(nnf.cell, static_cast<double>(y) + 0.5)),
                       __dadd_rn(nnf.org[2], __dmul_rn(nnf.cell, static_cast<double>(z) + 0.5))};
  int c0[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) c0[a] = cell_coord(q[a], pg.org[a], pg.cell, pg.dims[a]);
  const int r_cap = static_cast<int>(ceil(__ddiv_rn(max_dist, pg.cell))) + 1;
  double best2 = __dmul_rn(max_dist, max_dist);
  int32_t best = -1;
  for (int r = 0; r <= r_cap; ++r) {
    const double lb = __dmul_rn(static_cast<double>(r - 1), pg.cell);
    if (lb > 0.0 && __dmul_rn(lb, lb) > best2) break;
    const int z0 = max(c0[2] - r, 0), z1 = min(c0[2] + r, pg.dims[2] - 1);
    const int y0 = max(c0[1] - r, 0), y1 = min(c0[1] + r, pg.dims[1] - 1);
    const int x0 = max(c0[0] - r, 0), x1 = min(c0[0] + r, pg.dims[0] - 1);
    for (int zz = z0; zz <= z1; ++zz)
      for (int yy = y0; yy <= y1; ++yy) {
        const bool yz_shell = abs(zz - c0[2]) == r || abs(yy - c0[1]) == r;
        // Off the y/z shell only the two x faces belong to ring r.
        const int step = yz_shell ? 1 : max(2 * r, 1);
        for (int xx = yz_shell ? x0 : c0[0] - r; xx <= x1; xx += step) {
          if (xx < x0) continue;
          const int64_t ci = (static_cast<int64_t>(zz) * pg.dims[1] + yy) * pg.dims[0] + xx;
          for (int32_t j = offsets[ci]; j < offsets[ci + 1]; ++j) {
            const int32_t idx = order[j];
            const double dx = __dsub_rn(mu[3 * idx], q[0]), dy = __dsub_rn(mu[3 * idx + 1], q[1]),
                         dz = __dsub_rn(mu[3 * idx + 2], q[2]);
            const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
            if (d2 < best2 || (d2 == best2 && best >= 0 && idx < best)) {
              best2 = d2;
              best = idx;
            }
          }
        }
      }
  }
  cells[c] = best;
}

// Fast-map record of every cell: ((mu - corner).xyz, beta), (u.xyz, s), at
// its brick-layout slot (MapFast::index); padding slots of partial bricks
// stay empty.
__global__ void k_map_records(const int32_t* __restrict__ cells, int64_t n_cells, GridDev nnf,
                              const double* __restrict__ mu, const float4* __restrict__ plane, int brick,
                              float4* __restrict__ rec) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= n_cells) return;
  const int nx = nnf.dims[0], ny = nnf.dims[1];
  const int64_t ix = c % nx, iy = (c / nx) % ny, iz = c / (static_cast<int64_t>(nx) * ny);
  MapFast mf;
  mf.brick = brick;
  for (int a = 0; a < 3; ++a) mf.g.dims[a] = nnf.dims[a];
  const uint64_t slot = mf.index(static_cast<uint32_t>(ix), static_cast<uint32_t>(iy), static_cast<uint32_t>(iz));
  const int32_t mi = cells[c];
  if (mi < 0) {
    rec[2 * slot] = make_float4(0.f, 0.f, 0.f, -1.f);
    rec[2 * slot + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const double corner[3] = {__dadd_rn(nnf.org[0], __dmul_rn(static_cast<double>(ix), nnf.cell)),
                            __dadd_rn(nnf.org[1], __dmul_rn(static_cast<double>(iy), nnf.cell)),
                            __dadd_rn(nnf.org[2], __dmul_rn(static_cast<double>(iz), nnf.cell))};
  const float4 p0 = plane[2 * mi], p1 = plane[2 * mi + 1];  // (beta, s, -, -), (u.xyz, -)
  rec[2 * slot] = make_float4(__double2float_rn(__dsub_rn(mu[3 * mi], corner[0])),
                              __double2float_rn(__dsub_rn(mu[3 * mi + 1], corner[1])),
                              __double2float_rn(__dsub_rn(mu[3 * mi + 2], corner[2])), p0.x);
  rec[2 * slot + 1] = make_float4(p1.x, p1.y, p1.z, p0.y);
}

__global__ void k_fill_empty(float4* __restrict__ rec, uint64_t n) {
  const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= n) return;
  rec[2 * c] = make_float4(0.f, 0.f, 0.f, -1.f);
  rec[2 * c + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
}

GridDev grid_dev(const double org[3], double cell, const int dims[3]) {
  GridDev g;
  for (int a = 0; a < 3; ++a) {
    g.org[a] = org[a];
    g.dims[a] = dims[a];
  }
  g.cell = cell;
  return g;
}

}  // namespace

cudaError_t build_nnf_device(const double* d_mu, int64_t n, const double pg_org[3], const int pg_dims[3],
                      const double nnf_org[3], const int nnf_dims[3], double res, double max_query_dist,
                      int32_t* d_cells, cudaStream_t st) {
  const int64_t pg_cells = static_cast<int64_t>(pg_dims[0]) * pg_dims[1] * pg_dims[2];
  const int64_t n_cells = static_cast<int64_t>(nnf_dims[0]) * nnf_dims[1] * nnf_dims[2];
  const GridDev pg = grid_dev(pg_org, res, pg_dims);
  const GridDev ng = grid_dev(nnf_org, res, nnf_dims);
  // scratch
  int32_t *cid, *cid_sorted, *iota, *order, *counts, *offsets;
  uint8_t *occ, *tmp;
  size_t sort_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, static_cast<const int32_t*>(nullptr),
                                  static_cast<int32_t*>(nullptr), static_cast<const int32_t*>(nullptr),
                                  static_cast<int32_t*>(nullptr), static_cast<int>(n), 0, 32);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, static_cast<const int32_t*>(nullptr),
                                static_cast<int32_t*>(nullptr), static_cast<int>(pg_cells + 1));
  void* temp;
  const size_t temp_bytes = std::max(sort_bytes, scan_bytes);
  MB_CK(cudaMallocAsync(reinterpret_cast<void**>(&cid), sizeof(int32_t) * n, st));
  MB_CK(cudaMallocAsync(reinterpret_cast<void**>(&cid_sorted), sizeof(int32_t) * n, st));
  MB_CK(cudaMallocAsync(reinterpret_cast<void**>(&iota), sizeof(int32_t) * n, st));
  MB_CK(cudaMallocAsync(reinterpret_cast<void**>(&order), sizeof(int32_t) * n, st));
  MB_CK(cudaMallocAsync(reinterpret_cast<void**>(&counts), sizeof(int32_t) * (pg_cells + 1), st));
  MB_CK(cudaMallocAsync(reinterpret_cast<void**>(&offsets), sizeof(int32_t) * (pg_cells + 1), st));
  MB_CK(cudaMallocAsync(reinterpret_cast<void**>(&occ), static_cast<size_t>(n_cells), st));
  MB_CK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), static_cast<size_t>(n_cells), st));
  MB_CK(cudaMallocAsync(&temp, temp_bytes, st));
  // 1. point grid (CSR, ascending point index inside a cell)
  MB_CK(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (pg_cells + 1), st));
  count_launch();
  k_point_cells<<<blocks_for(n, 256), 256, 0, st>>>(d_mu, n, pg, cid, iota, counts);
  size_t tb = temp_bytes;
  MB_CK(cub::DeviceRadixSort::SortPairs(temp, tb, cid, cid_sorted, iota, order, static_cast<int>(n), 0, 32, st));
  tb = temp_bytes;
  MB_CK(cub::DeviceScan::ExclusiveSum(temp, tb, counts, offsets, static_cast<int>(pg_cells + 1), st));
  // 2. occupancy + Chebyshev dilation by hop_cap (nnf.cpp:37-80)
  MB_CK(cudaMemsetAsync(occ, 0, static_cast<size_t>(n_cells), st));
  count_launch();
  k_nnf_occupancy<<<blocks_for(n, 256), 256, 0, st>>>(d_mu, n, ng, occ);
  const int hop = static_cast<int>(std::ceil(max_query_dist / res)) + 2;
  count_launch(3);
  k_dilate<<<blocks_for(n_cells, 256), 256, 0, st>>>(occ, tmp, n_cells, nnf_dims[0], nnf_dims[1], nnf_dims[2], 0, hop);
  k_dilate<<<blocks_for(n_cells, 256), 256, 0, st>>>(tmp, occ, n_cells, nnf_dims[0], nnf_dims[1], nnf_dims[2], 1, hop);
  k_dilate<<<blocks_for(n_cells, 256), 256, 0, st>>>(occ, tmp, n_cells, nnf_dims[0], nnf_dims[1], nnf_dims[2], 2, hop);
  // 3. exact nearest point within max_query_dist at every reached cell centre
  count_launch();
  k_nnf_query<<<blocks_for(n_cells, 128), 128, 0, st>>>(tmp, n_cells, ng, max_query_dist, pg, offsets, order, d_mu,
                                                         d_cells);
  MB_CK(cudaGetLastError());
  for (void* p : {static_cast<void*>(cid), static_cast<void*>(cid_sorted), static_cast<void*>(iota),
                  static_cast<void*>(order), static_cast<void*>(counts), static_cast<void*>(offsets),
                  static_cast<void*>(occ), static_cast<void*>(tmp), temp})
    MB_CK(cudaFreeAsync(p, st));
  return cudaSuccess;
}

cudaError_t build_map_records_device(const int32_t* d_cells, int64_t n_cells, const double nnf_org[3], const int nnf_dims[3],
                              double res, const double* d_mu, const float4* d_plane, float4* d_rec, cudaStream_t st) {
  // partial bricks: every slot starts empty (beta = -1)
  const int brick = MapFast::choose_brick(nnf_dims);
  const uint64_t nrec = MapFast::n_records(nnf_dims, brick);
  count_launch();
  k_fill_empty<<<blocks_for(static_cast<int64_t>(nrec), 256), 256, 0, st>>>(d_rec, nrec);
  count_launch();
  k_map_records<<<blocks_for(n_cells, 256), 256, 0, st>>>(d_cells, n_cells, grid_dev(nnf_org, res, nnf_dims), d_mu,
                                                          d_plane, brick, d_rec);
  return cudaGetLastError();
}

}  // namespace smcl
