// Host-side map load and scan preparation (product). Restates
// /root/reference/proj/src/{gaussian_cloud,point_grid,nnf}.cpp and
// filter.cpp:86-100 (make_scan_cloud). One-time / per-frame host setup that
// feeds the device hot path.
#pragma once

#include <cstdint>
#include <vector>

namespace smcl::host {

struct V3 {
  double x, y, z;
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};

struct Aabb {
  double min[3], max[3];
};

Aabb compute_bounds(const V3* p, std::int64_t n);  // gaussian_cloud.cpp:14-22

// gaussian_cloud.cpp:36-90: kNN (k) sample covariance, eigenvalues replaced by
// lambda_max * (eps, 1, 1). sigma_out: n*9 row-major.
void estimate_covariances(const V3* p, std::int64_t n, int k, double eps, double* sigma_out);
// gaussian_cloud.cpp:110-144
std::vector<V3> voxel_downsample(const V3* p, std::int64_t n, double leaf);
std::vector<V3> downsample_to(const V3* p, std::int64_t n, std::size_t max_points, double leaf0);

// Symmetric 3x3 eigen-decomposition (ascending), eigenvectors in columns of v.
void sym_eig3(const double a[9], double w[3], double v[9]);

// nnf.cpp:10-96. dims/origin always returned; cells filled when non-null.
struct NnfGeometry {
  double origin[3];
  double resolution;
  double max_query_dist;
  int dims[3];
  std::int64_t n_cells;
};
NnfGeometry nnf_geometry(const Aabb& map_bounds, double resolution, double padding, double max_query_dist,
                         std::size_t max_cells);
void build_nnf_cells(const V3* mu, std::int64_t n, const NnfGeometry& g, std::int32_t* cells);

// point_grid.cpp: CSR uniform grid with exact k-NN / nearest-within queries.
class PointGrid {
 public:
  PointGrid(const V3* p, std::int64_t n, double cell);
  struct Nb {
    double d2;
    std::int32_t idx;
  };
  void k_nearest(const V3& q, int k, std::vector<Nb>& out) const;
  std::int32_t nearest_within(const V3& q, double max_dist) const;

 private:
  void cell_of(const V3& p, int c[3]) const;
  const V3* pts_;
  std::int64_t n_;
  double cell_, org_[3];
  int dims_[3];
  std::vector<std::int32_t> order_, offsets_;
};

}  // namespace smcl::host
