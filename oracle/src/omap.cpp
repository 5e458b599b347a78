// ORACLE — test infrastructure only. Map / scan preparation restated from
// /root/reference/proj/src/{gaussian_cloud,point_grid,nnf}.cpp.
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <unordered_map>

#include "oracle.hpp"

namespace orc {

// gaussian_cloud.cpp:14-22
Aabb compute_bounds(std::span<const V3> points) {
  if (points.empty()) throw std::invalid_argument("compute_bounds: empty point set");
  Aabb b{points[0], points[0]};
  for (const V3& p : points)
    for (int a = 0; a < 3; ++a) {
      b.min[a] = std::min(b.min[a], p[a]);
      b.max[a] = std::max(b.max[a], p[a]);
    }
  return b;
}

// Cyclic Jacobi eigen-solver for a symmetric 3x3 (stands in for Eigen's
// SelfAdjointEigenSolver; the plane-model covariance it feeds depends only on
// the smallest eigenvector and the largest eigenvalue, so any accurate solver
// agrees to ~1e-16 relative). Eigenvalues ascending, eigenvectors in columns.
void sym_eig3(const M3& a_in, double w[3], M3& v) {
  double a[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a[i][j] = a_in(i, j);
  double V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 50; ++sweep) {
    const double off = std::fabs(a[0][1]) + std::fabs(a[0][2]) + std::fabs(a[1][2]);
    const double scale = std::fabs(a[0][0]) + std::fabs(a[1][1]) + std::fabs(a[2][2]);
    if (off == 0.0 || off <= 1e-300 || off < 1e-18 * scale) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (a[p][q] == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {  // A <- A J
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {  // A <- J^T A
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          const double vkp = V[k][p], vkq = V[k][q];
          V[k][p] = c * vkp - s * vkq;
          V[k][q] = s * vkp + c * vkq;
        }
      }
  }
  int ord[3] = {0, 1, 2};
  std::sort(ord, ord + 3, [&](int x, int y) { return a[x][x] < a[y][y]; });
  for (int c = 0; c < 3; ++c) {
    w[c] = a[ord[c]][ord[c]];
    for (int r = 0; r < 3; ++r) v(r, c) = V[r][ord[c]];
  }
}

namespace {
// gaussian_cloud.cpp:25-30
double knn_cell_size(const Aabb& bounds, std::size_t n, int k) {
  V3 ext = bounds.extent();
  for (int a = 0; a < 3; ++a) ext[a] = std::max(ext[a], 1e-6);
  const double volume = (ext[0] * ext[1]) * ext[2];
  const double per_cell = std::max(1.0, static_cast<double>(k) / 2.0);
  return std::max(1e-6, std::cbrt(volume * per_cell / static_cast<double>(n)));
}
}  // namespace

// gaussian_cloud.cpp:36-90
GaussianCloud estimate_covariances(std::span<const V3> points, int k, double eps) {
  if (k < 4) throw std::invalid_argument("estimate_covariances: k must be >= 4");
  if (points.size() < static_cast<std::size_t>(k) + 1)
    throw std::invalid_argument("estimate_covariances: need at least k+1 points");
  GaussianCloud out;
  out.bounds = compute_bounds(points);
  out.mu.assign(points.begin(), points.end());
  out.sigma.resize(points.size());
  const PointBucketGrid grid(points, knn_cell_size(out.bounds, points.size(), k));
#pragma omp parallel
  {
    std::vector<PointBucketGrid::Neighbor> nn;
    std::vector<V3> nbr;
#pragma omp for schedule(static)
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(points.size()); ++i) {
      grid.k_nearest(points[static_cast<std::size_t>(i)], k + 1, nn);
      nbr.clear();
      for (const auto& c : nn) {
        if (c.index == i) continue;
        nbr.push_back(points[static_cast<std::size_t>(c.index)]);
        if (static_cast<int>(nbr.size()) == k) break;
      }
      std::sort(nbr.begin(), nbr.end(), [](const V3& a, const V3& b) {
        if (a[0] != b[0]) return a[0] < b[0];
        if (a[1] != b[1]) return a[1] < b[1];
        return a[2] < b[2];
      });
      V3 mean;
      for (const V3& p : nbr) mean = mean + p;
      const double nn_d = static_cast<double>(nbr.size());
      for (int a = 0; a < 3; ++a) mean[a] = mean[a] / nn_d;
      M3 cov;
      for (const V3& p : nbr) {
        const V3 d = p - mean;
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) cov(r, c) = cov(r, c) + d[r] * d[c];
      }
      for (double& c : cov.m) c = c / nn_d;
      double w[3];
      M3 v;
      sym_eig3(cov, w, v);
      const double lmax = std::max(w[2], 1e-12);
      const double reg[3] = {eps * lmax, lmax, lmax};
      M3 s;
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
          s(r, c) = ((v(r, 0) * reg[0]) * v(c, 0) + (v(r, 1) * reg[1]) * v(c, 1)) + (v(r, 2) * reg[2]) * v(c, 2);
      out.sigma[static_cast<std::size_t>(i)] = s;
    }
  }
  return out;
}

namespace {
struct CellKey {
  std::int64_t x, y, z;
  bool operator==(const CellKey&) const = default;
};
struct CellKeyHash {
  std::size_t operator()(const CellKey& c) const {
    std::uint64_t h = static_cast<std::uint64_t>(c.x) * 73856093ull;
    h ^= static_cast<std::uint64_t>(c.y) * 19349663ull;
    h ^= static_cast<std::uint64_t>(c.z) * 83492791ull;
    return static_cast<std::size_t>(h);
  }
};
}  // namespace

// gaussian_cloud.cpp:110-132: centroids in first-seen cell order.
std::vector<V3> voxel_downsample(std::span<const V3> points, double leaf) {
  if (!(leaf > 0.0)) throw std::invalid_argument("voxel_downsample: leaf must be positive");
  std::unordered_map<CellKey, std::pair<V3, int>, CellKeyHash> cells;
  cells.reserve(points.size());
  std::vector<CellKey> order;
  for (const V3& p : points) {
    const CellKey key{static_cast<std::int64_t>(std::floor(p[0] / leaf)),
                      static_cast<std::int64_t>(std::floor(p[1] / leaf)),
                      static_cast<std::int64_t>(std::floor(p[2] / leaf))};
    auto [it, fresh] = cells.try_emplace(key, V3{}, 0);
    if (fresh) order.push_back(key);
    it->second.first = it->second.first + p;
    it->second.second += 1;
  }
  std::vector<V3> out;
  out.reserve(order.size());
  for (const CellKey& key : order) {
    const auto& [sum, n] = cells.at(key);
    const double d = static_cast<double>(n);
    out.push_back(v3(sum[0] / d, sum[1] / d, sum[2] / d));
  }
  return out;
}

// gaussian_cloud.cpp:134-144
std::vector<V3> downsample_to(std::span<const V3> points, std::size_t max_points, double leaf0) {
  if (points.size() <= max_points) return {points.begin(), points.end()};
  double leaf = leaf0;
  std::vector<V3> out = voxel_downsample(points, leaf);
  while (out.size() > max_points) {
    leaf *= 2.0;
    out = voxel_downsample(points, leaf);
  }
  return out;
}

// point_grid.cpp:10-40
PointBucketGrid::PointBucketGrid(std::span<const V3> points, double cell_size)
    : points_(points.begin(), points.end()), cell_size_(cell_size) {
  if (points_.empty()) throw std::invalid_argument("PointBucketGrid: empty point set");
  if (!(cell_size > 0.0)) throw std::invalid_argument("PointBucketGrid: cell_size must be positive");
  V3 lo = points_[0], hi = points_[0];
  for (const V3& p : points_)
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], p[a]);
      hi[a] = std::max(hi[a], p[a]);
    }
  origin_ = lo;
  for (int a = 0; a < 3; ++a) dims_[a] = static_cast<int>(std::floor((hi[a] - lo[a]) / cell_size_)) + 1;
  const std::size_t n_cells = static_cast<std::size_t>(dims_[0]) * dims_[1] * dims_[2];
  std::vector<std::int32_t> counts(n_cells + 1, 0), cell(points_.size());
  for (std::size_t i = 0; i < points_.size(); ++i) {
    int c[3];
    cell_of(points_[i], c);
    cell[i] = cell_index(c[0], c[1], c[2]);
    ++counts[static_cast<std::size_t>(cell[i]) + 1];
  }
  offsets_.assign(n_cells + 1, 0);
  for (std::size_t c = 0; c < n_cells; ++c) offsets_[c + 1] = offsets_[c] + counts[c + 1];
  order_.resize(points_.size());
  std::vector<std::int32_t> cursor(offsets_.begin(), offsets_.end() - 1);
  for (std::size_t i = 0; i < points_.size(); ++i)
    order_[static_cast<std::size_t>(cursor[static_cast<std::size_t>(cell[i])]++)] = static_cast<std::int32_t>(i);
}

void PointBucketGrid::cell_of(const V3& p, int c[3]) const {  // point_grid.cpp:42-49
  for (int a = 0; a < 3; ++a) {
    const int v = static_cast<int>(std::floor((p[a] - origin_[a]) / cell_size_));
    c[a] = std::clamp(v, 0, dims_[a] - 1);
  }
}

// point_grid.cpp:51-107
void PointBucketGrid::k_nearest(const V3& query, int k, std::vector<Neighbor>& out) const {
  out.clear();
  if (k <= 0) return;
  int c0[3];
  cell_of(query, c0);
  const int r_max = std::max({dims_[0], dims_[1], dims_[2]});
  double worst = std::numeric_limits<double>::infinity();
  auto offer = [&](std::int32_t idx) {
    const double d2 = sqnorm(points_[static_cast<std::size_t>(idx)] - query);
    if (static_cast<int>(out.size()) < k) {
      out.push_back({d2, idx});
      if (static_cast<int>(out.size()) == k) {
        std::sort(out.begin(), out.end(), [](const Neighbor& a, const Neighbor& b) { return a.dist2 < b.dist2; });
        worst = out.back().dist2;
      }
      return;
    }
    if (d2 >= worst) return;
    out.back() = {d2, idx};
    for (std::size_t j = out.size() - 1; j > 0 && out[j].dist2 < out[j - 1].dist2; --j) std::swap(out[j], out[j - 1]);
    worst = out.back().dist2;
  };
  for (int r = 0; r <= r_max; ++r) {
    if (static_cast<int>(out.size()) >= k) {
      const double lb = (r - 1) * cell_size_;
      if (lb > 0.0 && lb * lb > worst) break;
    }
    const int xlo = std::max(c0[0] - r, 0), xhi = std::min(c0[0] + r, dims_[0] - 1);
    const int ylo = std::max(c0[1] - r, 0), yhi = std::min(c0[1] + r, dims_[1] - 1);
    const int zlo = std::max(c0[2] - r, 0), zhi = std::min(c0[2] + r, dims_[2] - 1);
    for (int z = zlo; z <= zhi; ++z)
      for (int y = ylo; y <= yhi; ++y)
        for (int x = xlo; x <= xhi; ++x) {
          const int cheb = std::max({std::abs(x - c0[0]), std::abs(y - c0[1]), std::abs(z - c0[2])});
          if (cheb != r) continue;
          const std::int32_t ci = cell_index(x, y, z);
          for (std::int32_t j = offsets_[static_cast<std::size_t>(ci)]; j < offsets_[static_cast<std::size_t>(ci) + 1]; ++j)
            offer(order_[static_cast<std::size_t>(j)]);
        }
  }
  if (static_cast<int>(out.size()) < k)
    std::sort(out.begin(), out.end(), [](const Neighbor& a, const Neighbor& b) { return a.dist2 < b.dist2; });
}

// point_grid.cpp:109-141: ties go to the lower index.
std::int32_t PointBucketGrid::nearest_within(const V3& query, double max_dist) const {
  int c0[3];
  cell_of(query, c0);
  const int r_cap = static_cast<int>(std::ceil(max_dist / cell_size_)) + 1;
  double best2 = max_dist * max_dist;
  std::int32_t best = -1;
  for (int r = 0; r <= r_cap; ++r) {
    const double lb = (r - 1) * cell_size_;
    if (lb > 0.0 && lb * lb > best2) break;
    const int xlo = std::max(c0[0] - r, 0), xhi = std::min(c0[0] + r, dims_[0] - 1);
    const int ylo = std::max(c0[1] - r, 0), yhi = std::min(c0[1] + r, dims_[1] - 1);
    const int zlo = std::max(c0[2] - r, 0), zhi = std::min(c0[2] + r, dims_[2] - 1);
    for (int z = zlo; z <= zhi; ++z)
      for (int y = ylo; y <= yhi; ++y)
        for (int x = xlo; x <= xhi; ++x) {
          const int cheb = std::max({std::abs(x - c0[0]), std::abs(y - c0[1]), std::abs(z - c0[2])});
          if (cheb != r) continue;
          const std::int32_t ci = cell_index(x, y, z);
          for (std::int32_t j = offsets_[static_cast<std::size_t>(ci)]; j < offsets_[static_cast<std::size_t>(ci) + 1]; ++j) {
            const std::int32_t idx = order_[static_cast<std::size_t>(j)];
            const double d2 = sqnorm(points_[static_cast<std::size_t>(idx)] - query);
            if (d2 < best2 || (d2 == best2 && best >= 0 && idx < best)) {
              best2 = d2;
              best = idx;
            }
          }
        }
  }
  return best;
}

// nnf.cpp:10-96
NearestNeighborField build_nnf(const GaussianCloud& map, double resolution, double padding,
                               double max_query_dist, std::size_t max_cells) {
  if (map.empty()) throw std::invalid_argument("build_nnf: empty map");
  if (!(resolution > 0.0)) throw std::invalid_argument("build_nnf: resolution must be positive");
  if (padding < 0.0) throw std::invalid_argument("build_nnf: padding must be >= 0");
  NearestNeighborField nnf;
  nnf.resolution = resolution;
  nnf.max_query_dist = max_query_dist;
  const Aabb padded = map.bounds.padded(padding);
  nnf.origin = padded.min;
  std::size_t n_cells = 1;
  const V3 ext = padded.extent();
  for (int a = 0; a < 3; ++a) {
    nnf.dims[a] = static_cast<int>(std::floor(ext[a] / resolution)) + 1;
    n_cells *= static_cast<std::size_t>(nnf.dims[a]);
    if (n_cells > max_cells) throw std::runtime_error("build_nnf: cell count exceeds the memory budget");
  }
  nnf.cells.assign(n_cells, NearestNeighborField::k_empty);
  const int nx = nnf.dims[0], ny = nnf.dims[1], nz = nnf.dims[2];
  auto flat = [&](int x, int y, int z) { return (static_cast<std::size_t>(z) * ny + y) * nx + x; };

  const int hop_cap = static_cast<int>(std::ceil(max_query_dist / resolution)) + 2;
  std::vector<std::int16_t> hops(n_cells, -1);
  std::vector<std::int32_t> frontier, next;
  for (const V3& p : map.mu) {
    int c[3];
    for (int a = 0; a < 3; ++a)
      c[a] = std::clamp(static_cast<int>(std::floor((p[a] - nnf.origin[a]) / resolution)), 0, nnf.dims[a] - 1);
    const std::size_t ci = flat(c[0], c[1], c[2]);
    if (hops[ci] < 0) {
      hops[ci] = 0;
      frontier.push_back(static_cast<std::int32_t>(ci));
    }
  }
  for (int hop = 1; hop <= hop_cap && !frontier.empty(); ++hop) {
    next.clear();
    for (std::int32_t ci : frontier) {
      const int x = ci % nx, y = (ci / nx) % ny, z = ci / (nx * ny);
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const int xx = x + dx, yy = y + dy, zz = z + dz;
            if (static_cast<unsigned>(xx) >= static_cast<unsigned>(nx) ||
                static_cast<unsigned>(yy) >= static_cast<unsigned>(ny) ||
                static_cast<unsigned>(zz) >= static_cast<unsigned>(nz))
              continue;
            const std::size_t c = flat(xx, yy, zz);
            if (hops[c] < 0) {
              hops[c] = static_cast<std::int16_t>(hop);
              next.push_back(static_cast<std::int32_t>(c));
            }
          }
    }
    frontier.swap(next);
  }
  const PointBucketGrid grid(map.mu, resolution);
#pragma omp parallel for schedule(dynamic, 64)
  for (std::int64_t z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        const std::size_t c = flat(x, y, static_cast<int>(z));
        if (hops[c] < 0) continue;
        const V3 center = v3(nnf.origin[0] + resolution * (x + 0.5), nnf.origin[1] + resolution * (y + 0.5),
                             nnf.origin[2] + resolution * (static_cast<double>(z) + 0.5));
        nnf.cells[c] = grid.nearest_within(center, max_query_dist);
      }
  return nnf;
}

}  // namespace orc
