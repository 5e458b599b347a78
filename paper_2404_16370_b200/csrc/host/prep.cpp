// Host-side map load and scan preparation for the B200 engine. Restates the
// reference's setup path (gaussian_cloud.cpp, point_grid.cpp, nnf.cpp); the
// NNF build replaces the serial BFS (nnf.cpp:37-80) with an equivalent
// separable Chebyshev dilation, then does the same exact ring query per cell.
#include "prep.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>
#include <unordered_map>

namespace smcl::host {

Aabb compute_bounds(const V3* p, std::int64_t n) {
  if (n <= 0) throw std::invalid_argument("compute_bounds: empty point set");
  Aabb b{{p[0].x, p[0].y, p[0].z}, {p[0].x, p[0].y, p[0].z}};
  for (std::int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      b.min[a] = std::min(b.min[a], p[i][a]);
      b.max[a] = std::max(b.max[a], p[i][a]);
    }
  return b;
}

void sym_eig3(const double a_in[9], double w[3], double v[9]) {
  double a[3][3], V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a[i][j] = a_in[i * 3 + j];
  for (int sweep = 0; sweep < 50; ++sweep) {
    const double off = std::fabs(a[0][1]) + std::fabs(a[0][2]) + std::fabs(a[1][2]);
    const double scale = std::fabs(a[0][0]) + std::fabs(a[1][1]) + std::fabs(a[2][2]);
    if (off == 0.0 || off <= 1e-300 || off < 1e-18 * scale) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (a[p][q] == 0.0) continue;
        const double th = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {
          const double x = a[k][p], y = a[k][q];
          a[k][p] = c * x - s * y;
          a[k][q] = s * x + c * y;
        }
        for (int k = 0; k < 3; ++k) {
          const double x = a[p][k], y = a[q][k];
          a[p][k] = c * x - s * y;
          a[q][k] = s * x + c * y;
        }
        for (int k = 0; k < 3; ++k) {
          const double x = V[k][p], y = V[k][q];
          V[k][p] = c * x - s * y;
          V[k][q] = s * x + c * y;
        }
      }
  }
  int ord[3] = {0, 1, 2};
  std::sort(ord, ord + 3, [&](int x, int y) { return a[x][x] < a[y][y]; });
  for (int c = 0; c < 3; ++c) {
    w[c] = a[ord[c]][ord[c]];
    for (int r = 0; r < 3; ++r) v[r * 3 + c] = V[r][ord[c]];
  }
}

// ---------------------------------------------------------------- point grid
PointGrid::PointGrid(const V3* p, std::int64_t n, double cell) : pts_(p), n_(n), cell_(cell) {
  if (n <= 0) throw std::invalid_argument("PointBucketGrid: empty point set");
  if (!(cell > 0.0)) throw std::invalid_argument("PointBucketGrid: cell_size must be positive");
  const Aabb b = compute_bounds(p, n);
  for (int a = 0; a < 3; ++a) {
    org_[a] = b.min[a];
    dims_[a] = static_cast<int>(std::floor((b.max[a] - b.min[a]) / cell_)) + 1;
  }
  const std::size_t nc = static_cast<std::size_t>(dims_[0]) * dims_[1] * dims_[2];
  std::vector<std::int32_t> cid(static_cast<std::size_t>(n));
  offsets_.assign(nc + 1, 0);
  for (std::int64_t i = 0; i < n; ++i) {
    int c[3];
    cell_of(p[i], c);
    cid[static_cast<std::size_t>(i)] = (c[2] * dims_[1] + c[1]) * dims_[0] + c[0];
    ++offsets_[static_cast<std::size_t>(cid[static_cast<std::size_t>(i)]) + 1];
  }
  for (std::size_t c = 0; c < nc; ++c) offsets_[c + 1] += offsets_[c];
  order_.resize(static_cast<std::size_t>(n));
  std::vector<std::int32_t> cur(offsets_.begin(), offsets_.end() - 1);
  for (std::int64_t i = 0; i < n; ++i)
    order_[static_cast<std::size_t>(cur[static_cast<std::size_t>(cid[static_cast<std::size_t>(i)])]++)] =
        static_cast<std::int32_t>(i);
}

void PointGrid::cell_of(const V3& p, int c[3]) const {
  for (int a = 0; a < 3; ++a) c[a] = std::clamp(static_cast<int>(std::floor((p[a] - org_[a]) / cell_)), 0, dims_[a] - 1);
}

static inline double d2of(const V3& a, const V3& b) {
  const double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
  return (dx * dx + dy * dy) + dz * dz;
}

// point_grid.cpp:51-107 (ring search, insertion-sorted candidates, ties keep
// the first seen).
void PointGrid::k_nearest(const V3& q, int k, std::vector<Nb>& out) const {
  out.clear();
  if (k <= 0) return;
  int c0[3];
  cell_of(q, c0);
  const int r_max = std::max({dims_[0], dims_[1], dims_[2]});
  double worst = std::numeric_limits<double>::infinity();
  for (int r = 0; r <= r_max; ++r) {
    if (static_cast<int>(out.size()) >= k) {
      const double lb = (r - 1) * cell_;
      if (lb > 0.0 && lb * lb > worst) break;
    }
    const int z0 = std::max(c0[2] - r, 0), z1 = std::min(c0[2] + r, dims_[2] - 1);
    const int y0 = std::max(c0[1] - r, 0), y1 = std::min(c0[1] + r, dims_[1] - 1);
    const int x0 = std::max(c0[0] - r, 0), x1 = std::min(c0[0] + r, dims_[0] - 1);
    for (int z = z0; z <= z1; ++z)
      for (int y = y0; y <= y1; ++y) {
        const bool yz_shell = std::abs(z - c0[2]) == r || std::abs(y - c0[1]) == r;
        for (int x = x0; x <= x1; ++x) {
          if (!yz_shell && std::abs(x - c0[0]) != r) continue;
          const std::size_t ci = static_cast<std::size_t>((z * dims_[1] + y) * dims_[0] + x);
          for (std::int32_t j = offsets_[ci]; j < offsets_[ci + 1]; ++j) {
            const std::int32_t idx = order_[static_cast<std::size_t>(j)];
            const double d2 = d2of(pts_[idx], q);
            if (static_cast<int>(out.size()) < k) {
              out.push_back({d2, idx});
              if (static_cast<int>(out.size()) == k) {
                std::sort(out.begin(), out.end(), [](const Nb& a, const Nb& b) { return a.d2 < b.d2; });
                worst = out.back().d2;
              }
              continue;
            }
            if (d2 >= worst) continue;
            out.back() = {d2, idx};
            for (std::size_t s = out.size() - 1; s > 0 && out[s].d2 < out[s - 1].d2; --s) std::swap(out[s], out[s - 1]);
            worst = out.back().d2;
          }
        }
      }
  }
  if (static_cast<int>(out.size()) < k)
    std::sort(out.begin(), out.end(), [](const Nb& a, const Nb& b) { return a.d2 < b.d2; });
}

// point_grid.cpp:109-141 (ties go to the lower index).
std::int32_t PointGrid::nearest_within(const V3& q, double max_dist) const {
  int c0[3];
  cell_of(q, c0);
  const int r_cap = static_cast<int>(std::ceil(max_dist / cell_)) + 1;
  double best2 = max_dist * max_dist;
  std::int32_t best = -1;
  for (int r = 0; r <= r_cap; ++r) {
    const double lb = (r - 1) * cell_;
    if (lb > 0.0 && lb * lb > best2) break;
    const int z0 = std::max(c0[2] - r, 0), z1 = std::min(c0[2] + r, dims_[2] - 1);
    const int y0 = std::max(c0[1] - r, 0), y1 = std::min(c0[1] + r, dims_[1] - 1);
    const int x0 = std::max(c0[0] - r, 0), x1 = std::min(c0[0] + r, dims_[0] - 1);
    for (int z = z0; z <= z1; ++z)
      for (int y = y0; y <= y1; ++y) {
        const bool yz_shell = std::abs(z - c0[2]) == r || std::abs(y - c0[1]) == r;
        for (int x = x0; x <= x1; ++x) {
          if (!yz_shell && std::abs(x - c0[0]) != r) continue;
          const std::size_t ci = static_cast<std::size_t>((z * dims_[1] + y) * dims_[0] + x);
          for (std::int32_t j = offsets_[ci]; j < offsets_[ci + 1]; ++j) {
            const std::int32_t idx = order_[static_cast<std::size_t>(j)];
            const double d2 = d2of(pts_[idx], q);
            if (d2 < best2 || (d2 == best2 && best >= 0 && idx < best)) {
              best2 = d2;
              best = idx;
            }
          }
        }
      }
  }
  return best;
}

// ---------------------------------------------------------------- covariances
static double knn_cell_size(const Aabb& b, std::int64_t n, int k) {
  double ext[3];
  for (int a = 0; a < 3; ++a) ext[a] = std::max(b.max[a] - b.min[a], 1e-6);
  const double volume = (ext[0] * ext[1]) * ext[2];
  const double per_cell = std::max(1.0, static_cast<double>(k) / 2.0);
  return std::max(1e-6, std::cbrt(volume * per_cell / static_cast<double>(n)));
}

void estimate_covariances(const V3* p, std::int64_t n, int k, double eps, double* sigma_out) {
  if (k < 4) throw std::invalid_argument("estimate_covariances: k must be >= 4");
  if (n < static_cast<std::int64_t>(k) + 1) throw std::invalid_argument("estimate_covariances: need at least k+1 points");
  const PointGrid grid(p, n, knn_cell_size(compute_bounds(p, n), n, k));
#pragma omp parallel
  {
    std::vector<PointGrid::Nb> nn;
    std::vector<V3> nb;
#pragma omp for schedule(static)
    for (std::int64_t i = 0; i < n; ++i) {
      grid.k_nearest(p[i], k + 1, nn);
      nb.clear();
      for (const auto& c : nn) {
        if (c.idx == i) continue;
        nb.push_back(p[c.idx]);
        if (static_cast<int>(nb.size()) == k) break;
      }
      // Canonical accumulation order (gaussian_cloud.cpp:62-67).
      std::sort(nb.begin(), nb.end(), [](const V3& a, const V3& b) {
        if (a.x != b.x) return a.x < b.x;
        if (a.y != b.y) return a.y < b.y;
        return a.z < b.z;
      });
      double m[3] = {0, 0, 0};
      for (const V3& q : nb)
        for (int a = 0; a < 3; ++a) m[a] = m[a] + q[a];
      const double cnt = static_cast<double>(nb.size());
      for (double& c : m) c = c / cnt;
      double cov[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (const V3& q : nb) {
        const double d[3] = {q.x - m[0], q.y - m[1], q.z - m[2]};
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) cov[r * 3 + c] = cov[r * 3 + c] + d[r] * d[c];
      }
      for (double& c : cov) c = c / cnt;
      double w[3], v[9];
      sym_eig3(cov, w, v);
      const double lmax = std::max(w[2], 1e-12);
      const double reg[3] = {eps * lmax, lmax, lmax};
      double* s = sigma_out + 9 * i;
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
          s[r * 3 + c] = ((v[r * 3 + 0] * reg[0]) * v[c * 3 + 0] + (v[r * 3 + 1] * reg[1]) * v[c * 3 + 1]) +
                         (v[r * 3 + 2] * reg[2]) * v[c * 3 + 2];
    }
  }
}

// ---------------------------------------------------------------- downsampling
namespace {
struct Key {
  std::int64_t x, y, z;
  bool operator==(const Key&) const = default;
};
struct KeyHash {
  std::size_t operator()(const Key& c) const {
    std::uint64_t h = static_cast<std::uint64_t>(c.x) * 73856093ull;
    h ^= static_cast<std::uint64_t>(c.y) * 19349663ull;
    h ^= static_cast<std::uint64_t>(c.z) * 83492791ull;
    return static_cast<std::size_t>(h);
  }
};
}  // namespace

std::vector<V3> voxel_downsample(const V3* p, std::int64_t n, double leaf) {
  if (!(leaf > 0.0)) throw std::invalid_argument("voxel_downsample: leaf must be positive");
  struct Acc {
    double s[3];
    int c;
  };
  std::unordered_map<Key, std::size_t, KeyHash> slot;
  slot.reserve(static_cast<std::size_t>(n));
  std::vector<Acc> acc;
  for (std::int64_t i = 0; i < n; ++i) {
    const Key key{static_cast<std::int64_t>(std::floor(p[i].x / leaf)), static_cast<std::int64_t>(std::floor(p[i].y / leaf)),
                  static_cast<std::int64_t>(std::floor(p[i].z / leaf))};
    auto [it, fresh] = slot.try_emplace(key, acc.size());
    if (fresh) acc.push_back({{0.0, 0.0, 0.0}, 0});
    Acc& a = acc[it->second];
    a.s[0] = a.s[0] + p[i].x;
    a.s[1] = a.s[1] + p[i].y;
    a.s[2] = a.s[2] + p[i].z;
    a.c += 1;
  }
  std::vector<V3> out;
  out.reserve(acc.size());
  for (const Acc& a : acc) {
    const double d = static_cast<double>(a.c);
    out.push_back({a.s[0] / d, a.s[1] / d, a.s[2] / d});
  }
  return out;
}

std::vector<V3> downsample_to(const V3* p, std::int64_t n, std::size_t max_points, double leaf0) {
  if (static_cast<std::size_t>(n) <= max_points) return std::vector<V3>(p, p + n);
  double leaf = leaf0;
  std::vector<V3> out = voxel_downsample(p, n, leaf);
  while (out.size() > max_points) {
    leaf *= 2.0;
    out = voxel_downsample(p, n, leaf);
  }
  return out;
}

// ---------------------------------------------------------------- NNF
NnfGeometry nnf_geometry(const Aabb& b, double resolution, double padding, double max_query_dist,
                         std::size_t max_cells) {
  if (!(resolution > 0.0)) throw std::invalid_argument("build_nnf: resolution must be positive");
  if (padding < 0.0) throw std::invalid_argument("build_nnf: padding must be >= 0");
  NnfGeometry g;
  g.resolution = resolution;
  g.max_query_dist = max_query_dist;
  std::size_t cells = 1;
  for (int a = 0; a < 3; ++a) {
    const double lo = b.min[a] - padding, hi = b.max[a] + padding;
    g.origin[a] = lo;
    g.dims[a] = static_cast<int>(std::floor((hi - lo) / resolution)) + 1;
    cells *= static_cast<std::size_t>(g.dims[a]);
    if (cells > max_cells) throw std::runtime_error("build_nnf: cell count exceeds the memory budget");
  }
  g.n_cells = static_cast<std::int64_t>(cells);
  return g;
}

void build_nnf_cells(const V3* mu, std::int64_t n, const NnfGeometry& g, std::int32_t* cells) {
  const int nx = g.dims[0], ny = g.dims[1], nz = g.dims[2];
  const std::size_t nc = static_cast<std::size_t>(g.n_cells);
  // Occupancy of point cells, then Chebyshev dilation by hop_cap: exactly the
  // set of cells the reference BFS reaches (nnf.cpp:40-80).
  std::vector<std::uint8_t> m(nc, 0), t(nc, 0);
  for (std::int64_t i = 0; i < n; ++i) {
    int c[3];
    for (int a = 0; a < 3; ++a)
      c[a] = std::clamp(static_cast<int>(std::floor((mu[i][a] - g.origin[a]) / g.resolution)), 0, g.dims[a] - 1);
    m[(static_cast<std::size_t>(c[2]) * ny + c[1]) * nx + c[0]] = 1;
  }
  const int hop = static_cast<int>(std::ceil(g.max_query_dist / g.resolution)) + 2;
  auto dilate = [&](std::vector<std::uint8_t>& src, std::vector<std::uint8_t>& dst, int axis) {
    const int len = g.dims[axis];
    const std::size_t stride = axis == 0 ? 1 : (axis == 1 ? static_cast<std::size_t>(nx) : static_cast<std::size_t>(nx) * ny);
    const std::size_t lines = nc / static_cast<std::size_t>(len);
#pragma omp parallel for schedule(static)
    for (std::int64_t l = 0; l < static_cast<std::int64_t>(lines); ++l) {
      std::size_t base;
      if (axis == 0) {
        base = static_cast<std::size_t>(l) * nx;
      } else if (axis == 1) {
        const std::size_t z = static_cast<std::size_t>(l) / nx, x = static_cast<std::size_t>(l) % nx;
        base = z * nx * ny + x;
      } else {
        base = static_cast<std::size_t>(l);
      }
      int last = -(1 << 30);  // last occupied index seen so far (forward pass)
      for (int i = 0; i < len; ++i) {
        if (src[base + stride * i]) last = i;
        dst[base + stride * i] = (i - last) <= hop;
      }
      last = 1 << 30;
      for (int i = len - 1; i >= 0; --i) {
        if (src[base + stride * i]) last = i;
        if (last - i <= hop) dst[base + stride * i] = 1;
      }
    }
  };
  dilate(m, t, 0);
  dilate(t, m, 1);
  dilate(m, t, 2);
  const PointGrid grid(mu, n, g.resolution);
#pragma omp parallel for schedule(dynamic, 16)
  for (std::int64_t z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        const std::size_t c = (static_cast<std::size_t>(z) * ny + y) * nx + x;
        if (!t[c]) {
          cells[c] = -1;
          continue;
        }
        const V3 center{g.origin[0] + g.resolution * (x + 0.5), g.origin[1] + g.resolution * (y + 0.5),
                        g.origin[2] + g.resolution * (static_cast<double>(z) + 0.5)};
        cells[c] = grid.nearest_within(center, g.max_query_dist);
      }
}

}  // namespace smcl::host
