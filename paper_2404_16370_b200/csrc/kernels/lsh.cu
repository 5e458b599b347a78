// K3-K7: the LSH neighbour pass (reference neighbor_search.cpp:61-192,
// neighbor_graph.hpp:47-90, particle_set.cpp:7-47).
//   K3 lsh_keys     fp64 SE3 log in the pass frame -> 6-D cell -> XOR-prime
//                   hash -> 64-bit key [bucket | priority | index]   (bit exact)
//   sort            CUB radix sort of the unique keys (all 64 bits)
//   K4 reorder      gather-permute of the particle state + list remap
//   K5 segments     bucket runs from head flags + prefix sum
//   K6/K7           fused refresh + gather/offer, one thread per sorted
//                   position, lists staged in shared memory
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>

#include "../engine.cuh"
#include "../kernels.cuh"

namespace smcl {

namespace {

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

__constant__ uint64_t c_primes[6] = {73856093ull, 19349663ull, 83492791ull, 49979687ull, 39916801ull, 15485863ull};

// neighbor_search.cpp:25-35. Casts follow x86 (out-of-range -> INT64_MIN).
__device__ __forceinline__ uint64_t lsh_hash_dev(const Pose& pose, const Pose& frame, const double noise[6],
                                                 double alpha, double sr, double st) {
  double d[6];
  se3_log(inv_compose_x(frame, pose), d);
  uint64_t h = 0;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    const double w = c < 3 ? sr : st;
    const double zeta = xadd(xmul(alpha, xmul(w, d[c])), noise[c]);
    const double f = floor(zeta);
    const int64_t cell = (f >= -9223372036854775808.0 && f < 9223372036854775808.0) ? static_cast<int64_t>(f)
                                                                                    : INT64_MIN;
    h ^= static_cast<uint64_t>(cell) * c_primes[c];
  }
  return h;
}

__global__ void k_lsh_keys(const Pose* __restrict__ poses, int64_t n, int64_t gbase, LshPass lp,
                           uint64_t* __restrict__ keys) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t gi = static_cast<uint64_t>(gbase + i);
  const uint64_t h = lsh_hash_dev(poses[i], lp.frame, lp.noise, lp.alpha, lp.sigma_r, lp.sigma_t) %
                     static_cast<uint64_t>(lp.n_buckets);
  const uint64_t prio = lp.prio_bits > 0 ? mix_seed(lp.prio_seed, gi) >> (64 - lp.prio_bits) : 0;
  keys[i] = (h << (lp.prio_bits + lp.idx_bits)) | (prio << lp.idx_bits) | gi;
}

__global__ void k_hash_batch(const Pose* __restrict__ poses, int64_t n, LshPass lp, uint64_t* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = lsh_hash_dev(poses[i], lp.frame, lp.noise, lp.alpha, lp.sigma_r, lp.sigma_t);
}

// member_of[p] = key & mask; head flag of bucket runs.
__global__ void k_members(const uint64_t* __restrict__ skeys, int64_t n, uint64_t idx_mask, int shift,
                          int32_t* __restrict__ member_of, int32_t* __restrict__ head) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint64_t k = skeys[p];
  member_of[p] = static_cast<int32_t>(k & idx_mask);
  head[p] = (p == 0 || (skeys[p - 1] >> shift) != (k >> shift)) ? 1 : 0;
}

__global__ void k_inverse_perm(const int32_t* __restrict__ member_of, int64_t n, int32_t* __restrict__ new_of_old) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p < n) new_of_old[member_of[p]] = static_cast<int32_t>(p);
}

// particle_set.cpp:7-47: dst slot p takes the particle at old_of_new[p];
// list indices are remapped through new_of_old.
__global__ void k_reorder(const int32_t* __restrict__ old_of_new, const int32_t* __restrict__ new_of_old, int64_t n,
                          int k, const Pose* __restrict__ poses, const double* __restrict__ lp,
                          const int32_t* __restrict__ id, const int32_t* __restrict__ idx,
                          const float* __restrict__ kval, const int32_t* __restrict__ count, Pose* __restrict__ poses2,
                          double* __restrict__ lp2, int32_t* __restrict__ id2, int32_t* __restrict__ idx2,
                          float* __restrict__ kval2, int32_t* __restrict__ count2) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t src = old_of_new[p];
  poses2[p] = poses[src];
  lp2[p] = lp[src];
  id2[p] = id[src];
  const int c = count[src];
  count2[p] = c;
  for (int s = 0; s < k; ++s) {
    if (s < c) {
      idx2[p * k + s] = new_of_old[idx[src * k + s]];
      kval2[p * k + s] = kval[src * k + s];
    } else {  // particle_set.cpp:17-19 value-initialises the new arrays
      idx2[p * k + s] = 0;
      kval2[p * k + s] = 0.0f;
    }
  }
}

__global__ void k_segments(const int32_t* __restrict__ head, const int32_t* __restrict__ seg_id, int64_t n,
                           int32_t* __restrict__ seg_start) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p < n && head[p]) seg_start[seg_id[p] - 1] = static_cast<int32_t>(p);
}

// Bucket-size statistics (neighbor_search.cpp:172-181); integer atomics are
// order independent, so the histogram is exact.
__global__ void k_seg_stats(const int32_t* __restrict__ seg_start, int32_t n_seg, int64_t n, int cap,
                            unsigned long long* __restrict__ hist, unsigned long long* __restrict__ overflow) {
  // Block-private histogram in shared memory, one global atomic per bin per block.
  extern __shared__ unsigned long long s_hist[];  // cap + 3 (last = overflow)
  for (int b = threadIdx.x; b < cap + 3; b += blockDim.x) s_hist[b] = 0ull;
  __syncthreads();
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < n_seg;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t end = s + 1 < n_seg ? seg_start[s + 1] : n;
    const int64_t size = end - seg_start[s];
    const int64_t bin = size < cap + 1 ? size : cap + 1;
    atomicAdd(s_hist + bin, 1ull);
    if (size > cap) atomicAdd(s_hist + cap + 2, static_cast<unsigned long long>(size - cap));
  }
  __syncthreads();
  for (int b = threadIdx.x; b < cap + 2; b += blockDim.x)
    if (s_hist[b]) atomicAdd(hist + b, s_hist[b]);
  if (threadIdx.x == 0 && s_hist[cap + 2]) atomicAdd(overflow, s_hist[cap + 2]);
}

// Exact float kernel value of the pair (a, b) (neighbor_graph.hpp:84-86,
// neighbor_search.cpp:161-166): 0 if the translation bound underflows, else
// (float)exp(-q) with q from the full SE3 log in the reference's order.
__device__ __forceinline__ float kval_exact(const Pose& a, const Pose& b, double sr, double st) {
  if (kernel_underflows(a, b, st)) return 0.0f;
  double d[6];
  se3_log(inv_compose_x(a, b), d);
  return __double2float_rn(exp(-kernel_q(d, sr, st)));
}

// Lower bound of the kernel exponent q = sr |w|^2 + st |v|^2 of the pair:
// |w| = rotation angle of Ra^T Rb, and |v| >= |tb - ta| because V^-1 of the
// SE3 log expands (svgd.hpp:40-44). fp32 acos with a 2e-3 rad margin covers
// its rounding and the <= 1e-7 non-orthonormality renormalize_if_needed allows.
__device__ __forceinline__ double q_lower_bound(const Pose& a, const Pose& b, double sr, double st) {
  double tr = 0.0;
#pragma unroll
  for (int q = 0; q < 9; ++q) tr = fma(a.R[q], b.R[q], tr);
  const float c = fminf(1.0f, fmaxf(-1.0f, static_cast<float>(0.5 * (tr - 1.0))));
  const float th = fmaxf(0.0f, acosf(c) - 2e-3f);
  const double d0 = b.t[0] - a.t[0], d1 = b.t[1] - a.t[1], d2 = b.t[2] - a.t[2];
  return (sr * static_cast<double>(th) * static_cast<double>(th) + st * (d0 * d0 + d1 * d1 + d2 * d2)) *
         (1.0 - 1e-9);
}

// Fused NeighborGraph::refresh (neighbor_graph.hpp:76-90) and the gather/offer
// loop (neighbor_search.cpp:151-169) for the particle at sorted position p.
// Refresh and gather of one particle touch only its own list, so fusing them
// per particle preserves the reference's two-phase result exactly. Two exact
// shortcuts avoid SE3 logs whose outcome is already decided:
//  * offer() ignores duplicates before looking at k_ij;
//  * with a full list, a candidate whose kernel upper bound exp(-q_lb) does
//    not exceed the weakest non-self entry can never be inserted.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_refresh_gather(const Pose* __restrict__ all_poses, int64_t n,
                                                          int64_t gbase, const int32_t* __restrict__ pos_list,
                                                          const int32_t* __restrict__ member_of,
                                                          const int32_t* __restrict__ seg_id,
                                                          const int32_t* __restrict__ seg_start, int32_t n_seg,
                                                          int64_t n_sorted, int32_t* __restrict__ idx,
                                                          float* __restrict__ kval, int32_t* __restrict__ count, int k,
                                                          int cap, double sr, double st) {
  extern __shared__ unsigned char rg_smem[];
  int32_t* s_idx = reinterpret_cast<int32_t*>(rg_smem);         // [k][BLOCK]
  float* s_kv = reinterpret_cast<float*>(s_idx + k * BLOCK);    // [k][BLOCK]
  const int t = threadIdx.x;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * BLOCK + t;
  if (r >= n) return;
  // Sorted position handled by this thread: the shard's owned positions in
  // sorted order (pos_list), or all positions on an unsharded engine.
  const int64_t gp = pos_list ? static_cast<int64_t>(pos_list[r]) : r;
  const int32_t gi = member_of[gp];                       // global particle index
  const int64_t li = static_cast<int64_t>(gi) - gbase;    // local storage slot
  const int32_t seg = seg_id[gp] - 1;
  const int64_t rb = seg_start[seg];
  const int64_t re = seg + 1 < n_seg ? seg_start[seg + 1] : n_sorted;
  const int64_t vis_end = re < rb + cap ? re : rb + cap;

  int cnt = count[li];
  for (int s = 0; s < cnt; ++s) s_idx[s * BLOCK + t] = idx[li * k + s];
  const Pose pi = all_poses[gi];
  for (int s = 0; s < cnt; ++s) {  // refresh
    const int32_t j = s_idx[s * BLOCK + t];
    s_kv[s * BLOCK + t] = (j == gi) ? 1.0f : kval_exact(pi, all_poses[j], sr, st);
  }
  // Weakest non-self entry (first strict minimum, neighbor_graph.hpp:60-72)
  // and its threshold in exponent space.
  int weakest = -1;
  float wk = __int_as_float(0x7f800000);
  double q_skip = 0.0;
  auto find_weakest = [&]() {
    weakest = -1;
    wk = __int_as_float(0x7f800000);
    for (int s = 0; s < cnt; ++s) {
      if (s_idx[s * BLOCK + t] == gi) continue;
      const float v = s_kv[s * BLOCK + t];
      if (v < wk) {
        wk = v;
        weakest = s;
      }
    }
    // k_ij <= exp(-q_lb) <= wk  <=>  q_lb >= -log(wk); 0.0f entries: only
    // k_ij that round to 0.0f (q > 150 ln 2) are excluded.
    q_skip = weakest < 0 ? 1e300 : (wk > 0.0f ? -log(static_cast<double>(wk)) * (1.0 + 1e-12) + 1e-12 : 104.0);
  };
  if (cnt == k) find_weakest();
  for (int64_t q = rb; q < vis_end; ++q) {  // gather / offer
    const int32_t j = member_of[q];
    if (j == gi) continue;
    bool dup = false;
    for (int s = 0; s < cnt; ++s) dup |= (s_idx[s * BLOCK + t] == j);
    if (dup) continue;
    const Pose pj = all_poses[j];
    if (cnt == k && (weakest < 0 || q_lower_bound(pi, pj, sr, st) >= q_skip)) continue;
    const float kij = kval_exact(pi, pj, sr, st);
    if (cnt < k) {
      s_idx[cnt * BLOCK + t] = j;
      s_kv[cnt * BLOCK + t] = kij;
      ++cnt;
      if (cnt == k) find_weakest();
      continue;
    }
    if (kij > wk) {
      s_idx[weakest * BLOCK + t] = j;
      s_kv[weakest * BLOCK + t] = kij;
      find_weakest();
    }
  }
  count[li] = cnt;
  for (int s = 0; s < cnt; ++s) {
    idx[li * k + s] = s_idx[s * BLOCK + t];
    kval[li * k + s] = s_kv[s * BLOCK + t];
  }
}

}  // namespace

void launch_lsh_keys(const Pose* poses, int64_t n, int64_t gbase, const LshPass& lp, uint64_t* keys, cudaStream_t st) {
  count_launch();
  if (n > 0) k_lsh_keys<<<blocks_for(n, 128), 128, 0, st>>>(poses, n, gbase, lp, keys);
}
void launch_hash_batch(const Pose* poses, int64_t n, const LshPass& lp, uint64_t* out, cudaStream_t st) {
  count_launch();
  if (n > 0) k_hash_batch<<<blocks_for(n, 128), 128, 0, st>>>(poses, n, lp, out);
}

size_t sort_temp_bytes(int64_t n) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, a, static_cast<const uint64_t*>(nullptr), static_cast<uint64_t*>(nullptr),
                                 static_cast<int>(n), 0, 64);
  cub::DeviceScan::InclusiveSum(nullptr, b, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                static_cast<int>(n));
  return a > b ? a : b;
}

void sort_keys(const uint64_t* in, uint64_t* out, int64_t n, int end_bit, void* temp, size_t temp_bytes,
               cudaStream_t st) {
  cub::DeviceRadixSort::SortKeys(temp, temp_bytes, in, out, static_cast<int>(n), 0, end_bit, st);
}

void launch_members(const uint64_t* skeys, int64_t n, uint64_t idx_mask, int shift, int32_t* member_of, int32_t* head,
                    cudaStream_t st) {
  count_launch();
  if (n > 0) k_members<<<blocks_for(n, 256), 256, 0, st>>>(skeys, n, idx_mask, shift, member_of, head);
}

void inclusive_sum_i32(const int32_t* in, int32_t* out, int64_t n, void* temp, size_t temp_bytes, cudaStream_t st) {
  cub::DeviceScan::InclusiveSum(temp, temp_bytes, in, out, static_cast<int>(n), st);
}

void launch_inverse_perm(const int32_t* member_of, int64_t n, int32_t* new_of_old, cudaStream_t st) {
  count_launch();
  if (n > 0) k_inverse_perm<<<blocks_for(n, 256), 256, 0, st>>>(member_of, n, new_of_old);
}

void launch_reorder(const int32_t* old_of_new, const int32_t* new_of_old, int64_t n, int k, const Pose* poses,
                    const double* lp, const int32_t* id, const int32_t* idx, const float* kval, const int32_t* count,
                    Pose* poses2, double* lp2, int32_t* id2, int32_t* idx2, float* kval2, int32_t* count2,
                    cudaStream_t st) {
  count_launch();
  if (n > 0)
    k_reorder<<<blocks_for(n, 128), 128, 0, st>>>(old_of_new, new_of_old, n, k, poses, lp, id, idx, kval, count, poses2,
                                                  lp2, id2, idx2, kval2, count2);
}

void launch_segments(const int32_t* head, const int32_t* seg_id, int64_t n, int32_t* seg_start, cudaStream_t st) {
  count_launch();
  if (n > 0) k_segments<<<blocks_for(n, 256), 256, 0, st>>>(head, seg_id, n, seg_start);
}

void launch_seg_stats(const int32_t* seg_start, int32_t n_seg, int64_t n, int cap, unsigned long long* hist,
                      unsigned long long* overflow, cudaStream_t st) {
  count_launch();
  if (n_seg > 0) {
    const unsigned g = static_cast<unsigned>(std::min<int64_t>(blocks_for(n_seg, 256), 296));
    k_seg_stats<<<g, 256, sizeof(unsigned long long) * (cap + 3), st>>>(seg_start, n_seg, n, cap, hist, overflow);
  }
}

void launch_refresh_gather(const Pose* all_poses, int64_t n, int64_t gbase, const int32_t* pos_list,
                           const int32_t* member_of,
                           const int32_t* seg_id, const int32_t* seg_start, int32_t n_seg, int64_t n_sorted,
                           int32_t* idx, float* kval, int32_t* count, int k, int cap, double sr, double st_,
                           cudaStream_t st) {
  count_launch();
  constexpr int B = 64;
  if (n > 0)
    k_refresh_gather<B><<<blocks_for(n, B), B, static_cast<size_t>(k) * B * 8, st>>>(all_poses, n, gbase, pos_list, member_of, seg_id, seg_start, n_seg,
                                                         n_sorted, idx, kval, count, k, cap, sr, st_);
}

}  // namespace smcl
