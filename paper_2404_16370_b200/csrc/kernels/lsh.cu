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
#include <cstdio>
#include <cstdlib>

#include "../engine.cuh"
#include "../kernels.cuh"

namespace smcl {

namespace {

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

// neighbor_search.cpp:20-21 (host and device; c is a compile-time index after unrolling)
__host__ __device__ __forceinline__ uint64_t lsh_prime(int c) {
  return c == 0 ? 73856093ull
                : c == 1 ? 19349663ull : c == 2 ? 83492791ull : c == 3 ? 49979687ull : c == 4 ? 39916801ull : 15485863ull;
}

// neighbor_search.cpp:25-35 on the host (glibc atan2 / sin, as the reference)
// and on the device (CUDA libm). Casts follow x86 (out-of-range -> INT64_MIN).
//
// Near-integer guard (device): CUDA's atan2 / sin differ from glibc's by up
// to ~2 ulp (glibc's are not correctly rounded either: ~0.1 % of arguments
// are 1 ulp off), so a cell coordinate zeta within a few ulp of an integer
// (or a rotation angle at one of se3_log's branch thresholds) may floor
// differently from the reference. *amb is set when that cannot be excluded:
// |zeta - round(zeta)| below a bound on the propagated libm discrepancy,
//   G_c = 64 eps (|zeta_c| + alpha w_c (theta + |t|_1 + 1)(2 + theta / sin theta)),
// (theta / sin theta: an angle error amplified by theta / (2 sin theta) near
// pi). The engine counts flagged particles; after the step it rehashes them
// on the host with glibc (the reference's own arithmetic) and replays the
// neighbour pass onward if any key differs (engine.cu verify_lsh_guard), so
// the keys are the reference's by construction. For random poses G ~ 1e-13:
// about one flag per 10^11 hashes, i.e. the check is free.
__host__ __device__ __forceinline__ uint64_t lsh_hash_hd(const Pose& pose, const Pose& frame, const double noise[6],
                                                         double alpha, double sr, double st, bool* amb) {
  const Pose rel = inv_compose_x(frame, pose);
  double d[6];
  se3_log(rel, d);
  uint64_t h = 0;
  double zeta[6];
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    const double w = c < 3 ? sr : st;
    zeta[c] = xadd(xmul(alpha, xmul(w, d[c])), noise[c]);
    const double f = floor(zeta[c]);
    const int64_t cell = (f >= -9223372036854775808.0 && f < 9223372036854775808.0) ? static_cast<int64_t>(f)
                                                                                    : INT64_MIN;
    h ^= static_cast<uint64_t>(cell) * lsh_prime(c);
  }
#ifdef __CUDA_ARCH__
  if (amb) {
    constexpr double kEps = 2.220446049250313e-16;
    const double th = sqrt(fma(d[0], d[0], fma(d[1], d[1], d[2] * d[2])));
    const double tn = fabs(rel.t[0]) + fabs(rel.t[1]) + fabs(rel.t[2]);
    const double amp = 2.0 + (th > 1e-300 ? th / fmax(sin(th), 1e-300) : 1.0);
    bool a = fabs(th - (kPi - 1e-6)) <= 1e-9 || fabs(th - 1e-8) <= 1e-17 || fabs(th * th - 1e-8) <= 1e-17;
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      const double w = c < 3 ? sr : st;
      const double g = 64.0 * kEps * (fabs(zeta[c]) + alpha * w * (th + tn + 1.0) * amp);
      const double fr = zeta[c] - floor(zeta[c]);
      a = a || !(fr >= g && 1.0 - fr >= g) || !(fabs(zeta[c]) < 1e15);
    }
    *amb = a;
  }
#else
  if (amb) *amb = false;
#endif
  return h;
}

__global__ void k_lsh_keys(const Pose* __restrict__ poses, int64_t n, int64_t gbase, LshPass lp,
                           uint64_t* __restrict__ keys, unsigned* __restrict__ flagged) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t gi = static_cast<uint64_t>(gbase + i);
  bool amb = false;
  const uint64_t h = lsh_hash_hd(poses[i], lp.frame, lp.noise, lp.alpha, lp.sigma_r, lp.sigma_t, &amb) %
                     static_cast<uint64_t>(lp.n_buckets);
  const uint64_t prio = lp.prio_bits > 0 ? mix_seed(lp.prio_seed, gi) >> (64 - lp.prio_bits) : 0;
  keys[i] = (h << (lp.prio_bits + lp.idx_bits)) | (prio << lp.idx_bits) | gi;
  if (amb && flagged) {  // flagged[0] = count, flagged[1 ..] = the first kGuardListCap local indices
    const unsigned s = atomicAdd(flagged, 1u);
    if (s < static_cast<unsigned>(kGuardListCap)) flagged[1 + s] = static_cast<unsigned>(i);
  }
}

// The flagged particles' poses and keys, gathered for the host check.
__global__ void k_gather_flagged(const Pose* __restrict__ poses, const uint64_t* __restrict__ keys,
                                 const unsigned* __restrict__ list, int m, Pose* __restrict__ out_pose,
                                 uint64_t* __restrict__ out_key) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  out_pose[q] = poses[list[q]];
  out_key[q] = keys[list[q]];
}
__global__ void k_scatter_keys(uint64_t* __restrict__ keys, const unsigned* __restrict__ list, int m,
                               const uint64_t* __restrict__ vals) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < m) keys[list[q]] = vals[q];
}

__global__ void k_hash_batch(const Pose* __restrict__ poses, int64_t n, LshPass lp, uint64_t* __restrict__ out,
                             unsigned char* __restrict__ amb_out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool amb = false;
  out[i] = lsh_hash_hd(poses[i], lp.frame, lp.noise, lp.alpha, lp.sigma_r, lp.sigma_t, &amb);
  amb_out[i] = amb ? 1 : 0;
}

// member_of[p] = key & mask; head flag of bucket runs.
// new_of_old (optional): the inverse permutation of the reorder, in the same sweep.
__global__ void k_members(const uint64_t* __restrict__ skeys, int64_t n, uint64_t idx_mask, int shift,
                          int32_t* __restrict__ member_of, int32_t* __restrict__ head,
                          int32_t* __restrict__ new_of_old) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint64_t k = skeys[p];
  const int32_t m = static_cast<int32_t>(k & idx_mask);
  member_of[p] = m;
  head[p] = (p == 0 || (skeys[p - 1] >> shift) != (k >> shift)) ? 1 : 0;
  if (new_of_old) new_of_old[m] = static_cast<int32_t>(p);
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

// K = 20 rows (80 B, 16-byte aligned): 128-bit row copies, all 20 remap
// gathers issued together, 128-bit pose copy.
// kMirror: also write the neighbour pass's fp32 pose mirror of the reordered
// poses and its max |t - c| (what k_pose_mirror computes), in the same sweep.
template <int K, bool kMirror = false>
__global__ void __launch_bounds__(128, 1) k_reorder_k(const int32_t* __restrict__ old_of_new,
                                                   const int32_t* __restrict__ new_of_old, int64_t n,
                                                   const Pose* __restrict__ poses, const double* __restrict__ lp,
                                                   const int32_t* __restrict__ id, const int32_t* __restrict__ idx,
                                                   const float* __restrict__ kval, const int32_t* __restrict__ count,
                                                   Pose* __restrict__ poses2, double* __restrict__ lp2,
                                                   int32_t* __restrict__ id2, int32_t* __restrict__ idx2,
                                                   float* __restrict__ kval2, int32_t* __restrict__ count2,
                                                   float4* __restrict__ mir = nullptr,
                                                   unsigned int* __restrict__ tmax_bits = nullptr,
                                                   double3 anc = double3{0.0, 0.0, 0.0}) {
  static_assert(K % 4 == 0, "rows must be whole 16-byte vectors");
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (kMirror) {  // the block's max |t - c| needs every thread: no early return
    float tm = 0.f;
    if (p < n) {
      const Pose q = ldg_pose(poses + old_of_new[p]);
      const float t0 = static_cast<float>(q.t[0] - anc.x), t1 = static_cast<float>(q.t[1] - anc.y),
                  t2 = static_cast<float>(q.t[2] - anc.z);
      mir[3 * p] = make_float4(q.R[0], q.R[1], q.R[2], q.R[3]);
      mir[3 * p + 1] = make_float4(q.R[4], q.R[5], q.R[6], q.R[7]);
      mir[3 * p + 2] = make_float4(q.R[8], t0, t1, t2);
      tm = fmaxf(fabsf(t0), fmaxf(fabsf(t1), fabsf(t2)));
      if (!(tm <= 3.0e38f)) tm = 3.0e38f;  // NaN / inf poses: the margin becomes useless (filter passes all)
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, o));
    __shared__ float wmax[4];  // 128 threads
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = tm;
    __syncthreads();
    if (threadIdx.x == 0) {
      const float b = fmaxf(fmaxf(wmax[0], wmax[1]), fmaxf(wmax[2], wmax[3]));
      if (b > 0.f) atomicMax(tmax_bits, __float_as_uint(b));
    }
  }
  if (p >= n) return;
  const int64_t src = old_of_new[p];
  poses2[p] = ldg_pose(poses + src);
  lp2[p] = lp[src];
  id2[p] = id[src];
  const int c = count[src];
  count2[p] = c;
  const int4* ir = reinterpret_cast<const int4*>(idx + src * K);
  const float4* kr = reinterpret_cast<const float4*>(kval + src * K);
  int j[K];
  float w[K];
#pragma unroll
  for (int v = 0; v < K / 4; ++v) {
    const int4 a = __ldg(ir + v);
    const float4 b = __ldg(kr + v);
    j[4 * v] = a.x, j[4 * v + 1] = a.y, j[4 * v + 2] = a.z, j[4 * v + 3] = a.w;
    w[4 * v] = b.x, w[4 * v + 1] = b.y, w[4 * v + 2] = b.z, w[4 * v + 3] = b.w;
  }
#pragma unroll
  for (int s = 0; s < K; ++s) {  // particle_set.cpp:17-19 value-initialises the unused slots
    j[s] = s < c ? __ldg(new_of_old + j[s]) : 0;
    w[s] = s < c ? w[s] : 0.0f;
  }
  int4* io = reinterpret_cast<int4*>(idx2 + p * K);
  float4* ko = reinterpret_cast<float4*>(kval2 + p * K);
#pragma unroll
  for (int v = 0; v < K / 4; ++v) {
    io[v] = make_int4(j[4 * v], j[4 * v + 1], j[4 * v + 2], j[4 * v + 3]);
    ko[v] = make_float4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
  }
}

// dst[p] = src[perm[p]] for whole 96-byte poses (128-bit copies).
__global__ void k_permute_poses(const int32_t* __restrict__ perm, int64_t n, const Pose* __restrict__ src,
                                Pose* __restrict__ dst) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const double2* a = reinterpret_cast<const double2*>(src + perm[p]);
  double2* b = reinterpret_cast<double2*>(dst + p);
#pragma unroll
  for (int v = 0; v < 6; ++v) b[v] = __ldg(a + v);
}

// ---- Cross-shard reorder by all-to-all (the permutation
// of particle_set.cpp:7-47 over the global sorted order). New position p
// belongs to shard p / n_local; its old state lives on shard member_of[p] /
// n_local. Every rank holds the global member_of, so the shard-to-shard count
// matrix is computed locally (no count exchange) and only the non-pose state
// moves, one record per migrating particle (poses are permuted from the
// gathered pose array instead).
struct MigHeader {
  double lp;
  int32_t id, count, pnew, pad;
};
static_assert(sizeof(MigHeader) == 24, "record header");

// mat[d * world + s] = number of new positions on shard d whose old state is on shard s.
__global__ void k_migrate_counts(const int32_t* __restrict__ member_of, int64_t n, int64_t nl, int world,
                                 unsigned int* __restrict__ mat) {
  extern __shared__ unsigned int hist[];
  const int cells = world * world;
  for (int c = threadIdx.x; c < cells; c += blockDim.x) hist[c] = 0;
  __syncthreads();
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int d = static_cast<int>(p / nl), src = static_cast<int>(member_of[p] / nl);
    atomicAdd(&hist[d * world + src], 1u);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < cells; c += blockDim.x)
    if (hist[c]) atomicAdd(&mat[c], hist[c]);
}

// Packs the records this rank sends, grouped by destination shard in rank
// order (offsets from the count matrix); order inside a destination's chunk
// is immaterial because each record carries its new position. Blocks of 256
// never straddle two destinations (n_local is a multiple of 4096).
__global__ void __launch_bounds__(256) k_migrate_pack(const int32_t* __restrict__ member_of, int64_t n, int64_t nl,
                                                      int world, int rank, const unsigned int* __restrict__ mat,
                                                      unsigned int* __restrict__ cursor, const double* __restrict__ lp,
                                                      const int32_t* __restrict__ id,
                                                      const int32_t* __restrict__ count,
                                                      const int32_t* __restrict__ idx,
                                                      const float* __restrict__ kval, int k,
                                                      unsigned char* __restrict__ send) {
  __shared__ unsigned int warp_n[8];
  __shared__ unsigned int base;
  const int64_t p = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
  const int64_t o = p < n ? static_cast<int64_t>(member_of[p]) - static_cast<int64_t>(rank) * nl : -1;
  const bool mine = p < n && o >= 0 && o < nl;
  const unsigned int bal = __ballot_sync(0xffffffffu, mine);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) warp_n[w] = __popc(bal);
  __syncthreads();
  const int d = static_cast<int>((static_cast<int64_t>(blockIdx.x) * 256) / nl);
  if (threadIdx.x == 0) {
    unsigned int tot = 0;
    for (int i = 0; i < 8; ++i) tot += warp_n[i];
    unsigned int off = 0;  // records this rank sends to shards before d
    for (int e = 0; e < d; ++e) off += mat[e * world + rank];
    base = off + (tot ? atomicAdd(&cursor[d], tot) : 0u);
  }
  __syncthreads();
  if (!mine) return;
  unsigned int pos = base + __popc(bal & ((1u << lane) - 1u));
  for (int i = 0; i < w; ++i) pos += warp_n[i];
  const size_t rec = sizeof(MigHeader) + 8 * static_cast<size_t>(k);
  unsigned char* r = send + static_cast<size_t>(pos) * rec;
  MigHeader h;
  h.lp = lp[o];
  h.id = id[o];
  h.count = count[o];
  h.pnew = static_cast<int32_t>(p);
  h.pad = 0;
  *reinterpret_cast<MigHeader*>(r) = h;
  int32_t* ri = reinterpret_cast<int32_t*>(r + sizeof(MigHeader));
  float* rk = reinterpret_cast<float*>(ri + k);
  for (int s = 0; s < k; ++s) {
    ri[s] = idx[o * k + s];
    rk[s] = kval[o * k + s];
  }
}

// Scatters the received records to their new local positions, remapping the
// neighbour ids to new global indices (particle_set.cpp:17-19 as k_reorder).
__global__ void k_migrate_unpack(const unsigned char* __restrict__ recv, int64_t nl, int64_t gbase, int k,
                                 const int32_t* __restrict__ new_of_old, double* __restrict__ lp2,
                                 int32_t* __restrict__ id2, int32_t* __restrict__ count2,
                                 int32_t* __restrict__ idx2, float* __restrict__ kval2) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= nl) return;
  const size_t rec = sizeof(MigHeader) + 8 * static_cast<size_t>(k);
  const unsigned char* r = recv + static_cast<size_t>(j) * rec;
  const MigHeader h = *reinterpret_cast<const MigHeader*>(r);
  const int32_t* ri = reinterpret_cast<const int32_t*>(r + sizeof(MigHeader));
  const float* rk = reinterpret_cast<const float*>(ri + k);
  const int64_t p = h.pnew - gbase;
  lp2[p] = h.lp;
  id2[p] = h.id;
  count2[p] = h.count;
  for (int s = 0; s < k; ++s) {
    idx2[p * k + s] = s < h.count ? new_of_old[ri[s]] : 0;
    kval2[p * k + s] = s < h.count ? rk[s] : 0.0f;
  }
}

__global__ void k_segments(const int32_t* __restrict__ head, const int32_t* __restrict__ seg_id, int64_t n,
                           int32_t* __restrict__ seg_start) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p < n && head[p]) seg_start[seg_id[p] - 1] = static_cast<int32_t>(p);
  if (p == n - 1) seg_start[seg_id[p]] = static_cast<int32_t>(n);  // sentinel: seg_start[n_seg] = n
}

// Bucket-size statistics (neighbor_search.cpp:172-181); integer atomics are
// order independent, so the histogram is exact.
__global__ void k_seg_stats(const int32_t* __restrict__ seg_start, const int32_t* __restrict__ n_seg_ptr, int cap,
                            unsigned long long* __restrict__ hist, unsigned long long* __restrict__ overflow) {
  // Block-private histogram in shared memory, one global atomic per bin per block.
  extern __shared__ unsigned long long s_hist[];  // cap + 3 (last = overflow)
  for (int b = threadIdx.x; b < cap + 3; b += blockDim.x) s_hist[b] = 0ull;
  __syncthreads();
  const int64_t n_seg = *n_seg_ptr;
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < n_seg;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t end = seg_start[s + 1];
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

// Float kernel value of a pair as the reference caches it
// (neighbor_graph.hpp:84-86, neighbor_search.cpp:161-166): 0 if the
// translation bound underflows, else (float)exp(-q) with q from the SE3 log.
//
// Fast evaluation. With Rrel = Ra^T Rb,
// vee = (Rrel - Rrel^T)^vee, s = |vee|/2, c = (tr Rrel - 1)/2, r = hypot(s, c),
// theta = atan2(s, c), the reference's log (se3.hpp:103-149) gives
// |w| = theta*r, and V^-1 acts as the identity along w and as a scaled
// rotation with |V^-1 x|^2 = |x|^2 (th/2)^2 / sin^2(th/2) across it, so
//   q = sr th^2 + st ( (u.w^)^2 + (|u|^2 - (u.w^)^2) th^2 / (4 sin^2(th/2)) ),
// u = Ra^T (tb - ta), th = theta*r. No sin/cos calls: sin/cos of th follow
// from s/r, c/r and the tiny th - theta. q agrees with the reference's to
// ~1e-14 relative; the float is returned only if exp(-q)*(1 -+ 4e-12) round
// to the same float, otherwise *ok = false and kval_of takes the reference-order log.
__device__ __forceinline__ float kval_fast(const Pose& a, const Pose& b, double sr, double st, bool* ok) {
  double m[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      m[i * 3 + j] = fma(a.R[0 * 3 + i], b.R[0 * 3 + j], fma(a.R[1 * 3 + i], b.R[1 * 3 + j], a.R[2 * 3 + i] * b.R[2 * 3 + j]));
  const double d0 = b.t[0] - a.t[0], d1 = b.t[1] - a.t[1], d2 = b.t[2] - a.t[2];
  double u[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) u[i] = fma(a.R[0 * 3 + i], d0, fma(a.R[1 * 3 + i], d1, a.R[2 * 3 + i] * d2));
  const double v0 = m[7] - m[5], v1 = m[2] - m[6], v2 = m[3] - m[1];
  const double vv = fma(v0, v0, fma(v1, v1, v2 * v2));  // |vee|^2 = 4 s^2
  const double c = fmin(1.0, fmax(-1.0, 0.5 * ((m[0] + m[4]) + m[8] - 1.0)));
  const double uu = fma(u[0], u[0], fma(u[1], u[1], u[2] * u[2]));
  double q;
  if (vv == 0.0) {  // identical rotations: w = 0, v = u
    q = st * uu;
  } else {
    const double ivs = rsqrt_nr(vv);  // 1 / |vee|
    const double s = 0.5 * (vv * ivs);
    const double theta = atan2_pos(s, c);
    if (theta > 3.14159265358979323846 - 1e-2) {  // near the pi branch: reference path
      *ok = false;
      return 0.0f;
    }
    const double r2 = fma(s, s, c * c);
    const double inv_r = rsqrt_nr(r2);
    const double r = r2 * inv_r;
    const double th = theta * r;  // |w|
    const double th2 = th * th;
    const double uw = fma(u[0], v0, fma(u[1], v1, u[2] * v2)) * ivs;
    const double par = uw * uw;  // (u . w^)^2
    const double perp = fmax(uu - par, 0.0);
    double F;  // th^2 / (4 sin^2(th/2))
    if (th2 < 1e-6) {
      F = fma(th2, fma(th2, 1.0 / 240.0, 1.0 / 12.0), 1.0);
    } else {
      const double S = s * inv_r, Cc = c * inv_r, dl = theta * (r - 1.0);  // th = theta + dl
      const double sin_th = fma(dl, Cc, S) - 0.5 * dl * dl * S;
      const double cos_th = fma(-dl, S, Cc) - 0.5 * dl * dl * Cc;
      // 4 sin^2(th/2) = 2(1 - cos th) = 2 sin^2 th / (1 + cos th)
      F = cos_th < 0.0 ? th2 * rcp_nr(2.0 * (1.0 - cos_th)) : th2 * (1.0 + cos_th) * rcp_nr(2.0 * sin_th * sin_th);
    }
    q = fma(sr, th2, st * fma(perp, F, par));
  }
  if (!(q == q)) {
    *ok = false;
    return 0.0f;
  }
  // The reference forms u as Ra^T tb + (-Ra^T ta) (se3.hpp inverse, compose):
  // both products are of size |t|, so its u carries up to ~10 ulp(|t|) of
  // cancellation error that this u = Ra^T (tb - ta) does not. The guard grows
  // with it: |dq| <= st F (2 |u| du sqrt 3 + 3 du^2), F = |V^-1|^2 <= pi^2/4,
  // du = 4e-15 (|ta| + |tb|), |u| <= (1 + |u|^2) / 2.
  const double T = fmax(fmax(fabs(a.t[0]), fabs(a.t[1])), fabs(a.t[2])) +
                   fmax(fmax(fabs(b.t[0]), fabs(b.t[1])), fabs(b.t[2]));
  const double du = 4e-15 * T;
  const double gq = 4e-12 + st * 2.5 * fma(3.5 * du, 0.5 * (1.0 + uu), 3.0 * du * du);
  const double k = exp(-q);
  const float lo = __double2float_rn(k * (1.0 - gq)), hi = __double2float_rn(k * (1.0 + gq));
  *ok = lo == hi;
  return hi;
}

// Kernel value of the pair as the reference computes it, via kval_fast when
// its float is provably the same.
__device__ __forceinline__ float kval_of(const Pose& a, const Pose& b, double sr, double st) {
  if (kernel_underflows(a, b, st)) return 0.0f;
  bool ok;
  const float f = kval_fast(a, b, sr, st, &ok);
  if (ok) return f;
  double d[6];
  se3_log(inv_compose_x(a, b), d);
  return __double2float_rn(exp(-kernel_q(d, sr, st)));
}

// Fused NeighborGraph::refresh (neighbor_graph.hpp:76-90) and the gather/offer
// loop (neighbor_search.cpp:151-169) for the particle at sorted position p.
// Refresh and gather of one particle touch only its own list, so fusing them
// per particle preserves the reference's two-phase result exactly. offer()
// ignores duplicates before looking at k_ij, so duplicates skip the kernel
// evaluation; every evaluation goes through kval_of (bit-exact float).
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_refresh_gather(const Pose* __restrict__ all_poses, int64_t n,
                                                          int64_t gbase, const int32_t* __restrict__ pos_list,
                                                          const int32_t* __restrict__ member_of,
                                                          const int32_t* __restrict__ seg_id,
                                                          const int32_t* __restrict__ seg_start,
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
  const int64_t re = seg_start[seg + 1];  // sentinel seg_start[n_seg] = n
  const int64_t vis_end = re < rb + cap ? re : rb + cap;

  int cnt = count[li];
  for (int s = 0; s < cnt; ++s) s_idx[s * BLOCK + t] = idx[li * k + s];
  const Pose pi = ldg_pose(all_poses + gi);
  for (int s = 0; s < cnt; ++s) {  // refresh
    const int32_t j = s_idx[s * BLOCK + t];
    s_kv[s * BLOCK + t] = (j == gi) ? 1.0f : kval_of(pi, ldg_pose(all_poses + j), sr, st);
  }
  // Weakest non-self entry (first strict minimum, neighbor_graph.hpp:60-72).
  int weakest = -1;
  float wk = __int_as_float(0x7f800000);
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
  };
  if (cnt == k) find_weakest();
  for (int64_t q = rb; q < vis_end; ++q) {  // gather / offer
    const int32_t j = member_of[q];
    if (j == gi) continue;
    bool dup = false;
    for (int s = 0; s < cnt; ++s) dup |= (s_idx[s * BLOCK + t] == j);
    if (dup) continue;
    if (cnt == k && weakest < 0) continue;  // self-only full list (k == 1): nothing evictable
    const float kij = kval_of(pi, ldg_pose(all_poses + j), sr, st);
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

// fp32 mirror of the poses for the window filter: (R0..R3), (R4..R7),
// (R8, t - c) with c a per-pass anchor, plus max |t - c|_inf of all particles
// (float bits, atomicMax) that sizes the filter's rounding margin.
__global__ void k_pose_mirror(const Pose* __restrict__ poses, int64_t n, double3 c, float4* __restrict__ mir,
                              unsigned int* __restrict__ tmax_bits) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  float tm = 0.f;
  if (i < n) {
    const Pose p = ldg_pose(poses + i);
    const float t0 = static_cast<float>(p.t[0] - c.x), t1 = static_cast<float>(p.t[1] - c.y),
                t2 = static_cast<float>(p.t[2] - c.z);
    mir[3 * i] = make_float4(p.R[0], p.R[1], p.R[2], p.R[3]);
    mir[3 * i + 1] = make_float4(p.R[4], p.R[5], p.R[6], p.R[7]);
    mir[3 * i + 2] = make_float4(p.R[8], t0, t1, t2);
    tm = fmaxf(fabsf(t0), fmaxf(fabsf(t1), fabsf(t2)));
    if (!(tm <= 3.0e38f)) tm = 3.0e38f;  // NaN / inf poses: the margin becomes useless (filter passes all)
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, o));
  __shared__ float wmax[8];  // launched with 256 threads: one atomic per block
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = tm;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = 0.f;
    for (int w = 0; w < 8; ++w) b = fmaxf(b, wmax[w]);
    if (b > 0.f) atomicMax(tmax_bits, __float_as_uint(b));
  }
}

// Filtered variant of k_refresh_gather (same results). Once the list is full,
// a candidate is inserted only if its float kernel value beats the weakest
// entry wk, and wk never decreases during the window scan. The reference's
// q = sr|w|^2 + st|V^-1 u|^2 (svgd.hpp:30-44) satisfies |w|^2 = theta^2 >=
// 2(1 - cos theta) = 3 - tr(Ra^T Rb) and |V^-1 u| >= |u| = |tb - ta| (V^-1
// scales the plane across w by (theta/2)/sin(theta/2) >= 1), so
//   q >= L = sr (3 - tr(Ra^T Rb)) + st |tb - ta|^2
// and L > -log(wk) proves float(exp(-q)) <= wk: the offer would be dropped
// whatever the list holds. L is evaluated in fp32 on the pose mirror
// (k_pose_mirror) and only trusted beyond its rounding margin (kernel prologue).
// Duplicates: offer() ignores a candidate already listed. Window members are
// unique, so a member inserted during the scan is never offered again, and a
// member listed at the start that gets evicted before its turn is never
// re-inserted (it was the weakest, kv = wk_then <= wk_now, and an insert needs
// kij > wk_now with kij = the same float). Hence "duplicate" = "listed before
// the window scan": a 64-bit mask over window offsets (cap <= 64) marks those
// members and the filter drops them before any evaluation.
// Each lane filters its window into a chunk of up to kRgChunk survivors; the
// warp evaluates all lanes' survivors together (full-width kval_of), then each
// lane replays its offers in window order.
constexpr int kRgChunk = 16;


// SMCL_RG_STATS=1 (diagnostics only): window members considered, survivors
// of the filter (exact evaluations), insertions, refresh evaluations.
__device__ unsigned long long g_rg_stats[4];

// 8 CTAs x 2 warps per SM: 128 registers without spills (a window-evaluation
// pose prefetch measured slower: 184 registers 2.03 ms, capped at 128 with
// spills 1.69, against 1.48).
template <int BLOCK, int KMAX, bool kStats = false>
__global__ void __launch_bounds__(BLOCK, 8) k_refresh_gather_f(const Pose* __restrict__ all_poses, int64_t n,
                                                            int64_t gbase, const int32_t* __restrict__ pos_list,
                                                            const int32_t* __restrict__ member_of,
                                                            const int32_t* __restrict__ seg_id,
                                                            const int32_t* __restrict__ seg_start,
                                                            int64_t n_sorted, const int32_t* __restrict__ pos_of,
                                                            int32_t* __restrict__ idx,
                                                            float* __restrict__ kval, int32_t* __restrict__ count,
                                                            int k, int cap, double sr, double st,
                                                            const float4* __restrict__ mir,
                                                            const unsigned int* __restrict__ tmax_bits,
                                                            bool members_identity) {
  extern __shared__ __align__(16) unsigned char rg_smem[];
  int32_t* s_idx = reinterpret_cast<int32_t*>(rg_smem);                  // [k][BLOCK]
  // List values per thread row [BLOCK][KMAX] (16-byte aligned rows: the
  // weakest-entry scan reads them with 128-bit loads). Empty slots and the
  // self slot hold +inf while the window is scanned, so the scan is a plain
  // first-strict-minimum; self's 1.0f is restored on write-out.
  float* s_kv = reinterpret_cast<float*>(s_idx + k * BLOCK);             // [BLOCK][KMAX]
  int32_t* s_cand = reinterpret_cast<int32_t*>(s_kv + KMAX * BLOCK);     // [kRgChunk][BLOCK]
  float* s_ckv = reinterpret_cast<float*>(s_cand + kRgChunk * BLOCK);    // [kRgChunk][BLOCK]
  int32_t* s_gi = reinterpret_cast<int32_t*>(s_ckv + kRgChunk * BLOCK);  // [BLOCK]
  uint16_t* s_flat = reinterpret_cast<uint16_t*>(s_gi + BLOCK);          // [BLOCK/32][32*kRgChunk]
  const unsigned FULL = 0xffffffffu;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  uint16_t* w_flat = s_flat + wid * 32 * kRgChunk;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * BLOCK + t;
  const bool active = r < n;
  int32_t gi = -1;
  int64_t li = 0, q = 0, q_end = 0, rb = 0;
  int cnt = 0;
  unsigned long long listed = 0ull;  // window offsets (q - rb) of the members listed before the scan
  if (active) {
    const int64_t gp = pos_list ? static_cast<int64_t>(pos_list[r]) : r;
    gi = member_of[gp];
    li = static_cast<int64_t>(gi) - gbase;
    const int32_t seg = seg_id[gp] - 1;
    rb = seg_start[seg];
    const int64_t re = seg_start[seg + 1];  // sentinel seg_start[n_seg] = n
    q = rb;
    q_end = re < rb + cap ? re : rb + cap;
    cnt = count[li];
    for (int s = 0; s < cnt; ++s) {
      const int32_t e = idx[li * k + s];
      s_idx[s * BLOCK + t] = e;
      // sorted position of the listed particle (identity after a reorder)
      const int64_t o = static_cast<int64_t>(pos_of ? pos_of[e] : e) - rb;
      if (o >= 0 && o < q_end - rb) listed |= 1ull << o;
    }
    const Pose pi = ldg_pose(all_poses + gi);
#pragma unroll
    for (int s = 0; s < KMAX; ++s) s_kv[t * KMAX + s] = __int_as_float(0x7f800000);
    // refresh (neighbor_graph.hpp:76-90); self stays +inf (see above). The
    // next entry's pose is loaded while the current one is evaluated.
    Pose nxt;
    if (cnt > 0) nxt = ldg_pose(all_poses + s_idx[t]);
    for (int s = 0; s < cnt; ++s) {
      const int32_t j = s_idx[s * BLOCK + t];
      const Pose pj = nxt;
      if (s + 1 < cnt) nxt = ldg_pose(all_poses + s_idx[(s + 1) * BLOCK + t]);
      if (j != gi) s_kv[t * KMAX + s] = kval_of(pi, pj, sr, st);
    }
    if (kStats) atomicAdd(&g_rg_stats[3], static_cast<unsigned long long>(cnt > 0 ? cnt - 1 : 0));
  }
  s_gi[t] = gi;
  // Rounding margins of the fp32 filter. Mirror rotations carry 2^-24 relative
  // error per entry: |tr32 - tr| <= 4e-6. Mirror translations (|t - c| <=
  // tmax) carry tmax 2^-24 each: |dt32 - dt| <= eps = tmax 2^-22 per axis;
  // where the bound can matter (st |dt|^2 <= 110 + margin) |dt| <= D =
  // sqrt(120 / st), so |uu32 - uu| <= 2 sqrt(3) D eps + 3 eps^2 + 3 D^2 2^-22.
  const float sr32 = static_cast<float>(sr), st32 = static_cast<float>(st);
  float mt, mL;
  {
    const double tmax = static_cast<double>(__uint_as_float(*tmax_bits));
    const double eps = tmax * 0x1p-22, D = sqrt(120.0 / st);
    const double duu = 2.0 * 1.7320508075688772 * D * eps + 3.0 * eps * eps + 3.0 * D * D * 0x1p-22;
    mt = static_cast<float>(st * duu * 1.01 + 1e-6);
    mL = static_cast<float>(sr * 4e-6 + st * duu * 1.01 + 1e-5);
    if (!(mL < 1e30f)) mt = mL = 3.0e38f;  // huge or non-finite poses: filter off
  }
  // Self never leaves its slot (offers never evict it): locate it once, so the
  // weakest-entry scan reads only values. Loops run over KMAX >= k slots,
  // unrolled and predicated.
  int self_slot = -1;
#pragma unroll
  for (int s = 0; s < KMAX; ++s)
    if (s < cnt && s_idx[s * BLOCK + t] == gi) self_slot = s;
  int weakest = -1;
  float wk = __int_as_float(0x7f800000);
  auto find_weakest = [&]() {  // first strict minimum (neighbor_graph.hpp:60-72)
    weakest = -1;
    wk = __int_as_float(0x7f800000);
    const float4* row = reinterpret_cast<const float4*>(s_kv + t * KMAX);
#pragma unroll
    for (int v4 = 0; v4 < KMAX / 4; ++v4) {
      const float4 a = row[v4];
      const float vals[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (vals[u] < wk) {
          wk = vals[u];
          weakest = 4 * v4 + u;
        }
    }
  };
  if (active && cnt == k) find_weakest();

  while (__any_sync(FULL, q < q_end)) {
    // ---- filter (no list access): up to kRgChunk survivors in window order
    const bool full = cnt == k;
    double thr = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    if (full && wk > 0.0f) thr = -log(static_cast<double>(wk));
    int ns = 0;
    if (active) {
      // fp32 bound on the mirror: L32 - margin > thr proves L > thr (and
      // st |dt|^2 - margin_t > 110 proves the translation underflow).
      const float thr32 = static_cast<float>(thr);
      const float4 a0 = __ldg(mir + 3 * gi), a1 = __ldg(mir + 3 * gi + 1), a2 = __ldg(mir + 3 * gi + 2);
      // Members are examined kFB at a time: their member_of and mirror loads
      // are all issued before any test (the loop is load-latency bound), then
      // the survivors are appended in window order until the chunk is full;
      // the thresholds only change in the offer phase, so batching leaves the
      // survivor sequence unchanged. A member not consumed because the chunk
      // filled up is examined again in the next chunk, as in the serial loop.
      constexpr int kFB = 4;
      while (q < q_end && ns < kRgChunk) {
        int32_t jj[kFB];
        bool cand[kFB];
#pragma unroll
        for (int u = 0; u < kFB; ++u) {
          const int64_t qq = q + u;
          const bool in = qq < q_end && !((listed >> (qq - rb)) & 1ull);  // listed: a duplicate offer (also self)
          jj[u] = in ? (members_identity ? static_cast<int32_t>(qq) : member_of[qq]) : gi;
          cand[u] = in;
        }
#pragma unroll
        for (int u = 0; u < kFB; ++u) cand[u] = cand[u] && jj[u] != gi;
        bool pass[kFB];
        if (full) {
          float4 b0[kFB], b1[kFB], b2[kFB];
#pragma unroll
          for (int u = 0; u < kFB; ++u) {
            const int32_t j = cand[u] ? jj[u] : gi;
            b0[u] = __ldg(mir + 3 * j);
            b1[u] = __ldg(mir + 3 * j + 1);
            b2[u] = __ldg(mir + 3 * j + 2);
          }
#pragma unroll
          for (int u = 0; u < kFB; ++u) {
            const float d0 = b2[u].y - a2.y, d1 = b2[u].z - a2.z, d2 = b2[u].w - a2.w;
            const float uu = fmaf(d0, d0, fmaf(d1, d1, d2 * d2));
            const float tr = fmaf(a0.x, b0[u].x, fmaf(a0.y, b0[u].y, fmaf(a0.z, b0[u].z, a0.w * b0[u].w))) +
                             fmaf(a1.x, b1[u].x, fmaf(a1.y, b1[u].y, fmaf(a1.z, b1[u].z, a1.w * b1[u].w))) +
                             a2.x * b2[u].x;
            const float L = fmaf(sr32, 3.0f - tr, st32 * uu);
            // kernel_underflows (k = 0 <= wk), or float(exp(-q)) <= wk: dropped;
            // a self-only full list (k == 1) has nothing evictable
            pass[u] = cand[u] && weakest >= 0 && !(fmaf(st32, uu, -mt) > 110.0f) &&
                      !(L * (1.0f - 1e-5f) - mL > thr32);
          }
        } else {
#pragma unroll
          for (int u = 0; u < kFB; ++u) pass[u] = cand[u];
        }
        int used = kFB;
#pragma unroll
        for (int u = 0; u < kFB; ++u) {
          if (u < used && q + u < q_end) {
            if (kStats && cand[u]) atomicAdd(&g_rg_stats[0], 1ull);
            if (pass[u]) {
              s_cand[ns * BLOCK + t] = jj[u];
              ++ns;
              if (ns == kRgChunk) used = u + 1;  // chunk full: the rest of the batch waits
            }
          }
        }
        q += used;
      }
      if (kStats) atomicAdd(&g_rg_stats[1], static_cast<unsigned long long>(ns));
    }
    // ---- warp-wide evaluation of all lanes' survivors
    int incl = ns;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(FULL, incl, 31);
    for (int s = 0, f = incl - ns; s < ns; ++s, ++f) w_flat[f] = static_cast<uint16_t>((lane << 5) | s);
    __syncwarp();
    for (int f = lane; f < total; f += 32) {
      const int e = w_flat[f];
      const int ot = (wid << 5) | (e >> 5), sl = e & 31;
      s_ckv[sl * BLOCK + ot] =
          kval_of(ldg_pose(all_poses + s_gi[ot]), ldg_pose(all_poses + s_cand[sl * BLOCK + ot]), sr, st);
    }
    __syncwarp();
    // ---- offers in window order (neighbor_graph.hpp:47-74)
    for (int s = 0; s < ns; ++s) {
      const float kij = s_ckv[s * BLOCK + t];
      if (cnt == k && !(weakest >= 0 && kij > wk)) continue;  // dropped
      const int32_t j = s_cand[s * BLOCK + t];
      if (kStats) atomicAdd(&g_rg_stats[2], 1ull);
      if (cnt < k) {
        s_idx[cnt * BLOCK + t] = j;
        s_kv[t * KMAX + cnt] = kij;
        ++cnt;
        if (cnt == k) find_weakest();
        continue;
      }
      s_idx[weakest * BLOCK + t] = j;
      s_kv[t * KMAX + weakest] = kij;
      find_weakest();
    }
    __syncwarp();
  }
  if (active) {
    count[li] = cnt;
    for (int s = 0; s < cnt; ++s) {
      idx[li * k + s] = s_idx[s * BLOCK + t];
      kval[li * k + s] = s == self_slot ? 1.0f : s_kv[t * KMAX + s];
    }
  }
}

// Sharded pass: flag sorted positions whose particle this shard owns, then
// scatter them (inclusive-sum ranks) into a dense list in sorted order.
__global__ void k_owned_flags(const int32_t* __restrict__ member_of, int64_t n, int64_t gbase, int64_t n_local,
                              int32_t* __restrict__ flag) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t gi = member_of[p];
  flag[p] = (gi >= gbase && gi < gbase + n_local) ? 1 : 0;
}
__global__ void k_owned_scatter(const int32_t* __restrict__ flag, const int32_t* __restrict__ incl, int64_t n,
                                int32_t* __restrict__ pos_list) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p < n && flag[p]) pos_list[incl[p] - 1] = static_cast<int32_t>(p);
}

}  // namespace

void launch_owned_flags(const int32_t* member_of, int64_t n, int64_t gbase, int64_t n_local, int32_t* flag,
                        cudaStream_t st) {
  count_launch();
  if (n > 0) k_owned_flags<<<blocks_for(n, 256), 256, 0, st>>>(member_of, n, gbase, n_local, flag);
}
void launch_owned_scatter(const int32_t* flag, const int32_t* incl, int64_t n, int32_t* pos_list, cudaStream_t st) {
  count_launch();
  if (n > 0) k_owned_scatter<<<blocks_for(n, 256), 256, 0, st>>>(flag, incl, n, pos_list);
}

void launch_lsh_keys(const Pose* poses, int64_t n, int64_t gbase, const LshPass& lp, uint64_t* keys,
                     unsigned* flagged, cudaStream_t st) {
  count_launch();
  if (flagged) cudaMemsetAsync(flagged, 0, sizeof(unsigned), st);
  if (n > 0) k_lsh_keys<<<blocks_for(n, 128), 128, 0, st>>>(poses, n, gbase, lp, keys, flagged);
}
void launch_gather_flagged(const Pose* poses, const uint64_t* keys, const unsigned* list, int m, Pose* out_pose,
                           uint64_t* out_key, cudaStream_t st) {
  count_launch();
  if (m > 0) k_gather_flagged<<<(m + 127) / 128, 128, 0, st>>>(poses, keys, list, m, out_pose, out_key);
}
void launch_scatter_keys(uint64_t* keys, const unsigned* list, int m, const uint64_t* vals, cudaStream_t st) {
  count_launch();
  if (m > 0) k_scatter_keys<<<(m + 127) / 128, 128, 0, st>>>(keys, list, m, vals);
}
void launch_hash_batch(const Pose* poses, int64_t n, const LshPass& lp, uint64_t* out, unsigned char* amb,
                       cudaStream_t st) {
  count_launch();
  if (n > 0) k_hash_batch<<<blocks_for(n, 128), 128, 0, st>>>(poses, n, lp, out, amb);
}
uint64_t lsh_hash_host(const Pose& pose, const LshPass& lp) {
  return lsh_hash_hd(pose, lp.frame, lp.noise, lp.alpha, lp.sigma_r, lp.sigma_t, nullptr);
}
uint64_t lsh_key_host(const Pose& pose, uint64_t gi, const LshPass& lp) {
  const uint64_t h = lsh_hash_host(pose, lp) % static_cast<uint64_t>(lp.n_buckets);
  const uint64_t prio = lp.prio_bits > 0 ? mix_seed(lp.prio_seed, gi) >> (64 - lp.prio_bits) : 0;
  return (h << (lp.prio_bits + lp.idx_bits)) | (prio << lp.idx_bits) | gi;
}

size_t sort_temp_bytes(int64_t n) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, a, static_cast<const uint64_t*>(nullptr), static_cast<uint64_t*>(nullptr),
                                 static_cast<int>(n), 0, 64);
  cub::DeviceScan::InclusiveSum(nullptr, b, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                static_cast<int>(n));
  return a > b ? a : b;
}

// Keys [begin_bit, end_bit) with a stable LSD radix sort: when the low bits
// hold the particle index and the input is in index order, sorting only the
// bits above them gives the order of the full 64-bit sort.
void sort_keys(const uint64_t* in, uint64_t* out, int64_t n, int begin_bit, int end_bit, void* temp, size_t temp_bytes,
               cudaStream_t st) {
  cub::DeviceRadixSort::SortKeys(temp, temp_bytes, in, out, static_cast<int>(n), begin_bit, end_bit, st);
}

void launch_members(const uint64_t* skeys, int64_t n, uint64_t idx_mask, int shift, int32_t* member_of, int32_t* head,
                    cudaStream_t st, int32_t* new_of_old) {
  count_launch();
  if (n > 0) k_members<<<blocks_for(n, 256), 256, 0, st>>>(skeys, n, idx_mask, shift, member_of, head, new_of_old);
}

void inclusive_sum_i32(const int32_t* in, int32_t* out, int64_t n, void* temp, size_t temp_bytes, cudaStream_t st) {
  cub::DeviceScan::InclusiveSum(temp, temp_bytes, in, out, static_cast<int>(n), st);
}

void launch_inverse_perm(const int32_t* member_of, int64_t n, int32_t* new_of_old, cudaStream_t st) {
  count_launch();
  if (n > 0) k_inverse_perm<<<blocks_for(n, 256), 256, 0, st>>>(member_of, n, new_of_old);
}

bool launch_reorder(const int32_t* old_of_new, const int32_t* new_of_old, int64_t n, int k, const Pose* poses,
                    const double* lp, const int32_t* id, const int32_t* idx, const float* kval, const int32_t* count,
                    Pose* poses2, double* lp2, int32_t* id2, int32_t* idx2, float* kval2, int32_t* count2,
                    cudaStream_t st, float4* mir, unsigned int* tmax_bits, const double* anchor) {
  count_launch();
  if (n > 0 && k == 20) {
    if (mir) {
      cudaMemsetAsync(tmax_bits, 0, sizeof(unsigned int), st);
      k_reorder_k<20, true><<<blocks_for(n, 128), 128, 0, st>>>(
          old_of_new, new_of_old, n, poses, lp, id, idx, kval, count, poses2, lp2, id2, idx2, kval2, count2, mir,
          tmax_bits, make_double3(anchor[0], anchor[1], anchor[2]));
      return true;
    }
    k_reorder_k<20><<<blocks_for(n, 128), 128, 0, st>>>(old_of_new, new_of_old, n, poses, lp, id, idx, kval, count,
                                                        poses2, lp2, id2, idx2, kval2, count2);
    return false;
  }
  if (n > 0)
    k_reorder<<<blocks_for(n, 128), 128, 0, st>>>(old_of_new, new_of_old, n, k, poses, lp, id, idx, kval, count, poses2,
                                                  lp2, id2, idx2, kval2, count2);
  return false;
}

void launch_permute_poses(const int32_t* perm, int64_t n, const Pose* src, Pose* dst, cudaStream_t st) {
  count_launch();
  if (n > 0) k_permute_poses<<<blocks_for(n, 128), 128, 0, st>>>(perm, n, src, dst);
}

size_t migrate_record_bytes(int k) { return sizeof(MigHeader) + 8 * static_cast<size_t>(k); }

void launch_migrate_counts(const int32_t* member_of, int64_t n, int64_t nl, int world, unsigned int* mat,
                           cudaStream_t st) {
  count_launch();
  const int blocks = static_cast<int>(std::min<int64_t>(blocks_for(n, 256), 4 * 148));
  if (n > 0)
    k_migrate_counts<<<blocks, 256, sizeof(unsigned int) * world * world, st>>>(member_of, n, nl, world, mat);
}

void launch_migrate_pack(const int32_t* member_of, int64_t n, int64_t nl, int world, int rank, const unsigned int* mat,
                         unsigned int* cursor, const double* lp, const int32_t* id, const int32_t* count,
                         const int32_t* idx, const float* kval, int k, void* send, cudaStream_t st) {
  count_launch();
  if (n > 0)
    k_migrate_pack<<<blocks_for(n, 256), 256, 0, st>>>(member_of, n, nl, world, rank, mat, cursor, lp, id, count, idx,
                                                       kval, k, static_cast<unsigned char*>(send));
}

void launch_migrate_unpack(const void* recv, int64_t nl, int64_t gbase, int k, const int32_t* new_of_old, double* lp2,
                           int32_t* id2, int32_t* count2, int32_t* idx2, float* kval2, cudaStream_t st) {
  count_launch();
  if (nl > 0)
    k_migrate_unpack<<<blocks_for(nl, 128), 128, 0, st>>>(static_cast<const unsigned char*>(recv), nl, gbase, k,
                                                          new_of_old, lp2, id2, count2, idx2, kval2);
}

void launch_segments(const int32_t* head, const int32_t* seg_id, int64_t n, int32_t* seg_start, cudaStream_t st) {
  count_launch();
  if (n > 0) k_segments<<<blocks_for(n, 256), 256, 0, st>>>(head, seg_id, n, seg_start);
}

void launch_seg_stats(const int32_t* seg_start, const int32_t* n_seg, int64_t n, int cap, unsigned long long* hist,
                      unsigned long long* overflow, cudaStream_t st) {
  count_launch();
  if (n > 0) {
    const unsigned g = static_cast<unsigned>(std::min<int64_t>(blocks_for(n, 256), 296));
    k_seg_stats<<<g, 256, sizeof(unsigned long long) * (cap + 3), st>>>(seg_start, n_seg, cap, hist, overflow);
  }
}

void launch_refresh_gather(const Pose* all_poses, int64_t n, int64_t gbase, const int32_t* pos_list,
                           const int32_t* member_of,
                           const int32_t* seg_id, const int32_t* seg_start, int64_t n_sorted,
                           const int32_t* pos_of, int32_t* idx, float* kval, int32_t* count, int k, int cap,
                           double sr, double st_, const double anchor[3], float4* mir, unsigned int* tmax_bits,
                           cudaStream_t st, bool mirror_ready) {
  count_launch();
  constexpr int B = 64;
  if (n <= 0) return;
  static const bool filtered = std::getenv("SMCL_RG_PLAIN") == nullptr;
  if (filtered && k <= 32 && cap <= 64) {
    // fp32 pose mirror of every particle (the window members may be any shard's)
    if (!mirror_ready) {  // (the unsharded reorder writes it with the reordered poses)
      count_launch();
      cudaMemsetAsync(tmax_bits, 0, sizeof(unsigned int), st);
      k_pose_mirror<<<blocks_for(n_sorted, 256), 256, 0, st>>>(all_poses, n_sorted,
                                                              make_double3(anchor[0], anchor[1], anchor[2]), mir,
                                                              tmax_bits);
    }
#define RGF(KM)                                                                                               \
  k_refresh_gather_f<B, KM><<<blocks_for(n, B), B,                                                                 \
                              static_cast<size_t>(k) * B * 4 + static_cast<size_t>(KM) * B * 4 +                   \
                                  static_cast<size_t>(kRgChunk) * B * 8 + B * 4 + static_cast<size_t>(B) * kRgChunk * 2, \
                              st>>>(all_poses, n, gbase, pos_list, member_of, seg_id, \
                                                               seg_start, n_sorted, pos_of, idx, kval,            \
                                                               count, k,                                          \
                                                               cap, sr, st_, mir, tmax_bits, pos_of == nullptr)
    static const bool stats = std::getenv("SMCL_RG_STATS") != nullptr;
    if (stats && k == 20) {
      const unsigned long long z[4] = {0, 0, 0, 0};
      cudaMemcpyToSymbolAsync(g_rg_stats, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
#define B_ B
      k_refresh_gather_f<B, 20, true><<<blocks_for(n, B), B,
                                        static_cast<size_t>(k) * B * 4 + static_cast<size_t>(20) * B * 4 +
                                            static_cast<size_t>(kRgChunk) * B * 8 + B * 4 +
                                            static_cast<size_t>(B) * kRgChunk * 2,
                                        st>>>(all_poses, n, gbase, pos_list, member_of, seg_id, seg_start, n_sorted,
                                              pos_of, idx, kval, count, k, cap, sr, st_, mir, tmax_bits,
                                              pos_of == nullptr);
#undef B_
      unsigned long long h[4];
      cudaMemcpyFromSymbolAsync(h, g_rg_stats, sizeof(h), 0, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      std::fprintf(stderr, "[rg] n %lld considered %.2f evaluated %.2f inserted %.2f refresh %.2f per particle\n",
                   static_cast<long long>(n), h[0] / double(n), h[1] / double(n), h[2] / double(n), h[3] / double(n));
      return;
    }
    if (k <= 8)
      RGF(8);
    else if (k <= 20)
      RGF(20);
    else
      RGF(32);
#undef RGF

    return;
  }
  k_refresh_gather<B><<<blocks_for(n, B), B, static_cast<size_t>(k) * B * 8, st>>>(all_poses, n, gbase, pos_list,
                                                                                 member_of, seg_id, seg_start,
                                                                                 n_sorted, idx, kval, count, k, cap,
                                                                                 sr, st_);
}

}  // namespace smcl
