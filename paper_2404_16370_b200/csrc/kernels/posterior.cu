// K11-K13: Bayes update, log-sum-exp normalisation, graph smoothing and MAP
// (reference posterior.cpp:13-108, reduce.hpp:14-69).
//
// Determinism: floating-point sums follow reduce.hpp exactly — 4096-element
// chunks summed serially in index order (one thread per chunk), chunk partials
// then summed serially in chunk order. Chunk boundaries are global indices, so
// a shard owning a 4096-aligned range produces the same partials. Max / argmax
// (ties -> lowest index) and integer counts are order independent and use
// ordinary tree reductions.
#include <cuda_runtime.h>

#include <algorithm>

#include "../engine.cuh"
#include "../kernels.cuh"

namespace smcl {

namespace {

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

// log_post += beta * ll / max(nm, 1)   (posterior.cpp:50-56)
// matched != nullptr (device branch of posterior.cpp:29-41): when no particle
// matched, every value becomes fill (the uniform reset) instead.
__global__ void k_bayes_numer(double* __restrict__ lp, const double* __restrict__ ll, const int32_t* __restrict__ nm,
                              int64_t n, double beta, const unsigned long long* __restrict__ matched,
                              double fill) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (matched && *matched == 0ull) {
    lp[i] = fill;
    return;
  }
  const double denom = static_cast<double>(nm[i] > 1 ? nm[i] : 1);
  lp[i] = xadd(lp[i], xmul(beta, ll[i]) / denom);
}
// Sum of the per-shard (matched, sum n_matched) pairs, in rank order.
__global__ void k_sum_pairs(const unsigned long long* __restrict__ g, int world, unsigned long long* __restrict__ out) {
  unsigned long long a = 0, b = 0;
  for (int r = 0; r < world; ++r) {
    a += g[2 * r];
    b += g[2 * r + 1];
  }
  out[0] = a;
  out[1] = b;
}

__global__ void k_fill(double* __restrict__ v, int64_t n, double value) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) v[i] = value;
}

// Per-block partial of (count of ll > sentinel, sum of nm): exact integers.
__global__ void k_match_counts(const double* __restrict__ ll, const int32_t* __restrict__ nm, int64_t n,
                               unsigned long long* __restrict__ out /* [0]=matched particles, [1]=sum nm */) {
  __shared__ unsigned long long s0[32], s1[32];
  unsigned long long a = 0, b = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (ll) a += ll[i] > -1e30 ? 1ull : 0ull;
    b += static_cast<unsigned long long>(nm[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    s0[w] = a;
    s1[w] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long ta = 0, tb = 0;
    for (int q = 0; q < (blockDim.x >> 5); ++q) {
      ta += s0[q];
      tb += s1[q];
    }
    atomicAdd(out, ta);
    atomicAdd(out + 1, tb);
  }
}

// Max with a deterministic result (max is order independent). Writes one
// partial per block; the caller reduces partials with the same kernel.
__device__ __forceinline__ void argmax_merge(double& v, long long& ix, double v2, long long i2) {
  if (v2 > v || (v2 == v && i2 >= 0 && (ix < 0 || i2 < ix))) {
    v = v2;
    ix = i2;
  }
}

__global__ void k_argmax(const double* __restrict__ v, const long long* __restrict__ vidx, int64_t n, int64_t gbase,
                         double* __restrict__ out_v, long long* __restrict__ out_i) {
  __shared__ double sv[32];
  __shared__ long long si[32];
  double best = -__longlong_as_double(0x7ff0000000000000ll);  // -inf
  long long bi = -1;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    argmax_merge(best, bi, v[i], vidx ? vidx[i] : gbase + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
    const long long i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    argmax_merge(best, bi, v2, i2);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (blockDim.x >> 5); ++q) argmax_merge(best, bi, sv[q], si[q]);
    out_v[blockIdx.x] = best;
    out_i[blockIdx.x] = bi;
  }
}


// Per-particle list sums for mean_kernel (neighbor_search.cpp:182-190): the
// kval sum in slot order and the entry count.
__global__ void k_list_sums(const float* __restrict__ kval, const int32_t* __restrict__ count, int64_t n, int k,
                            double* __restrict__ ksum, double* __restrict__ csum) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  const int cnt = count[i];
  for (int q = 0; q < cnt; ++q) s = xadd(s, static_cast<double>(kval[i * k + q]));
  ksum[i] = s;
  csum[i] = static_cast<double>(cnt);
}

// reduce.hpp:22-27: one block per 4096-element chunk. The block's 256
// threads stage the whole chunk in shared memory (16 independent loads each:
// a single warp streaming 32 KB with a few loads in flight was load-latency
// bound, ~25 us), then thread 0 adds it serially in index order, so every
// chunk partial is bit-identical to the reference's. Two independent vectors
// per launch (blocks [0, chunks) sum v0, [chunks, 2*chunks) sum v1). The
// serial chain is DADD-latency bound: thread 0 reads the staged values 16 at
// a time (LDS.128) ahead of the adds.
// m_ptr != nullptr: the staged values are exp(v - *m_ptr) (the value_at of
// posterior.cpp:17), computed by the block while staging.
constexpr int kChunkThreads = 256;
__global__ void __launch_bounds__(kChunkThreads) k_chunk_serial(const double* __restrict__ v0,
                                                                const double* __restrict__ v1, int64_t n,
                                                                int64_t chunks, double* __restrict__ p0,
                                                                double* __restrict__ p1,
                                                                const double* __restrict__ m_ptr,
                                                                const double* __restrict__ m_parts = nullptr,
                                                                int n_parts = 0, double* __restrict__ m_out = nullptr) {
  __shared__ __align__(16) double s[kReduceChunk];
  const bool second = blockIdx.x >= chunks;
  const double* __restrict__ v = second ? v1 : v0;
  double* __restrict__ partial = second ? p1 : p0;
  const int64_t c = second ? blockIdx.x - chunks : blockIdx.x;
  const int64_t begin = c * kReduceChunk;
  const int m = static_cast<int>(begin + kReduceChunk < n ? kReduceChunk : n - begin);
  if (m_ptr || m_parts) {
    double mv;
    if (m_parts) {  // the max of the argmax kernel's per-block partial values (exact, order-free)
      __shared__ double s_max[kChunkThreads / 32];
      double b = -__longlong_as_double(0x7ff0000000000000ll);
      for (int q = threadIdx.x; q < n_parts; q += kChunkThreads) b = fmax(b, __ldg(m_parts + q));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
      if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = b;
      __syncthreads();
      mv = s_max[0];
#pragma unroll
      for (int w = 1; w < kChunkThreads / 32; ++w) mv = fmax(mv, s_max[w]);
      if (blockIdx.x == 0 && threadIdx.x == 0 && m_out) *m_out = mv;
    } else {
      mv = *m_ptr;
    }
#pragma unroll 4
    for (int q = threadIdx.x; q < m; q += kChunkThreads) s[q] = exp(xsub(__ldg(v + begin + q), mv));
  } else {
#pragma unroll 8
    for (int q = threadIdx.x; q < m; q += kChunkThreads) s[q] = __ldg(v + begin + q);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double acc = 0.0;
  int q = 0;
  const double2* s2 = reinterpret_cast<const double2*>(s);
  if (m >= 16) {  // the next 16 values are read while the current 16 are added
    double2 x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = s2[u];
    for (; q + 32 <= m; q += 16) {
      double2 y[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) y[u] = s2[(q + 16) / 2 + u];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc = xadd(acc, x[u].x);
        acc = xadd(acc, x[u].y);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = y[u];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc = xadd(acc, x[u].x);
      acc = xadd(acc, x[u].y);
    }
    q += 16;
  }
  for (; q < m; ++q) acc = xadd(acc, s[q]);
  partial[c] = acc;
}

// Serial combine of chunk partials (single thread): lse = m + log(sum).
// Serial combines of the chunk partials (reduce.hpp order) by lane 0 of one
// warp, after the warp has staged the partials in shared memory (coalesced).
constexpr int kFinStage = 2048;
__device__ __forceinline__ double serial_sum_staged(const double* __restrict__ a, int64_t n, double* s) {
  double t = 0.0;
  for (int64_t b = 0; b < n; b += kFinStage) {
    const int m = static_cast<int>(n - b < kFinStage ? n - b : kFinStage);
    for (int q = threadIdx.x; q < m; q += 32) s[q] = a[b + q];
    __syncwarp();
    if (threadIdx.x == 0) {
      int q = 0;
      for (; q + 8 <= m; q += 8) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = s[q + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) t = xadd(t, x[u]);
      }
      for (; q < m; ++q) t = xadd(t, s[q]);
    }
    __syncwarp();
  }
  return t;
}

__global__ void __launch_bounds__(32) k_finish_lse(const double* __restrict__ partial, int64_t n_chunks,
                                                   const double* __restrict__ m_ptr, double* __restrict__ lse_out) {
  __shared__ double s[kFinStage];
  const double t = serial_sum_staged(partial, n_chunks, s);
  if (threadIdx.x == 0) *lse_out = xadd(*m_ptr, log(t));
}

__global__ void __launch_bounds__(32) k_finish_sum2(const double* __restrict__ a, const double* __restrict__ b,
                                                    int64_t n_chunks, double* __restrict__ out) {
  __shared__ double s[kFinStage];
  const double ta = serial_sum_staged(a, n_chunks, s);
  const double tb = serial_sum_staged(b, n_chunks, s);
  if (threadIdx.x == 0) {
    out[0] = ta;
    out[1] = tb;
  }
}

// skip_if_zero != nullptr and *skip_if_zero == 0: leave v unchanged (the
// rejected observation of posterior.cpp:29-33 returns before normalizing).
__global__ void k_apply_lse(double* __restrict__ v, int64_t n, const double* __restrict__ lse_ptr, double floor_v,
                            const unsigned long long* __restrict__ skip_if_zero) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (skip_if_zero && *skip_if_zero == 0ull) return;
  const double r = xsub(v[i], *lse_ptr);
  v[i] = r < floor_v ? floor_v : r;  // std::max(v - lse, floor)
}

// finish_lse + apply_lse in one kernel (unsharded normalisation): every
// block's first warp forms lse = m + log(serial sum of the chunk partials)
// exactly as k_finish_lse does (same order, same operations), then the block
// applies it grid-stride; p_out (optional): exp of the result, the smoothing
// pass's input, written in the same sweep.
__global__ void __launch_bounds__(256) k_apply_lse_fin(double* __restrict__ v, int64_t n,
                                                       const double* __restrict__ partial, int64_t n_chunks,
                                                       const double* __restrict__ m_ptr, double floor_v,
                                                       const unsigned long long* __restrict__ skip_if_zero,
                                                       double* __restrict__ lse_out, double* __restrict__ p_out,
                                                       int64_t gbase, double* __restrict__ am_v,
                                                       long long* __restrict__ am_i) {
  __shared__ double s[kFinStage];
  __shared__ double s_lse;
  if (threadIdx.x < 32) {
    const double t = serial_sum_staged(partial, n_chunks, s);
    if (threadIdx.x == 0) {
      s_lse = xadd(*m_ptr, log(t));
      if (blockIdx.x == 0 && lse_out) *lse_out = s_lse;
    }
  }
  __syncthreads();
  const double lse = s_lse;
  const bool skip = skip_if_zero && *skip_if_zero == 0ull;
  double best = -__longlong_as_double(0x7ff0000000000000ll);  // am_v: per-block argmax of the result
  long long bi = -1;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double r = v[i];
    if (!skip) {
      r = xsub(r, lse);
      r = r < floor_v ? floor_v : r;  // std::max(v - lse, floor)
      v[i] = r;
    }
    if (p_out) p_out[i] = exp(r);
    if (am_v) argmax_merge(best, bi, r, gbase + i);
  }
  if (am_v) {  // the representative's argmax partials (posterior.cpp:99-108), merged as k_argmax does
    __shared__ double sv[8];
    __shared__ long long si[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
      const long long i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      argmax_merge(best, bi, v2, i2);
    }
    if ((threadIdx.x & 31) == 0) {
      sv[threadIdx.x >> 5] = best;
      si[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 1; q < 8; ++q) argmax_merge(best, bi, sv[q], si[q]);
      am_v[blockIdx.x] = best;
      am_i[blockIdx.x] = bi;
    }
  }
}

__global__ void k_exp(const double* __restrict__ lp, double* __restrict__ p, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = exp(lp[i]);
}

// One Jacobi round of posterior.cpp:75-90 (q_i = sum_s w_s p[idx_s] / sum_s w_s).
__global__ void k_smooth_round(const double* __restrict__ p_all, double* __restrict__ q, int64_t n,
                               const int32_t* __restrict__ idx, const float* __restrict__ kval,
                               const int32_t* __restrict__ count, int k, int take_log) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double num = 0.0, den = 0.0;
  const int cnt = count[i];
  for (int s = 0; s < cnt; ++s) {
    const double w = static_cast<double>(kval[i * k + s]);
    num = xadd(num, xmul(w, p_all[idx[i * k + s]]));
    den = xadd(den, w);
  }
  const double r = num / den;
  q[i] = take_log ? log(r) : r;  // last round: posterior.cpp's log pass fused
}

// K = 20 (the default list size): the particle's idx / kval rows (80 B
// each, 16-byte aligned) are read with five 128-bit loads each and all 20 p
// gathers are issued before the (reference-order) sums. reverse: blocks walk
// the particles from the top, so a round starts on the rows the previous
// round read last (the 160 MB of rows at 1M exceed L2; an always-ascending
// sweep evicts each row before the next round needs it). Rounds are Jacobi
// sweeps: the order does not change any value.
template <int K, int kMinB = 1>
__global__ void __launch_bounds__(128, kMinB) k_smooth_round_k(const double* __restrict__ p_all, double* __restrict__ q,
                                                        int64_t n, const int32_t* __restrict__ idx,
                                                        const float* __restrict__ kval,
                                                        const int32_t* __restrict__ count, int take_log,
                                                        int reverse, int pdl) {
  static_assert(K % 4 == 0, "rows must be whole 16-byte vectors");
  // Programmatic dependent launch (pdl): the next round's CTAs may start as
  // soon as every CTA of this one is running; they load their rows (constant
  // through the smoothing) and then wait for this round's grid to complete
  // before reading p or writing q.
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t blk = reverse ? gridDim.x - 1 - blockIdx.x : blockIdx.x;
  const int64_t i = blk * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int cnt = count[i];
  int32_t j[K];
  float w[K];
  const int4* ir = reinterpret_cast<const int4*>(idx + i * K);
  const float4* kr = reinterpret_cast<const float4*>(kval + i * K);
#pragma unroll
  for (int v = 0; v < K / 4; ++v) {
    const int4 a = ir[v];
    const float4 b = kr[v];
    j[4 * v] = a.x, j[4 * v + 1] = a.y, j[4 * v + 2] = a.z, j[4 * v + 3] = a.w;
    w[4 * v] = b.x, w[4 * v + 1] = b.y, w[4 * v + 2] = b.z, w[4 * v + 3] = b.w;
  }
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  // p is the previous round's output: plain (coherent) loads, ordered after
  // the wait (volatile asm is never hoisted above it)
  double pv[K];
#pragma unroll
  for (int s = 0; s < K; ++s) {
    pv[s] = 0.0;
    if (s < cnt) asm volatile("ld.global.f64 %0, [%1];" : "=d"(pv[s]) : "l"(p_all + j[s]));
  }
  double num = 0.0, den = 0.0;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    if (s < cnt) {
      const double ws = static_cast<double>(w[s]);
      num = xadd(num, xmul(ws, pv[s]));
      den = xadd(den, ws);
    }
  }
  const double r = num / den;
  q[i] = take_log ? log(r) : r;  // last round: posterior.cpp's log pass fused
}

// Merge of the per-shard (value, index) argmax pairs gathered as
// [v0, i0, v1, i1, ...] (ties -> lowest index, as argmax_merge).
__global__ void k_merge_pairs(const double* __restrict__ g, int world, double* __restrict__ out_v,
                              long long* __restrict__ out_i) {
  double v = -INFINITY;
  long long ix = -1;
  for (int r = 0; r < world; ++r) argmax_merge(v, ix, g[2 * r], __double_as_longlong(g[2 * r + 1]));
  *out_v = v;
  *out_i = ix;
}

// Representative (posterior.cpp:99-108) without a host round trip: the
// winning index is read on the device. Stage layout: [0] value, [1] index
// (bits), [2..13] pose, [14] id (as double).
__global__ void k_rep_local(const double* __restrict__ v_ptr, const long long* __restrict__ ix_ptr, int64_t n_local,
                            int rank, int sharded, const Pose* __restrict__ poses, const int32_t* __restrict__ id,
                            const unsigned* __restrict__ flagged, Pose* __restrict__ dst_pose,
                            int32_t* __restrict__ dst_id, double* __restrict__ stage) {
  const long long ix = *ix_ptr;
  const long long owner = sharded ? ix / n_local : 0;
  const long long li = ix - owner * n_local;
  const long long mine = (owner == rank && li >= 0 && li < n_local) ? li : 0;
  const double fl = flagged ? static_cast<double>(*flagged) : 0.0;
  if (sharded) {  // this rank's slot of the all-gathered candidates (pose, id, hash-guard flags: one record)
    *dst_pose = poses[mine];
    *reinterpret_cast<int32_t*>(dst_pose + 1) = id[mine];
    reinterpret_cast<double*>(dst_pose)[13] = fl;
    return;
  }
  stage[0] = *v_ptr;
  stage[1] = __longlong_as_double(ix);
  const Pose p = poses[mine];
  for (int q = 0; q < 9; ++q) stage[2 + q] = p.R[q];
  for (int a = 0; a < 3; ++a) stage[11 + a] = p.t[a];
  stage[14] = static_cast<double>(id[mine]);
  stage[15] = fl;
}
// g_rec: per rank one record of 14 doubles (pose, the id in the 13th, the
// rank's hash-guard flag count in the 14th).
__global__ void k_rep_select(const double* __restrict__ v_ptr, const long long* __restrict__ ix_ptr, int64_t n_local,
                             int world, const double* __restrict__ g_rec, double* __restrict__ stage) {
  const long long ix = *ix_ptr;
  long long owner = ix / n_local;
  owner = owner < 0 ? 0 : (owner >= world ? world - 1 : owner);
  stage[0] = *v_ptr;
  stage[1] = __longlong_as_double(ix);
  const double* r = g_rec + 14 * owner;
  for (int q = 0; q < 12; ++q) stage[2 + q] = r[q];
  stage[14] = static_cast<double>(*reinterpret_cast<const int32_t*>(r + 12));
  double fl = 0.0;
  for (int w = 0; w < world; ++w) fl += g_rec[14 * w + 13];
  stage[15] = fl;
}

}  // namespace

void launch_rep_local(const double* v, const long long* ix, int64_t n_local, int rank, bool sharded, const Pose* poses,
                      const int32_t* id, const unsigned* flagged, Pose* dst_pose, int32_t* dst_id, double* stage,
                      cudaStream_t st) {
  count_launch();
  k_rep_local<<<1, 1, 0, st>>>(v, ix, n_local, rank, sharded ? 1 : 0, poses, id, flagged, dst_pose, dst_id, stage);
}
void launch_rep_select(const double* v, const long long* ix, int64_t n_local, int world, const double* g_rec,
                       double* stage, cudaStream_t st) {
  count_launch();
  k_rep_select<<<1, 1, 0, st>>>(v, ix, n_local, world, g_rec, stage);
}
void launch_merge_pairs(const double* g, int world, double* out_v, long long* out_i, cudaStream_t st) {
  count_launch();
  k_merge_pairs<<<1, 1, 0, st>>>(g, world, out_v, out_i);
}

void launch_bayes_numer(double* lp, const double* ll, const int32_t* nm, int64_t n, double beta,
                        const unsigned long long* matched, double fill, cudaStream_t st) {
  count_launch();
  if (n > 0) k_bayes_numer<<<blocks_for(n, 256), 256, 0, st>>>(lp, ll, nm, n, beta, matched, fill);
}
void launch_sum_pairs(const unsigned long long* g, int world, unsigned long long* out, cudaStream_t st) {
  count_launch();
  k_sum_pairs<<<1, 1, 0, st>>>(g, world, out);
}
void launch_fill(double* v, int64_t n, double value, cudaStream_t st) {
  count_launch();
  if (n > 0) k_fill<<<blocks_for(n, 256), 256, 0, st>>>(v, n, value);
}
void launch_match_counts(const double* ll, const int32_t* nm, int64_t n, unsigned long long* out, cudaStream_t st,
                         bool zero) {
  count_launch();
  if (zero) cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), st);
  if (n > 0) {
    const unsigned g = static_cast<unsigned>(std::min<int64_t>(blocks_for(n, 256), 1184));
    k_match_counts<<<g, 256, 0, st>>>(ll, nm, n, out);
  }
}
int argmax_partials(int64_t n) { return static_cast<int>(std::min<int64_t>(blocks_for(n, 256), 1184)); }
void launch_argmax(const double* v, int64_t n, int64_t gbase, double* scratch_v, long long* scratch_i, double* out_v,
                   long long* out_i, cudaStream_t st) {
  count_launch();
  const int g = argmax_partials(n);
  k_argmax<<<g, 256, 0, st>>>(v, nullptr, n, gbase, scratch_v, scratch_i);
  k_argmax<<<1, 256, 0, st>>>(scratch_v, scratch_i, g, 0, out_v, out_i);
}
void launch_max_of_partials(const double* pv, const long long* pi, int64_t n, double* out_v, long long* out_i,
                            cudaStream_t st) {
  count_launch();
  k_argmax<<<1, 256, 0, st>>>(pv, pi, n, 0, out_v, out_i);
}
static void chunk_serial2(const double* a, const double* b, int64_t n, double* pa, double* pb, cudaStream_t st) {
  count_launch();
  const int64_t chunks = (n + kReduceChunk - 1) / kReduceChunk;
  if (chunks > 0) k_chunk_serial<<<static_cast<unsigned>(2 * chunks), kChunkThreads, 0, st>>>(a, b, n, chunks, pa, pb, nullptr);
}
void launch_chunk_sum_exp(const double* v, int64_t n, const double* m, double* partial, cudaStream_t st) {
  count_launch();
  if (n <= 0) return;
  const int64_t chunks = (n + kReduceChunk - 1) / kReduceChunk;
  k_chunk_serial<<<static_cast<unsigned>(chunks), kChunkThreads, 0, st>>>(v, v, n, chunks, partial, partial, m);
}
void launch_chunk_sum_kernel(const float* kval, const int32_t* count, int64_t n, int k, double* s1, double* s2,
                             double* pk, double* pc, cudaStream_t st) {
  count_launch();
  if (n <= 0) return;
  k_list_sums<<<blocks_for(n, 256), 256, 0, st>>>(kval, count, n, k, s1, s2);
  chunk_serial2(s1, s2, n, pk, pc, st);
}
void launch_finish_lse(const double* partial, int64_t n_chunks, const double* m, double* lse, cudaStream_t st) {
  count_launch();
  k_finish_lse<<<1, 32, 0, st>>>(partial, n_chunks, m, lse);
}
void launch_finish_sum2(const double* a, const double* b, int64_t n_chunks, double* out, cudaStream_t st) {
  count_launch();
  k_finish_sum2<<<1, 32, 0, st>>>(a, b, n_chunks, out);
}
void launch_apply_lse(double* v, int64_t n, const double* lse, double floor_v, cudaStream_t st,
                      const unsigned long long* skip_if_zero) {
  count_launch();
  if (n > 0) k_apply_lse<<<blocks_for(n, 256), 256, 0, st>>>(v, n, lse, floor_v, skip_if_zero);
}
void launch_chunk_sum_exp_parts(const double* v, int64_t n, const double* m_parts, int n_parts, double* m_out,
                                double* partial, cudaStream_t st) {
  count_launch();
  if (n <= 0) return;
  const int64_t chunks = (n + kReduceChunk - 1) / kReduceChunk;
  k_chunk_serial<<<static_cast<unsigned>(chunks), kChunkThreads, 0, st>>>(v, v, n, chunks, partial, partial, nullptr,
                                                                          m_parts, n_parts, m_out);
}
int apply_fin_blocks(int64_t n) {
  static const int n_sm = [] {
    int dev, v;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return static_cast<int>(std::min<int64_t>(blocks_for(n, 256), 4LL * n_sm));
}
void launch_apply_lse_fin(double* v, int64_t n, const double* partial, int64_t n_chunks, const double* m,
                          double floor_v, const unsigned long long* skip_if_zero, double* lse_out, double* p_out,
                          int64_t gbase, double* am_v, long long* am_i, cudaStream_t st) {
  count_launch();
  if (n <= 0) return;
  const unsigned g = static_cast<unsigned>(apply_fin_blocks(n));
  k_apply_lse_fin<<<g, 256, 0, st>>>(v, n, partial, n_chunks, m, floor_v, skip_if_zero, lse_out, p_out, gbase, am_v,
                                     am_i);
}
// Bayes numerator (k_bayes_numer) and the normalisation's argmax partials in
// one grid-stride sweep (unsharded step).
__global__ void __launch_bounds__(256) k_numer_argmax(double* __restrict__ lp, const double* __restrict__ ll,
                                                      const int32_t* __restrict__ nm, int64_t n, int64_t gbase,
                                                      double beta, const unsigned long long* __restrict__ matched,
                                                      double fill, double* __restrict__ out_v,
                                                      long long* __restrict__ out_i) {
  __shared__ double sv[8];
  __shared__ long long si[8];
  const bool reset = matched && *matched == 0ull;
  double best = -__longlong_as_double(0x7ff0000000000000ll);
  long long bi = -1;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double r;
    if (reset) {
      r = fill;
    } else {
      const double denom = static_cast<double>(nm[i] > 1 ? nm[i] : 1);
      r = xadd(lp[i], xmul(beta, ll[i]) / denom);
    }
    lp[i] = r;
    argmax_merge(best, bi, r, gbase + i);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
    const long long i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    argmax_merge(best, bi, v2, i2);
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < 8; ++q) argmax_merge(best, bi, sv[q], si[q]);
    out_v[blockIdx.x] = best;
    out_i[blockIdx.x] = bi;
  }
}
void launch_numer_argmax_partials(double* lp, const double* ll, const int32_t* nm, int64_t n, int64_t gbase,
                                  double beta, const unsigned long long* matched, double fill, double* scratch_v,
                                  long long* scratch_i, cudaStream_t st) {
  count_launch();
  if (n <= 0) return;
  k_numer_argmax<<<argmax_partials(n), 256, 0, st>>>(lp, ll, nm, n, gbase, beta, matched, fill, scratch_v, scratch_i);
}
void launch_argmax_partials(const double* v, int64_t n, int64_t gbase, double* scratch_v, long long* scratch_i,
                            cudaStream_t st) {
  count_launch();
  const int g = argmax_partials(n);
  k_argmax<<<g, 256, 0, st>>>(v, nullptr, n, gbase, scratch_v, scratch_i);
}
void launch_exp(const double* lp, double* p, int64_t n, cudaStream_t st) {
  count_launch();
  if (n > 0) k_exp<<<blocks_for(n, 256), 256, 0, st>>>(lp, p, n);
}
void launch_smooth_round(const double* p_all, double* q, int64_t n, const int32_t* idx, const float* kval,
                         const int32_t* count, int k, cudaStream_t st, bool take_log, bool reverse) {
  count_launch();
  if (n <= 0) return;
  // __launch_bounds__(128, 1): 80 registers, the 20 gathers and row loads
  // all in flight (0.666 ms for 10 rounds at 1M; capped at 48 / 40
  // registers: 0.729 / 0.740; the previous default heuristic, 56: 0.687).
  if (k == 20)
  {
    // Consecutive rounds overlap through programmatic dependent launch (the
    // first round's predecessor simply completes before its wait returns).
    static const bool no_pdl = std::getenv("SMCL_SMOOTH_NOPDL") != nullptr;  // A/B
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(static_cast<unsigned>(blocks_for(n, 128)));
    lc.blockDim = dim3(128);
    lc.dynamicSmemBytes = 0;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = no_pdl ? 0 : 1;
    cudaLaunchKernelEx(&lc, k_smooth_round_k<20>, p_all, q, n, idx, kval, count, take_log ? 1 : 0,
                       reverse ? 1 : 0, no_pdl ? 0 : 1);
  }
  else
    k_smooth_round<<<blocks_for(n, 128), 128, 0, st>>>(p_all, q, n, idx, kval, count, k, take_log ? 1 : 0);
}

}  // namespace smcl
