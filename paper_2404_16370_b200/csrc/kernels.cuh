// Kernel parameter blocks and host launchers (one per .cu file in kernels/).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "engine.cuh"

namespace smcl {

// Number of hand-written kernel launches issued so far (bench gpu_launches).
void count_launch(int n = 1);
long long launch_count();

struct PredictParams {  // filter.cpp:67-84
  Pose delta;
  double L[36];  // lower-triangular sqrt of the odometry covariance (row-major)
  uint64_t frame_seed;
  int noiseless;
};

struct InitParams {  // filter.cpp:39-65
  uint64_t stream;  // mix_seed(seed, k_stream_init)
  double bmin[3], bmax[3];
  double log_post0;
  int full_rotation;
};

struct SvgdParams {  // svgd.hpp:13-21
  double sigma_r, sigma_t, repulsion_gain;
};

struct LshPass {  // neighbor_search.cpp:71-90
  Pose frame;
  double noise[6];
  double alpha, sigma_r, sigma_t;
  int64_t n_buckets;
  int idx_bits, h_bits, prio_bits;
  uint64_t prio_seed;
};

// particles.cu
void launch_predict(Pose* poses, int64_t n, int64_t gbase, const PredictParams& pp, cudaStream_t st);
void launch_init_uniform(Pose* poses, double* log_post, int32_t* id, int32_t* idx, float* kval, int32_t* count,
                         int64_t n, int64_t gbase, int k, const InitParams& ip, cudaStream_t st);
void launch_svgd(const Pose* all_poses, const double* all_steps, int64_t n, int64_t gbase, const int32_t* idx,
                 const int32_t* count, int k, const SvgdParams& sp, double* phi_out, Pose* poses_out,
                 cudaStream_t st);
void launch_apply(Pose* poses, const double* phis, int64_t n, cudaStream_t st);
void launch_exp_batch(const double* xi, int64_t n, Pose* out, cudaStream_t st);
void launch_log_batch(const Pose* p, int64_t n, double* out, cudaStream_t st);
void launch_kernel_batch(const Pose* a, const Pose* b, int64_t n, double sr, double st_, double* out, cudaStream_t st);

// lsh.cu
// K3. flagged (may be null): count of particles whose hash the host must
// verify with glibc (lsh.cu near-integer guard).
// LSH near-integer guard: K3 appends up to kGuardListCap flagged local
// indices after the count (flagged[0]); the host checks only those.
constexpr int kGuardListCap = 4096;
void launch_gather_flagged(const Pose* poses, const uint64_t* keys, const unsigned* list, int m, Pose* out_pose,
                           uint64_t* out_key, cudaStream_t st);
void launch_scatter_keys(uint64_t* keys, const unsigned* list, int m, const uint64_t* vals, cudaStream_t st);
void launch_lsh_keys(const Pose* poses, int64_t n, int64_t gbase, const LshPass& lp, uint64_t* keys,
                     unsigned* flagged, cudaStream_t st);
// out: raw hashes (no modulo); amb[i] = 1 where the host must rehash (lsh_hash_host).
void launch_hash_batch(const Pose* poses, int64_t n, const LshPass& lp, uint64_t* out, unsigned char* amb,
                       cudaStream_t st);
uint64_t lsh_hash_host(const Pose& pose, const LshPass& lp);  // glibc, as the reference
uint64_t lsh_key_host(const Pose& pose, uint64_t gi, const LshPass& lp);  // K3's key, host (glibc)
size_t sort_temp_bytes(int64_t n);
void sort_keys(const uint64_t* in, uint64_t* out, int64_t n, int begin_bit, int end_bit, void* temp, size_t temp_bytes,
               cudaStream_t st);
void launch_members(const uint64_t* skeys, int64_t n, uint64_t idx_mask, int shift, int32_t* member_of, int32_t* head,
                    cudaStream_t st, int32_t* new_of_old = nullptr);
void inclusive_sum_i32(const int32_t* in, int32_t* out, int64_t n, void* temp, size_t temp_bytes, cudaStream_t st);
void launch_permute_poses(const int32_t* perm, int64_t n, const Pose* src, Pose* dst, cudaStream_t st);
size_t migrate_record_bytes(int k);
void launch_migrate_counts(const int32_t* member_of, int64_t n, int64_t nl, int world, unsigned int* mat,
                           cudaStream_t st);
void launch_migrate_pack(const int32_t* member_of, int64_t n, int64_t nl, int world, int rank, const unsigned int* mat,
                         unsigned int* cursor, const double* lp, const int32_t* id, const int32_t* count,
                         const int32_t* idx, const float* kval, int k, void* send, cudaStream_t st);
void launch_migrate_unpack(const void* recv, int64_t nl, int64_t gbase, int k, const int32_t* new_of_old, double* lp2,
                           int32_t* id2, int32_t* count2, int32_t* idx2, float* kval2, cudaStream_t st);
void launch_inverse_perm(const int32_t* member_of, int64_t n, int32_t* new_of_old, cudaStream_t st);
// mir / tmax_bits / anchor (optional, K = 20): also write the neighbour
// pass's fp32 pose mirror of the reordered poses; returns whether it did.
bool launch_reorder(const int32_t* old_of_new, const int32_t* new_of_old, int64_t n, int k, const Pose* poses,
                    const double* lp, const int32_t* id, const int32_t* idx, const float* kval, const int32_t* count,
                    Pose* poses2, double* lp2, int32_t* id2, int32_t* idx2, float* kval2, int32_t* count2,
                    cudaStream_t st, float4* mir = nullptr, unsigned int* tmax_bits = nullptr,
                    const double* anchor = nullptr);
void launch_segments(const int32_t* head, const int32_t* seg_id, int64_t n, int32_t* seg_start, cudaStream_t st);
void launch_seg_stats(const int32_t* seg_start, const int32_t* n_seg, int64_t n, int cap, unsigned long long* hist,
                      unsigned long long* overflow, cudaStream_t st);
void launch_owned_flags(const int32_t* member_of, int64_t n, int64_t gbase, int64_t n_local, int32_t* flag,
                        cudaStream_t st);
void launch_owned_scatter(const int32_t* flag, const int32_t* incl, int64_t n, int32_t* pos_list, cudaStream_t st);
void launch_refresh_gather(const Pose* all_poses, int64_t n, int64_t gbase, const int32_t* pos_list,
                           const int32_t* member_of, const int32_t* seg_id, const int32_t* seg_start,
                           int64_t n_sorted, const int32_t* pos_of, int32_t* idx, float* kval, int32_t* count, int k,
                           int cap, double sr, double st_, const double anchor[3], float4* mir,
                           unsigned int* tmax_bits, cudaStream_t st, bool mirror_ready = false);

// map_build.cu (device map load: NNF + fast-map records)
cudaError_t build_nnf_device(const double* d_mu, int64_t n, const double pg_org[3], const int pg_dims[3],
                             const double nnf_org[3], const int nnf_dims[3], double res, double max_query_dist,
                             int32_t* d_cells, cudaStream_t st);
// d_plane: per map point (beta, s, -, -), (u.xyz, -)
cudaError_t build_map_records_device(const int32_t* d_cells, int64_t n_cells, const double nnf_org[3],
                                     const int nnf_dims[3], double res, const double* d_mu, const float4* d_plane,
                                     float4* d_rec, cudaStream_t st);

// scan_prep.cu (device make_scan_cloud, compiled with -fmad=false)
struct ScanPrepWork;
ScanPrepWork* scan_prep_create();
void scan_prep_destroy(ScanPrepWork* w);
cudaError_t scan_voxel_downsample(ScanPrepWork* w, const double* d_pts, int n, double leaf, double* d_out, int* n_out,
                                  bool* overflow, cudaStream_t st);
cudaError_t scan_bounds(ScanPrepWork* w, const double* d_pts, int n, double b[6], cudaStream_t st);
cudaError_t scan_records(ScanPrepWork* w, const double* d_mu, const double* d_sigma, int n, float4* d_rec,
                         double* d_l1, bool* structured, double* l1max, cudaStream_t st);
// n <= 4096: the whole leaf-doubling downsample in one block; bounds of the result.
cudaError_t scan_downsample_block(ScanPrepWork* w, const double* d_pts, int n, double leaf0, int max_points,
                                  double* d_out, int* n_out, bool* overflow, double bounds[6], cudaStream_t st);
// kNN covariances + noise + fast records + L1 bound, one sync.
cudaError_t scan_knn_cov_records(ScanPrepWork* w, const double* d_pts, int n, int k, double eps, double noise_var,
                                 const double grid_org[3], double grid_cell, const int grid_dims[3],
                                 double* d_sigma, float4* d_rec, bool* structured, double* l1max, cudaStream_t st);
cudaError_t scan_gather_stride(const double* d_mu, const double* d_sigma, int n_out, int stride, double* mu_out,
                               double* sigma_out, cudaStream_t st);

// posterior.cu
// flagged: the last K3's hash-guard count (stage[15], or the record's 14th double when sharded).
void launch_rep_local(const double* v, const long long* ix, int64_t n_local, int rank, bool sharded, const Pose* poses,
                      const int32_t* id, const unsigned* flagged, Pose* dst_pose, int32_t* dst_id, double* stage,
                      cudaStream_t st);
void launch_rep_select(const double* v, const long long* ix, int64_t n_local, int world, const double* g_rec,
                       double* stage, cudaStream_t st);
void launch_merge_pairs(const double* g, int world, double* out_v, long long* out_i, cudaStream_t st);
void launch_bayes_numer(double* lp, const double* ll, const int32_t* nm, int64_t n, double beta,
                        const unsigned long long* matched, double fill, cudaStream_t st);
void launch_sum_pairs(const unsigned long long* g, int world, unsigned long long* out, cudaStream_t st);
void launch_fill(double* v, int64_t n, double value, cudaStream_t st);
// out[0] += particles with ll > -1e30 (ll may be null: not counted), out[1] += sum nm;
// zero: clear out[0..1] first.
void launch_match_counts(const double* ll, const int32_t* nm, int64_t n, unsigned long long* out, cudaStream_t st,
                         bool zero = true);
int argmax_partials(int64_t n);
void launch_argmax(const double* v, int64_t n, int64_t gbase, double* scratch_v, long long* scratch_i, double* out_v,
                   long long* out_i, cudaStream_t st);
void launch_max_of_partials(const double* pv, const long long* pi, int64_t n, double* out_v, long long* out_i,
                            cudaStream_t st);
// Chunked (4096) serial sums, reduce.hpp order; scratch arrays hold n doubles.
void launch_chunk_sum_exp(const double* v, int64_t n, const double* m, double* partial, cudaStream_t st);
void launch_chunk_sum_kernel(const float* kval, const int32_t* count, int64_t n, int k, double* s1, double* s2,
                             double* pk, double* pc, cudaStream_t st);
void launch_finish_lse(const double* partial, int64_t n_chunks, const double* m, double* lse, cudaStream_t st);
void launch_finish_sum2(const double* a, const double* b, int64_t n_chunks, double* out, cudaStream_t st);
void launch_apply_lse(double* v, int64_t n, const double* lse, double floor_v, cudaStream_t st,
                      const unsigned long long* skip_if_zero = nullptr);
void launch_exp(const double* lp, double* p, int64_t n, cudaStream_t st);
// Unsharded normalisation in three launches: per-block argmax partials, chunk
// sums with the max taken from those partials (block 0 stores it in m_out),
// then finish + apply (+ p_out = exp of the result) in one kernel.
int argmax_partials(int64_t n);
void launch_argmax_partials(const double* v, int64_t n, int64_t gbase, double* scratch_v, long long* scratch_i,
                            cudaStream_t st);
void launch_numer_argmax_partials(double* lp, const double* ll, const int32_t* nm, int64_t n, int64_t gbase,
                                  double beta, const unsigned long long* matched, double fill, double* scratch_v,
                                  long long* scratch_i, cudaStream_t st);
void launch_chunk_sum_exp_parts(const double* v, int64_t n, const double* m_parts, int n_parts, double* m_out,
                                double* partial, cudaStream_t st);
// am_v / am_i (optional): per-block argmax partials of the result (apply_fin_blocks(n) of them).
int apply_fin_blocks(int64_t n);
void launch_apply_lse_fin(double* v, int64_t n, const double* partial, int64_t n_chunks, const double* m,
                          double floor_v, const unsigned long long* skip_if_zero, double* lse_out, double* p_out,
                          int64_t gbase, double* am_v, long long* am_i, cudaStream_t st);
void launch_smooth_round(const double* p_all, double* q, int64_t n, const int32_t* idx, const float* kval,
                         const int32_t* count, int k, cudaStream_t st, bool take_log = false,
                         bool reverse = false);

}  // namespace smcl
