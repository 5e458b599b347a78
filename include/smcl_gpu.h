/*
 * smcl_gpu.h — C ABI of the B200-native Stein-particle-filter step
 * (MegaParticles, arXiv 2404.16370), exported by libsmcl_gpu.so.
 *
 * This is the drop-in boundary for the reference library `steinmcl`
 * (/root/reference/proj, a header-declared C++ library with no FFI of its own).
 * Every entry point names the reference interface it replaces (file:line
 * relative to /root/reference/proj). Plain pointers and sizes only; no torch
 * or CUDA types cross this boundary.
 *
 * Layouts (host side, caller-owned buffers, copied in/out):
 *   pose     12 doubles: R row-major (9) then t (3).  (The reference stores
 *            Eigen column-major R + t; the C++ facade converts.)
 *   tangent   6 doubles [omega; v] (rotation first, se3.hpp:15-17).
 *   sigma     9 doubles, row-major symmetric 3x3.
 *   bounds    6 doubles: min xyz, max xyz (Aabb, gaussian_cloud.hpp:21-31).
 *   neighbor lists: flat stride-K arrays idx[n*K] (int32), kval[n*K] (float),
 *            count[n] (int32), self-first init (neighbor_graph.hpp:16-33).
 *
 * Errors: every int-returning call returns SMCL_OK or an SMCL_E* code and
 * records a message readable with smcl_last_error(); the C++ facade rethrows
 * invalid_argument / runtime_error / logic_error as the reference does.
 * Threading: an engine handle is single-caller; calls on one
 * handle must be serialised. Every call is synchronous at return.
 */
#ifndef SMCL_GPU_H
#define SMCL_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMCL_ABI_VERSION 3
#define SMCL_MAX_HIST 1026

enum {
  SMCL_OK = 0,
  SMCL_EINVAL = 1,   /* std::invalid_argument */
  SMCL_ERUNTIME = 2, /* std::runtime_error    */
  SMCL_ELOGIC = 3,   /* std::logic_error      */
  SMCL_ECUDA = 4,
  SMCL_ENCCL = 5
};

/* FilterConfig (include/steinmcl/filter.hpp:17-51) flattened with its
 * KernelParams (svgd.hpp:13-21), LshConfig (neighbor_search.hpp:13-21) and
 * GicpParams (gicp.hpp:45-57). smcl_config_default() gives the reference
 * defaults. */
typedef struct smcl_config {
  int32_t n_particles;
  int32_t k_neighbors;
  double sigma_r, sigma_t, repulsion_gain;
  double lsh_alpha, lsh_noise_sigma, lsh_buckets_factor;
  int32_t lsh_n_buckets, lsh_bucket_capacity;
  int32_t reorder_particles, smooth_iters;
  double nnf_resolution, nnf_max_query_dist, nnf_padding;
  double beta;
  int32_t n_svgd_iters, gn_scan_stride;
  double damping_scale, omega_max, v_max, min_match_fraction, miss_cost;
  double log_post_floor;
  int32_t covariance_k, n_scan_max;
  double epsilon_plane, scan_voxel_leaf, sensor_noise_sigma;
  double diffusion_sigma_rot, diffusion_sigma_trans;
  int32_t full_rotation, likelihood_mode; /* likelihood_mode: 0 auto, 1 exact fp64, 2 fast structured */
  uint64_t seed;
} smcl_config;

/* GaussianCloud (gaussian_cloud.hpp:32-40). bounds may be NULL (computed). */
typedef struct smcl_cloud {
  int64_t n;
  const double* mu;     /* n*3 */
  const double* sigma;  /* n*9 */
  const double* bounds; /* 6 or NULL */
} smcl_cloud;

/* OdometryInput (filter.hpp:56-60). */
typedef struct smcl_odom {
  double delta[12];
  double cov[36]; /* row-major 6x6 */
  int32_t valid;
} smcl_odom;

/* NeighborStats (neighbor_search.hpp:33-39); hist_len = bucket_capacity + 2. */
typedef struct smcl_neighbor_stats {
  int64_t n_buckets, buckets_used, overflow_dropped;
  double mean_kernel;
  int32_t hist_len;
  int64_t occupancy_hist[SMCL_MAX_HIST];
} smcl_neighbor_stats;

/* FrameResult + StageTimes (filter.hpp:62-82). Stage times are CUDA-event
 * device times of each stage. */
typedef struct smcl_frame_result {
  double representative[12];
  double rep_log_post;
  int64_t rep_index;
  int32_t rep_id;
  int32_t scan_empty, observation_rejected;
  int64_t n_particles;
  double mean_n_matched;
  double predict_ms, neighbor_ms, likelihood_ms, update_ms, posterior_ms, total_ms;
  smcl_neighbor_stats neighbor_stats;
} smcl_frame_result;

/* ParticleSet (particle_set.hpp:16-27) as caller-owned SoA buffers. */
typedef struct smcl_particles_view {
  int64_t n;
  int32_t k;
  double* poses;    /* n*12 */
  double* log_post; /* n    */
  int32_t* id;      /* n    */
  int32_t* idx;     /* n*k  */
  float* kval;      /* n*k  */
  int32_t* count;   /* n    */
} smcl_particles_view;

typedef struct smcl_engine smcl_engine;

/* ------------------------------------------------------------ library */
int smcl_abi_version(void);
const char* smcl_last_error(void); /* message of the last failed call on this thread */
void smcl_config_default(smcl_config* cfg);
int smcl_device_count(int* out);

/* ------------------------------------------------------------ engine
 * FilterEngine (filter.hpp:104-130 / filter.cpp:102-213). */

/* FilterEngine::FilterEngine(GaussianCloud map, FilterConfig) — builds the
 * nearest-neighbour field (nnf.cpp:10-96) and uploads the map. map may be NULL
 * for stage-only use (no likelihood calls). device < 0: current device. */
int smcl_create(const smcl_cloud* map, const smcl_config* cfg, int device, smcl_engine** out);
/* Collective backend of a sharded engine (one engine per rank / GPU).
 * allgather: every rank contributes `bytes` at `send` (device memory of the
 * engine's device); `recv` (device, world*bytes) receives the contributions in
 * rank order. `stream` is the engine's cudaStream_t: the callee must order its
 * work after everything already enqueued on it and before anything enqueued
 * after the call returns (e.g. NCCL on that stream). Returns 0 on success.
 * alltoallv (optional, may be NULL): rank r sends send_bytes[d] bytes to
 * every rank d (chunks packed in rank order at `send`) and receives
 * recv_bytes[s] bytes from every rank s (packed in rank order at `recv`);
 * send_bytes / recv_bytes are host arrays of `world` entries, same stream
 * contract. A sharded engine with reorder_particles = 1 migrates particle
 * state with it (1/world of the all-gather volume); without it the engine
 * falls back to all-gathering the state. */
typedef struct smcl_comm {
  void* ctx;
  int32_t rank, world;
  int (*allgather)(void* ctx, const void* send, void* recv, uint64_t bytes, void* stream);
  int (*alltoallv)(void* ctx, const void* send, const uint64_t* send_bytes, void* recv, const uint64_t* recv_bytes,
                   void* stream);
} smcl_comm;

/* Sharded engine: this rank owns the particles with global indices
 * [rank*N/world, (rank+1)*N/world) (N/world must be a multiple of 4096 so
 * reduction chunks never straddle shards); the map is replicated. Results are
 * bit-identical to a single engine with the same config. With
 * reorder_particles = 1 (the reference default) the LSH reorder migrates
 * particle state across shards: rank r always holds storage positions
 * [r*N/world, (r+1)*N/world) of the global sorted order. */
int smcl_create_sharded(const smcl_cloud* map, const smcl_config* cfg, int device, const smcl_comm* comm,
                        smcl_engine** out);
/* In-process loopback collectives for `world` engines driven by `world` host
 * threads (shard-count invariance tests on one device): fills comms[world]. */
int smcl_comm_loopback_create(int32_t world, smcl_comm* comms);
void smcl_comm_loopback_destroy(smcl_comm* comms);
/* Native NCCL communicator (libnccl.so.2 loaded at run time): the engine's
 * all-gathers become ncclAllGather on the engine stream over NVLink/NVSwitch.
 * Rank 0 calls smcl_nccl_get_unique_id and distributes the 128 bytes (any
 * host channel); every rank then calls smcl_comm_nccl_create with its CUDA
 * device current. The reference has no distributed backend. */
int smcl_nccl_get_unique_id(uint8_t id[128]);
int smcl_comm_nccl_create(const uint8_t id[128], int32_t rank, int32_t world, smcl_comm* out);
void smcl_comm_nccl_destroy(smcl_comm* comm);
int smcl_destroy(smcl_engine* h);

/* FilterEngine::init_uniform(const Aabb&) (filter.cpp:108-116). */
int smcl_init_uniform(smcl_engine* h, const double bounds[6]);
/* steinmcl::init_uniform(cfg, bounds, full_rotation, seed) (filter.cpp:39-65). */
int smcl_init_uniform_seeded(smcl_engine* h, int64_t n, const double bounds[6], int full_rotation, uint64_t seed);
/* FilterEngine::step(scan, odo) (filter.cpp:118-213). scan->n == 0: empty scan. */
int smcl_step(smcl_engine* h, const smcl_cloud* scan, const smcl_odom* odo, smcl_frame_result* out);
/* Device-resident scans: smcl_scan_upload stages a prepared scan into one of
 * SMCL_MAX_SCAN_SLOTS device slots; smcl_step_slot runs FilterEngine::step on
 * it (no host->device scan copy inside the step). smcl_step == upload to slot 0
 * + smcl_step_slot(0). */
#define SMCL_MAX_SCAN_SLOTS 64
int smcl_scan_upload(smcl_engine* h, int slot, const smcl_cloud* scan);
int smcl_step_slot(smcl_engine* h, int slot, const smcl_odom* odo, smcl_frame_result* out);
/* make_scan_cloud(points, cfg) (filter.cpp:86-100) on the device: raw sensor
 * points (n*3) -> voxel downsample with leaf doubling, kNN plane-model
 * covariances + sensor noise, staged into a device slot. Bit-identical to
 * smcl_make_scan_cloud. */
int smcl_scan_prepare(smcl_engine* h, int slot, const double* points, int64_t n);
/* Same preparation, asynchronous: the points are copied and prepared by the
 * engine's preparation thread on its own stream while other slots are being
 * stepped (2-stage pipeline); smcl_step_slot / smcl_scan_get on the slot wait
 * for it. Do not re-prepare a slot that a running step is using. */
int smcl_scan_prepare_async(smcl_engine* h, int slot, const double* points, int64_t n);
/* Prepared scan of a slot (mu_out n*3, sigma_out n*9; NULL pointers: count only). */
int smcl_scan_get(smcl_engine* h, int slot, double* mu_out, double* sigma_out, int64_t* n_out);
/* Scenario-runner frame (scenario.cpp:315-338): make_scan_cloud + step on raw
 * points == smcl_scan_prepare(slot 0) + smcl_step_slot(0). */
int smcl_step_points(smcl_engine* h, const double* points, int64_t n, const smcl_odom* odo, smcl_frame_result* out);

/* Per-kernel device times (CUDA events on the engine stream) of the last
 * step, and the algorithmic work they processed. */
typedef struct smcl_step_profile {
  double predict_ms, lsh_keys_ms, sort_ms, reorder_ms, segments_ms, refresh_gather_ms, nb_stats_ms;
  double gn_kernel_ms, solve_ms, svgd_ms, ll_kernel_ms, bayes_ms, smooth_ms, rep_ms, total_ms;
  int64_t gn_points, ll_points;   /* particle-point evaluations in each pass */
  int64_t gn_matched, ll_matched; /* matched particle-points in each pass */
  int32_t fast_path, n_svgd_iters;
  int64_t kernel_launches;        /* hand-written kernels launched by the step */
  int64_t h2d_bytes, d2h_bytes;   /* host<->device bytes: last scan upload, step read-backs */
  /* LSH near-integer guard (lsh.cu), engine lifetime totals: particles whose
   * hash K3 flagged for a host (glibc) check, and neighbour passes replayed
   * because a host key differed from the device's. */
  int64_t hash_guard_flagged, hash_guard_replays;
} smcl_step_profile;
/* Per-kernel stage times are read from the step's events on the first call
 * after a step (valid until the next step). */
int smcl_last_step_profile(smcl_engine* h, smcl_step_profile* out);
/* The same without reading the stage times (no driver calls): point counts,
 * matched counts, launches, copy bytes, total/predict/GN/solve/SVGD times. */
int smcl_last_step_counts(smcl_engine* h, smcl_step_profile* out);
/* Device timer on the engine stream (CUDA events): start, then stop returns
 * the elapsed milliseconds of everything the engine ran in between. */
int smcl_timer_start(smcl_engine* h);
int smcl_timer_stop(smcl_engine* h, double* ms);
int64_t smcl_frame_index(const smcl_engine* h);
int64_t smcl_num_particles(const smcl_engine* h);

/* FilterEngine::particles() / mutable_particles() (filter.hpp:111-113):
 * download / upload the whole particle state (upload may change n and k). */
int smcl_get_particles(smcl_engine* h, smcl_particles_view* view);
int smcl_set_particles(smcl_engine* h, const smcl_particles_view* view);
/* FilterEngine::nnf(): dims[3], origin[3], resolution; cells may be NULL. */
int smcl_get_nnf(smcl_engine* h, int32_t dims[3], double origin[3], double* resolution, int32_t* cells);

/* ------------------------------------------------------------ stage API
 * Each stage runs on the engine's device-resident particles. Host output
 * pointers may be NULL (result stays on the device for the next stage). */

/* predict(set, delta, cov, frame_seed) (filter.cpp:67-84). */
int smcl_predict(smcl_engine* h, const double delta[12], const double cov[36], uint64_t frame_seed);
/* update_neighbors(set, lsh, kernel, pass_seed, bounds) (neighbor_search.cpp:61-192). */
int smcl_update_neighbors(smcl_engine* h, uint64_t pass_seed, const double bounds[6], smcl_neighbor_stats* stats);
/* evaluate_all(map, nnf, scan, poses, gicp, steps, ll, nm) (gicp.cpp:87-107).
 * H_out (n*36) / b_out (n*6) optionally return each particle's GN system. */
int smcl_evaluate_all(smcl_engine* h, const smcl_cloud* scan, double* step_out, double* ll_out, int32_t* nm_out,
                      double* H_out, double* b_out);
/* evaluate_likelihoods(map, nnf, scan, poses, gicp, ll, nm) (gicp.cpp:109-137). */
int smcl_evaluate_likelihoods(smcl_engine* h, const smcl_cloud* scan, double* ll_out, int32_t* nm_out);
/* compute_phis(poses, steps, idx, count, K, kernel, phi) (svgd.cpp:36-49).
 * steps == NULL: use the device steps of the last evaluate_all. */
int smcl_compute_phis(smcl_engine* h, const double* steps, double* phi_out);
/* apply_updates(poses, phis) (svgd.cpp:51-62). phis == NULL: device phis. */
int smcl_apply_updates(smcl_engine* h, const double* phis);
/* bayes_update(log_post, ll, nm, beta, floor) (posterior.cpp:26-58).
 * ll/nm == NULL: device results of the last likelihood call. */
int smcl_bayes_update(smcl_engine* h, const double* ll, const int32_t* nm, double beta, double floor,
                      int32_t* rejected);
/* normalize_log_post(log_post, floor) (posterior.cpp:13-24). */
int smcl_normalize_log_post(smcl_engine* h, double floor);
/* smooth(log_post, graph, iters, floor) (posterior.cpp:60-97). */
int smcl_smooth(smcl_engine* h, int32_t iters, double floor);
/* representative(log_post, poses) (posterior.cpp:99-108). */
int smcl_representative(smcl_engine* h, int64_t* index, double pose[12], double* log_post);

/* ------------------------------------------------------------ batch device math
 * Handle-free kernels on the current device, for parity tests of the device
 * SE3 / hash / solver code. All pointers are host buffers. */
int smcl_se3_exp_batch(const double* xi, int64_t n, double* poses_out);   /* se3.hpp:73-97  */
int smcl_se3_log_batch(const double* poses, int64_t n, double* xi_out);   /* se3.hpp:103-149 */
int smcl_kernel_batch(const double* a, const double* b, int64_t n, double sigma_r, double sigma_t,
                      double* k_out);                                      /* svgd.hpp:36-38 */
int smcl_lsh_hash_batch(const double* poses, int64_t n, const double frame[12], const double noise[6],
                        double alpha, double sigma_r, double sigma_t, uint64_t* out); /* neighbor_search.cpp:25-35 */
int smcl_solve_step_batch(const double* H, const double* b, const double* lambda, int64_t n, double omega_max,
                          double v_max, double* step_out);                 /* gicp.cpp:47-75 */

/* ------------------------------------------------------------ host preparation
 * Product-side host C++ (map load / scan input). */
/* estimate_covariances(points, k, eps) (gaussian_cloud.cpp:36-90): sigma_out n*9. */
int smcl_estimate_covariances(const double* points, int64_t n, int k, double eps, double* sigma_out);
/* downsample_to(points, max, leaf) (gaussian_cloud.cpp:134-144); out capacity n*3. */
int smcl_downsample_to(const double* points, int64_t n, int64_t max_points, double leaf, double* out,
                       int64_t* n_out);
/* make_scan_cloud(points, cfg) (filter.cpp:86-100); mu_out n*3, sigma_out n*9. */
int smcl_make_scan_cloud(const double* points, int64_t n, const smcl_config* cfg, double* mu_out,
                         double* sigma_out, int64_t* n_out);
/* build_nnf(map, res, pad, max_query) (nnf.cpp:10-96): call with cells == NULL for dims. */
int smcl_build_nnf(const smcl_cloud* map, double resolution, double padding, double max_query_dist,
                   int32_t dims[3], double origin[3], int32_t* cells);

/* ------------------------------------------------------------ simulator (sim/world.cpp)
 * Rectangles are 9 doubles: origin(3), edge_u(3), edge_v(3). */
typedef struct smcl_corridor_spec {  /* sim/world.hpp:41-54 */
  double corridor_length, corridor_width, height;
  int32_t n_rooms, furniture;
  double room_width, room_depth, door_width, door_height;
} smcl_corridor_spec;
typedef struct smcl_sensor_spec {    /* sim/world.hpp:70-78 */
  int32_t n_azimuth, n_elevations;
  double elevations_deg[64];
  double max_range, min_range, noise_sigma;
} smcl_sensor_spec;
void smcl_sim_default_corridor(smcl_corridor_spec* spec);
void smcl_sim_default_sensor(smcl_sensor_spec* spec);
int smcl_sim_corridor_world(const smcl_corridor_spec* spec, double* rects, int32_t max_rects, int32_t* n_rects);
int smcl_sim_box_room(const double size[3], double* rects, int32_t max_rects, int32_t* n_rects);
/* sample_world (world.cpp:140-160): call with mu_out == NULL for the count. */
int smcl_sim_sample_world(const double* rects, int32_t n_rects, double density, uint64_t seed, int cov_k,
                          double eps, double* mu_out, double* sigma_out, int64_t* n_out);
/* simulate_scan_points (world.cpp:162-181); rng_state is the SplitMix64 state (in/out). */
int smcl_sim_scan(const double* rects, int32_t n_rects, const double pose[12], const smcl_sensor_spec* sensor,
                  uint64_t* rng_state, double* points_out, int64_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* SMCL_GPU_H */
