// B200 engine: device-resident particle state, per-stage orchestration of the
// hand-written kernels and the C ABI of include/smcl_gpu.h.
//
// Reference call structure: FilterEngine::step (filter.cpp:118-213) and the
// free stage functions it calls. One CUDA stream per engine; every ABI call is
// synchronous at return (only small results are read back).
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <bit>
#include <condition_variable>
#include <deque>
#include <exception>
#include <thread>
#include <mutex>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/smcl_gpu.h"
#include "engine.cuh"
#include "host/prep.hpp"
#include "kernels.cuh"

namespace smcl {

static std::atomic<long long> g_launches{0};
static std::atomic<long long> g_h2d{0}, g_d2h{0};  // host<->device bytes copied by the engine
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

// ---------------------------------------------------------------- errors
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
thread_local std::string g_last_error;

#define CK(x)                                                                                           \
  do {                                                                                                  \
    cudaError_t e_ = (x);                                                                               \
    if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));            \
  } while (0)

template <class F>
int guard(F&& f) {
  try {
    f();
    return SMCL_OK;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return SMCL_ECUDA;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return SMCL_EINVAL;
  } catch (const std::logic_error& e) {
    g_last_error = e.what();
    return SMCL_ELOGIC;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SMCL_ERUNTIME;
  }
}

// ---------------------------------------------------------------- buffers
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void ensure(size_t count) {
    if (count <= n && p) return;
    release();
    if (count == 0) count = 1;
    CK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void upload(const T* h, size_t count, cudaStream_t st) {
    ensure(count);
    if (count) {
      CK(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, st));
      g_h2d += static_cast<long long>(count * sizeof(T));
    }
  }
  void download(T* h, size_t count, cudaStream_t st) const {
    if (count) {
      CK(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, st));
      g_d2h += static_cast<long long>(count * sizeof(T));
    }
  }
  void swap(DBuf& o) {
    std::swap(p, o.p);
    std::swap(n, o.n);
  }
};

namespace {
constexpr uint64_t k_stream_init = 1, k_stream_predict = 2, k_stream_neighbors = 3;  // filter.cpp:22-23
constexpr int kFastMaxScan = 1500;

// ---------------------------------------------------------------- host math
// Eigen LLT (lower) on a 6x6, as the oracle / reference covariance_sqrt.
bool llt6(const double* a, double* l) {
  for (int q = 0; q < 36; ++q) l[q] = a[q];
  for (int k = 0; k < 6; ++k) {
    double x = l[k * 6 + k];
    if (k > 0) {
      double sq = 0.0;
      for (int j = 0; j < k; ++j) sq += l[k * 6 + j] * l[k * 6 + j];
      x -= sq;
    }
    if (x <= 0.0) return false;
    x = std::sqrt(x);
    l[k * 6 + k] = x;
    for (int i = k + 1; i < 6; ++i) {
      if (k > 0) {
        double s = 0.0;
        for (int j = 0; j < k; ++j) s += l[i * 6 + j] * l[k * 6 + j];
        l[i * 6 + k] -= s;
      }
      l[i * 6 + k] /= x;
    }
  }
  for (int i = 0; i < 6; ++i)
    for (int j = i + 1; j < 6; ++j) l[i * 6 + j] = 0.0;
  return true;
}

void sym_eig6(const double* a_in, double w[6], double v[36]) {
  double a[36];
  std::memcpy(a, a_in, sizeof(a));
  for (int i = 0; i < 36; ++i) v[i] = (i % 7 == 0) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, scale = 0.0;
    for (int i = 0; i < 6; ++i) {
      scale += std::fabs(a[i * 7]);
      for (int j = i + 1; j < 6; ++j) off += std::fabs(a[i * 6 + j]);
    }
    if (off == 0.0 || off < 1e-18 * scale) break;
    for (int p = 0; p < 5; ++p)
      for (int q = p + 1; q < 6; ++q) {
        if (a[p * 6 + q] == 0.0) continue;
        const double th = (a[q * 7] - a[p * 7]) / (2.0 * a[p * 6 + q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 6; ++k) {
          const double x = a[k * 6 + p], y = a[k * 6 + q];
          a[k * 6 + p] = c * x - s * y;
          a[k * 6 + q] = s * x + c * y;
        }
        for (int k = 0; k < 6; ++k) {
          const double x = a[p * 6 + k], y = a[q * 6 + k];
          a[p * 6 + k] = c * x - s * y;
          a[q * 6 + k] = s * x + c * y;
        }
        for (int k = 0; k < 6; ++k) {
          const double x = v[k * 6 + p], y = v[k * 6 + q];
          v[k * 6 + p] = c * x - s * y;
          v[k * 6 + q] = s * x + c * y;
        }
      }
  }
  int ord[6] = {0, 1, 2, 3, 4, 5};
  std::sort(ord, ord + 6, [&](int x, int y) { return a[x * 7] < a[y * 7]; });
  double vs[36];
  for (int c = 0; c < 6; ++c) {
    w[c] = a[ord[c] * 7];
    for (int r = 0; r < 6; ++r) vs[r * 6 + c] = v[r * 6 + ord[c]];
  }
  std::memcpy(v, vs, sizeof(vs));
}

// filter.cpp:25-35
void covariance_sqrt(const double* cov, double* L) {
  if (llt6(cov, L)) return;
  double jit[36];
  std::memcpy(jit, cov, sizeof(jit));
  for (int i = 0; i < 6; ++i) jit[i * 7] = cov[i * 7] + 1e-12;
  if (llt6(jit, L)) return;
  double w[6], v[36];
  sym_eig6(cov, w, v);
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) L[i * 6 + j] = v[i * 6 + j] * std::sqrt(std::max(w[j], 0.0));
}

int32_t next_prime_at_least(int32_t n) {  // neighbor_search.cpp:46-59
  if (n <= 2) return 2;
  int32_t p = n | 1;
  for (;; p += 2) {
    bool prime = true;
    for (int32_t d = 3; d * d <= p; d += 2)
      if (p % d == 0) {
        prime = false;
        break;
      }
    if (prime) return p;
  }
}

Pose load_pose(const double* p) {
  Pose q;
  std::memcpy(q.R, p, 9 * sizeof(double));
  std::memcpy(q.t, p + 9, 3 * sizeof(double));
  return q;
}
void store_pose(const Pose& q, double* p) {
  std::memcpy(p, q.R, 9 * sizeof(double));
  std::memcpy(p + 9, q.t, 3 * sizeof(double));
}

// Structured (plane-model) covariance: Sigma = a*I - beta*u u^T with the
// single eigenvalue s = a - beta the smallest one (u its axis) and the double
// eigenvalue a = beta + s. This is exactly the form the reference's
// estimate_covariances produces (gaussian_cloud.cpp:79-86), optionally plus an
// isotropic sensor term (filter.cpp:95-98). Returns false unless Sigma is of
// that form to 1e-10 relative.
bool structure_ab(const double* sig, float& beta, float& s, float u[3]) {
  double w[3], v[9];
  host::sym_eig3(sig, w, v);
  double mx = 0.0;
  for (int q = 0; q < 9; ++q) mx = std::max(mx, std::fabs(sig[q]));
  const double a = 0.5 * (w[1] + w[2]), sv = w[0];
  const double ax[3] = {v[0], v[3], v[6]};
  double err = 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      const double rec = (r == c ? a : 0.0) - (a - sv) * ax[r] * ax[c];
      err = std::max(err, std::fabs(rec - sig[r * 3 + c]));
    }
  if (!(err <= 1e-10 * mx) || !(sv >= 0.0) || !(a > 0.0)) return false;
  for (int q = 0; q < 3; ++q) u[q] = static_cast<float>(ax[q]);
  s = static_cast<float>(sv);
  beta = static_cast<float>(a - sv);
  return true;
}
}  // namespace

}  // namespace smcl

using namespace smcl;

// ---------------------------------------------------------------- engine object
struct smcl_engine {
  smcl_config cfg{};
  int device = 0;
  cudaStream_t st = nullptr;
  int rank = 0, world = 1;
  int64_t n_total = 0, n_local = 0, gbase = 0;
  int k = 20;
  int64_t frame = 0;

  // Sharding: particles [gbase, gbase + n_local) live here; the
  // global arrays below are assembled by all-gathers at the reference's
  // exchange points. Unsharded engines alias them to the local arrays.
  smcl_comm comm{};
  bool sharded = false;
  DBuf<Pose> g_poses, g_poses2;
  DBuf<double> g_steps, g_p, g_part, g_part2;
  DBuf<uint64_t> g_keys;
  DBuf<int32_t> g_flag, pos_list;
  // Sharded reorder: the full old particle state of every
  // shard, gathered before each rank permutes its new index range.
  DBuf<double> g_lp;
  DBuf<int32_t> g_id, g_idx, g_count;
  DBuf<float> g_kval;
  // ... or, when the communicator has alltoallv, only the migrating records
  // (count matrix + per-destination cursors, packed send and received records).
  DBuf<unsigned int> mig_mat;
  DBuf<unsigned char> mig_send, mig_recv;
  unsigned int* mig_host = nullptr;  // pinned copy of the count matrix (world x world)
  size_t mig_host_n = 0;
  cudaEvent_t ev_mig = nullptr;
  DBuf<unsigned long long> g_counts;
  DBuf<double> g_argv, arg_pair;
  DBuf<double> g_rep;  // per rank: representative pose (12 doubles) + id, 14-double (16-B aligned) records
  DBuf<double> rep_stage;  // representative: value, index, pose, id

  // All-gather `bytes` per rank from send (device) into recv (device).
  void allgather(const void* send, void* recv, size_t bytes) {
    if (!sharded) {
      if (send != recv) CK(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, st));
      return;
    }
    if (comm.allgather(comm.ctx, send, recv, static_cast<uint64_t>(bytes), st) != 0)
      throw std::runtime_error("smcl_comm allgather failed");
  }
  void alltoallv(const void* send, const uint64_t* send_bytes, void* recv, const uint64_t* recv_bytes) {
    if (comm.alltoallv(comm.ctx, send, send_bytes, recv, recv_bytes, st) != 0)
      throw std::runtime_error("smcl_comm alltoallv failed");
  }
  // Sharded reorder, non-pose state: count matrix from the replicated
  // member_of (one small device->host read), pack this rank's outgoing
  // records, alltoallv, scatter the received ones to their new positions.
  // The host needs the shard-to-shard counts to size the alltoallv. Their
  // read-back is asynchronous (pinned buffer + event): migrate_begin enqueues
  // the count kernel and the copy, the caller enqueues independent work (the
  // bucket segments), and migrate_finish waits for the event only, so the GPU
  // is busy with that work while the host reads the counts.
  void migrate_begin() {
    const size_t w = static_cast<size_t>(world);
    if (mig_host_n < w * w) {
      if (mig_host) CK(cudaFreeHost(mig_host));
      CK(cudaMallocHost(reinterpret_cast<void**>(&mig_host), sizeof(unsigned int) * w * w));
      mig_host_n = w * w;
    }
    if (!ev_mig) CK(cudaEventCreateWithFlags(&ev_mig, cudaEventDisableTiming));
    CK(cudaMemsetAsync(mig_mat.p, 0, sizeof(unsigned int) * (w * w + w), st));
    launch_migrate_counts(member_of.p, n_total, n_local, world, mig_mat.p, st);
    CK(cudaMemcpyAsync(mig_host, mig_mat.p, sizeof(unsigned int) * w * w, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(ev_mig, st));
  }
  void migrate_finish() {
    const size_t w = static_cast<size_t>(world), rec = migrate_record_bytes(k);
    CK(cudaEventSynchronize(ev_mig));
    std::vector<uint64_t> sb(w), rb(w);
    for (size_t d = 0; d < w; ++d) {
      sb[d] = rec * mig_host[d * w + static_cast<size_t>(rank)];
      rb[d] = rec * mig_host[static_cast<size_t>(rank) * w + d];
    }
    launch_migrate_pack(member_of.p, n_total, n_local, world, rank, mig_mat.p, mig_mat.p + w * w, log_post.p, id.p,
                        count.p, idx.p, kval.p, k, mig_send.p, st);
    alltoallv(mig_send.p, sb.data(), mig_recv.p, rb.data());
    launch_migrate_unpack(mig_recv.p, n_local, gbase, k, new_of_old.p, log_post2.p, id2.p, count2.p, idx2.p, kval2.p,
                          st);
  }
  // Gathered poses of every particle, cached until this rank's poses change
  // (predict, SVGD apply, init, set_particles): the neighbour pass and SVGD
  // share one gather per step; a sharded reorder permutes it locally.
  bool g_poses_valid = false;
  void poses_changed() { g_poses_valid = false; }
  const Pose* all_poses() {  // current poses of every particle
    if (!sharded) return poses.p;
    if (!g_poses_valid) {
      allgather(poses.p, g_poses.p, sizeof(Pose) * static_cast<size_t>(n_local));
      g_poses_valid = true;
    }
    return g_poses.p;
  }
  const double* all_steps() {
    if (!sharded) return steps.p;
    allgather(steps.p, g_steps.p, sizeof(double) * 6 * static_cast<size_t>(n_local));
    return g_steps.p;
  }

  // map
  bool has_map = false;
  bool map_structured = false;
  int map_brick = 0;  // fast-record table layout (MapFast::choose_brick)
  host::Aabb map_bounds{};
  NnfGeom geom{};
  int64_t n_cells = 0;
  std::vector<int32_t> h_cells;
  DBuf<int32_t> cells;
  DBuf<double> map_mu, map_sigma;
  DBuf<float4> map_fast;   // 2 float4 per record + one trailing empty record (MapFast::empty)
  DBuf<uint32_t> map_occ;   // occupancy bitmap by record index (MapFast::occ)
  uint64_t map_records = 0;
  DBuf<int32_t> live_list;  // K2a: particles the likelihood gate keeps
  DBuf<unsigned> live_count;
  DBuf<int32_t> sub_list;   // the gate split's predicted-dead particles (K2a's input)
  DBuf<unsigned> sub_count;
  // nm holds this step's GN-pass counts (a prediction for the likelihood
  // pass's gate) with the GN pass's own threshold
  bool nm_from_gn = false;
  int gn_gate_thr = 0;

  // particles
  DBuf<Pose> poses, poses2, poses3;  // poses3: SVGD's output never lands on the guard checkpoint
  DBuf<double> log_post, log_post2;
  DBuf<int32_t> id, id2, idx, idx2, count, count2;
  DBuf<float> kval, kval2;

  // per-stage work
  DBuf<double> sys, steps, phis, ll, raw_ll;  // sys: exact-path GN records (allocated on first use)
  DBuf<float> sysf;                           // fast-path GN records (kSysF floats per particle)
  DBuf<int32_t> nm;
  bool steps_valid = false, phis_valid = false, ll_valid = false;

  // lsh
  DBuf<uint64_t> keys, skeys;
  DBuf<int32_t> member_of, head, seg_id, seg_start, new_of_old, iota, pos_of_buf;
  DBuf<float4> pose_mirror;        // fp32 poses for the neighbour-pass window filter
  DBuf<unsigned int> mirror_tmax;  // max |t - anchor| (float bits) of that mirror
  DBuf<unsigned char> temp;
  size_t temp_bytes = 0;
  DBuf<unsigned long long> d_counts;

  // posterior
  DBuf<double> pbuf, qbuf, partial, partial2, scal;
  DBuf<long long> scal_i;
  DBuf<double> argv;
  DBuf<long long> argi;

  // scans (full and Gauss-Newton subset)
  struct ScanDev {
    int n = 0;
    bool structured = false;
    double l1max = 0.0;  // max_k |mu_k|_1 (fast-path error bound)
    DBuf<double> mu, sigma;
    DBuf<float4> rec;
  };
  struct ScanSlot {
    ScanDev full, gn;
    bool gn_alias = true;  // stride 1: the GN scan is the full scan
    bool valid = false;
    long long upload_bytes = 0;  // H2D bytes of the slot's last preparation
    const ScanDev& gn_view() const { return gn_alias ? full : gn; }
  };
  std::vector<std::unique_ptr<ScanSlot>> slots;
  // Device scan preparation (kernels/scan_prep.cu): raw points, downsampled
  // points, per-point L1 norms and the CUB/sort scratch.
  DBuf<double> raw_pts, down_pts, scan_l1;
  struct PrepDeleter {
    void operator()(ScanPrepWork* w) const { scan_prep_destroy(w); }
  };
  std::unique_ptr<ScanPrepWork, PrepDeleter> prep_work;
  ScanDev scan_tmp;  // stage-API scans

  // Step profile: one event per boundary, read after the step's final sync.
  enum Ev { E_START, E_PRED, E_KEYS, E_SORT, E_REORDER, E_SEG, E_RG, E_NB, E_LL0, E_LL1, E_BAYES, E_SMOOTH, E_END, E_COUNT };
  cudaEvent_t ev[E_COUNT] = {};
  // One (GN start, GN end, solve end, SVGD start, SVGD end) set per SVGD
  // iteration, all read after the step's single end-of-frame sync.
  enum ItEv { I_GN0, I_GN1, I_SOLVE, I_SV0, I_SVGD, I_COUNT };
  std::vector<cudaEvent_t> it_ev;
  int gn_iter = 0;  // SVGD iteration of the running step (event slot)
  void mark_it(int it, ItEv e) {
    const size_t q = static_cast<size_t>(it) * I_COUNT + e;
    if (it_ev.size() <= q) it_ev.resize(q + 1, nullptr);
    if (!it_ev[q]) CK(cudaEventCreate(&it_ev[q]));
    CK(cudaEventRecord(it_ev[q], st));
  }
  float since_it_ev(cudaEvent_t a, int it, ItEv b) const {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, it_ev[static_cast<size_t>(it) * I_COUNT + b]);
    return ms;
  }
  float since_it(int it, ItEv a, ItEv b) const {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, it_ev[static_cast<size_t>(it) * I_COUNT + a], it_ev[static_cast<size_t>(it) * I_COUNT + b]);
    return ms;
  }
  cudaEvent_t timer[2] = {};
  smcl_step_profile prof{};
  bool fast_used = false;
  bool profiling = false;
  int32_t rep_id = -1;                // id of the last representative
  unsigned long long last_nm_sum = 0;  // sum of n_matched over all shards (last Bayes update)
  // NVTX: one host range per step stage (opened at the stage's start event,
  // closed at the next), nested in the step's range; header-only NVTX v3, a
  // no-op unless a profiler (ncu --nvtx) is attached.
  bool nvtx_open = false;
  void nvtx_stage(Ev e) {
    static const char* names[E_COUNT] = {"predict",  "lsh_keys",  "sort",     "reorder", "segments",
                                         "refresh_gather", "nb_stats", "gn_svgd", "likelihood", "ll_gate",
                                         "bayes_update", "smooth", nullptr};
    if (nvtx_open) nvtxRangePop();
    nvtx_open = names[e] != nullptr;
    if (nvtx_open) nvtxRangePushA(names[e]);
  }
  // The step's per-kernel stage times stay in the events until the next step
  // records them again; read on demand (each cudaEventElapsedTime is a driver
  // call, ~20 us per step for all of them, on the host path between frames).
  bool prof_times_pending = false, prof_empty = false;
  void fill_prof_times() {
    if (!prof_times_pending) return;
    prof_times_pending = false;
    prof.lsh_keys_ms = since(E_PRED, E_KEYS);
    prof.sort_ms = since(E_KEYS, E_SORT);
    prof.reorder_ms = since(E_SORT, E_REORDER);
    prof.segments_ms = since(E_REORDER, E_SEG);
    prof.refresh_gather_ms = since(E_SEG, E_RG);
    prof.nb_stats_ms = since(E_RG, E_NB);
    prof.ll_kernel_ms = prof_empty ? 0.0 : since(E_LL0, E_LL1);
    prof.bayes_ms = since(E_LL1, E_SMOOTH);
    prof.smooth_ms = since(E_SMOOTH, E_END);
  }
  void mark(Ev e) {
    if (!ev[e]) CK(cudaEventCreate(&ev[e]));
    CK(cudaEventRecord(ev[e], st));
    if (profiling) nvtx_stage(e);
  }
  float since(Ev a, Ev b) const {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[a], ev[b]);
    return ms;
  }

  // Neighbour-pass statistics (neighbor_search.cpp:172-190) run on a side
  // stream, overlapped with the rest of the step, into their own buffers; the
  // host copy lands in pinned memory and fills the caller's struct after the
  // call's final sync (finish_nb_stats). Sharded engines keep them on the
  // engine stream (their all-gathers are stream-ordered there).
  struct NbHost {
    unsigned long long hist[SMCL_MAX_HIST];
    unsigned long long overflow;
    double sums[2];
    int32_t n_seg;
  };
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  NbHost* nb_host = nullptr;
  struct StepHost {  // end-of-step reads (pinned)
    double rep[16];
    unsigned long long cnt[6];
  };
  StepHost* step_host = nullptr;
  DBuf<unsigned long long> nb_hist;
  DBuf<double> nb_s1, nb_s2, nb_p1, nb_p2, nb_sum;
  smcl_neighbor_stats* nb_out = nullptr;
  int32_t nb_buckets = 0;
  int nb_hist_len = 0;
  bool aux_pending = false;
  void join_aux() {  // engine stream waits for the side-stream statistics
    if (aux_pending) CK(cudaStreamWaitEvent(st, ev_join, 0));
    aux_pending = false;
  }
  void finish_nb_stats() {  // after the call's final sync
    if (!nb_out) return;
    smcl_neighbor_stats* out = nb_out;
    nb_out = nullptr;
    out->n_buckets = nb_buckets;
    out->buckets_used = nb_host->n_seg;
    out->overflow_dropped = static_cast<int64_t>(nb_host->overflow);
    out->mean_kernel = nb_host->sums[1] > 0 ? nb_host->sums[0] / nb_host->sums[1] : 0.0;
    out->hist_len = std::min(nb_hist_len, SMCL_MAX_HIST);
    for (int q = 0; q < out->hist_len; ++q) out->occupancy_hist[q] = static_cast<int64_t>(nb_host->hist[q]);
  }

  ~smcl_engine() {
    if (prep_thread.joinable()) {
      {
        std::lock_guard<std::mutex> lk(prep_m);
        prep_stop = true;
      }
      prep_cv.notify_all();
      prep_thread.join();
    }
    if (prep_st) {
      cudaStreamSynchronize(prep_st);
      cudaStreamDestroy(prep_st);
    }
    if (st) cudaStreamSynchronize(st);
    if (aux) {
      cudaStreamSynchronize(aux);
      cudaStreamDestroy(aux);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (ev_mig) cudaEventDestroy(ev_mig);
    if (mig_host) cudaFreeHost(mig_host);
    if (nb_host) cudaFreeHost(nb_host);
    if (step_host) cudaFreeHost(step_host);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : it_ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : timer)
      if (e) cudaEventDestroy(e);
    if (st) cudaStreamDestroy(st);
  }

  void sync() { CK(cudaStreamSynchronize(st)); }

  // ------------------------------------------------------------ setup
  void setup_map(const smcl_cloud* m) {
    if (!m || m->n <= 0) throw std::invalid_argument("FilterEngine: empty map");
    const auto* pts = reinterpret_cast<const host::V3*>(m->mu);
    if (m->bounds) {
      for (int a = 0; a < 3; ++a) {
        map_bounds.min[a] = m->bounds[a];
        map_bounds.max[a] = m->bounds[3 + a];
      }
    } else {
      map_bounds = host::compute_bounds(pts, m->n);
    }
    const host::NnfGeometry g = host::nnf_geometry(map_bounds, cfg.nnf_resolution, cfg.nnf_padding,
                                                   cfg.nnf_max_query_dist, size_t(1) << 30);
    n_cells = g.n_cells;
    for (int a = 0; a < 3; ++a) {
      geom.origin[a] = g.origin[a];
      geom.dims[a] = g.dims[a];
    }
    geom.res = g.resolution;
    geom.inv_res = 1.0 / g.resolution;
    map_mu.upload(m->mu, static_cast<size_t>(m->n) * 3, st);
    map_sigma.upload(m->sigma, static_cast<size_t>(m->n) * 9, st);
    // Device map load (kernels/map_build.cu): NNF bit-identical to
    // host::build_nnf_cells (nnf.cpp:10-96); the point grid of
    // point_grid.cpp:10-49 over the map's own point bounds.
    const host::Aabb pb = host::compute_bounds(pts, m->n);
    int pg_dims[3];
    for (int a = 0; a < 3; ++a) pg_dims[a] = static_cast<int>(std::floor((pb.max[a] - pb.min[a]) / g.resolution)) + 1;
    cells.ensure(static_cast<size_t>(n_cells));
    CK(build_nnf_device(map_mu.p, m->n, pb.min, pg_dims, g.origin, g.dims, g.resolution, g.max_query_dist, cells.p,
                        st));
    h_cells.clear();  // host copy made on demand (smcl_get_nnf)
    // Structured (plane-model) map -> denormalised 32-byte cell records.
    std::vector<float4> plane(2 * static_cast<size_t>(m->n));
    bool ok = true;
    for (int64_t i = 0; i < m->n && ok; ++i) {
      float beta, sv, u[3];
      ok = structure_ab(m->sigma + 9 * i, beta, sv, u);
      plane[2 * i] = make_float4(beta, sv, 0.f, 0.f);
      plane[2 * i + 1] = make_float4(u[0], u[1], u[2], 0.f);
    }
    map_structured = ok;
    if (ok) {
      DBuf<float4> d_plane;
      d_plane.upload(plane.data(), plane.size(), st);
      map_brick = MapFast::choose_brick(g.dims);
      map_records = MapFast::n_records(g.dims, map_brick);
      map_fast.ensure(2 * static_cast<size_t>(map_records) + 2);
      CK(build_map_records_device(cells.p, n_cells, g.origin, g.dims, g.resolution, map_mu.p, d_plane.p, map_fast.p,
                                  st));
      const float4 empty_rec[2] = {make_float4(0.f, 0.f, 0.f, -1.f), make_float4(0.f, 0.f, 0.f, 0.f)};
      CK(cudaMemcpyAsync(map_fast.p + 2 * map_records, empty_rec, sizeof(empty_rec), cudaMemcpyHostToDevice, st));
      map_occ.ensure(static_cast<size_t>((map_records + 31) / 32));
      launch_build_occupancy(map_fast.p, map_records, map_occ.p, st);
      CK(cudaGetLastError());
      sync();
    }
    has_map = true;
    sync();
  }

  // Shard geometry for n_total particles: contiguous global
  // index ranges; 4096-aligned so reduction chunks never straddle shards.
  void set_shape(int64_t n) {
    if (sharded) {
      if (n % world != 0 || (n / world) % kReduceChunk != 0)
        throw std::invalid_argument("sharded engine: N/world must be a multiple of 4096");
    }
    n_total = n;
    n_local = n / world;
    gbase = static_cast<int64_t>(rank) * n_local;
  }

  void alloc_particles(int64_t n, int kk) {
    n_local = n;
    k = kk;
    const size_t un = static_cast<size_t>(std::max<int64_t>(n, 1));
    const size_t ug = static_cast<size_t>(std::max<int64_t>(n_total, 1));
    if (sharded) {
      const size_t w = static_cast<size_t>(world);
      g_poses.ensure(ug);
      g_steps.ensure(ug * 6);
      g_p.ensure(ug);
      g_keys.ensure(ug);
      g_flag.ensure(ug);
      pos_list.ensure(un);
      g_part.ensure(w * ((un + kReduceChunk - 1) / kReduceChunk));
      g_part2.ensure(w * ((un + kReduceChunk - 1) / kReduceChunk));
      g_counts.ensure(w * 2);
      g_argv.ensure(2 * w);  // (value, index) pairs
      arg_pair.ensure(2);
      g_rep.ensure(w * 14);   // per rank: pose (12 doubles) + id + pad
      if (cfg.reorder_particles) {
        g_poses2.ensure(ug);
        if (comm.alltoallv) {
          mig_mat.ensure(w * w + w);
          mig_send.ensure(un * migrate_record_bytes(kk));
          mig_recv.ensure(un * migrate_record_bytes(kk));
        } else {
          g_lp.ensure(ug);
          g_id.ensure(ug);
          g_count.ensure(ug);
          g_idx.ensure(ug * static_cast<size_t>(kk));
          g_kval.ensure(ug * static_cast<size_t>(kk));
        }
      }
    }
    poses.ensure(un);
    poses2.ensure(un);
    poses3.ensure(un);
    log_post.ensure(un);
    log_post2.ensure(un);
    id.ensure(un);
    id2.ensure(un);
    count.ensure(un);
    count2.ensure(un);
    idx.ensure(un * kk);
    idx2.ensure(un * kk);
    kval.ensure(un * kk);
    kval2.ensure(un * kk);
    sysf.ensure(un * kSysF);
    raw_ll.ensure(un);
    steps.ensure(un * 6);
    phis.ensure(un * 6);
    ll.ensure(un);
    nm.ensure(un);
    keys.ensure(un);
    skeys.ensure(ug);  // the sort and the bucket runs are over all N keys
    member_of.ensure(ug);
    head.ensure(ug);
    seg_id.ensure(ug);
    seg_start.ensure(ug + 1);  // + sentinel
    nb_hist.ensure(SMCL_MAX_HIST + 1);  // + overflow count
    nb_s1.ensure(un);
    nb_s2.ensure(un);
    nb_p1.ensure((un + kReduceChunk - 1) / kReduceChunk);
    nb_p2.ensure((un + kReduceChunk - 1) / kReduceChunk);
    nb_sum.ensure(2);
    new_of_old.ensure(ug);
    iota.ensure(ug);
    {
      std::vector<int32_t> h(ug);
      for (size_t i = 0; i < ug; ++i) h[i] = static_cast<int32_t>(i);
      iota.upload(h.data(), ug, st);
    }
    const size_t tb = sort_temp_bytes(static_cast<int64_t>(ug));
    if (tb > temp_bytes) {
      temp.ensure(tb);
      temp_bytes = tb;
    }
    pbuf.ensure(un);
    qbuf.ensure(un);
    const size_t chunks = (un + kReduceChunk - 1) / kReduceChunk;
    partial.ensure(chunks);
    partial2.ensure(chunks);
    scal.ensure(8);
    scal_i.ensure(8);
    argv.ensure(static_cast<size_t>(argmax_partials(static_cast<int64_t>(un))));
    argi.ensure(static_cast<size_t>(argmax_partials(static_cast<int64_t>(un))));
    d_counts.ensure(8);
    steps_valid = phis_valid = ll_valid = false;
  }

  // ------------------------------------------------------------ scans
  void upload_scan(ScanDev& sd, const double* mu, const double* sigma, int n, cudaStream_t us) {
    if (n > kMaxScan) throw std::invalid_argument("scan exceeds the device scan capacity");
    sd.n = n;
    sd.mu.upload(mu, static_cast<size_t>(n) * 3, us);
    sd.sigma.upload(sigma, static_cast<size_t>(n) * 9, us);
    std::vector<float4> rec(2 * static_cast<size_t>(std::max(n, 1)));
    bool ok = true;
    for (int q = 0; q < n && ok; ++q) {
      float beta, s, u[3];
      ok = structure_ab(sigma + 9 * q, beta, s, u);
      rec[2 * q] = make_float4(static_cast<float>(mu[3 * q]), static_cast<float>(mu[3 * q + 1]),
                               static_cast<float>(mu[3 * q + 2]), beta);
      rec[2 * q + 1] = make_float4(u[0], u[1], u[2], s);
    }
    sd.structured = ok;
    sd.l1max = 0.0;
    for (int q = 0; q < n; ++q)
      sd.l1max = std::max(sd.l1max, std::fabs(mu[3 * q]) + std::fabs(mu[3 * q + 1]) + std::fabs(mu[3 * q + 2]));
    if (ok) sd.rec.upload(rec.data(), rec.size(), us);
  }

  ScanSlot& slot_at(int i) {  // slots are created with the engine: safe from the preparation thread
    if (i < 0 || i >= SMCL_MAX_SCAN_SLOTS) throw std::invalid_argument("scan slot out of range");
    return *slots[static_cast<size_t>(i)];
  }

  // ------------------------------------------------------------ scan pipeline
  // smcl_scan_prepare_async: a preparation thread with its own stream runs
  // make_scan_cloud for slot f+1 while the engine stream runs the step on
  // slot f (the 2-stage stream pipeline of SURVEY §8f next-2). step_slot(i)
  // waits for slot i's pending preparation; synchronous preparations wait for
  // the queue to drain (they share the scratch buffers).
  struct PrepJob {
    int slot;
    std::vector<double> pts;
  };
  std::thread prep_thread;
  std::mutex prep_m;
  std::condition_variable prep_cv;
  std::deque<PrepJob> prep_q;
  int prep_pending[SMCL_MAX_SCAN_SLOTS] = {};
  bool prep_stop = false;
  std::exception_ptr prep_err;
  cudaStream_t prep_st = nullptr;

  void prep_worker() {
    cudaSetDevice(device);
    for (;;) {
      PrepJob job;
      {
        std::unique_lock<std::mutex> lk(prep_m);
        prep_cv.wait(lk, [&] { return prep_stop || !prep_q.empty(); });
        if (prep_q.empty()) return;
        job = std::move(prep_q.front());
        prep_q.pop_front();
      }
      try {
        prepare_slot(job.slot, job.pts.data(), static_cast<int64_t>(job.pts.size() / 3), prep_st);
      } catch (...) {
        std::lock_guard<std::mutex> lk(prep_m);
        if (!prep_err) prep_err = std::current_exception();
      }
      {
        std::lock_guard<std::mutex> lk(prep_m);
        --prep_pending[job.slot];
      }
      prep_cv.notify_all();
    }
  }
  void prepare_async(int slot, const double* points, int64_t n) {
    slot_at(slot);
    if (n < 0 || (n > 0 && !points)) throw std::invalid_argument("scan_prepare: null points");
    if (!prep_thread.joinable()) {
      CK(cudaStreamCreateWithFlags(&prep_st, cudaStreamNonBlocking));
      prep_thread = std::thread([this] { prep_worker(); });
    }
    PrepJob job{slot, std::vector<double>(points, points + 3 * n)};  // the caller may reuse its buffer
    {
      std::lock_guard<std::mutex> lk(prep_m);
      ++prep_pending[slot];
      prep_q.push_back(std::move(job));
    }
    prep_cv.notify_all();
  }
  void rethrow_prep_error() {
    if (prep_err) {
      std::exception_ptr e = prep_err;
      prep_err = nullptr;
      std::rethrow_exception(e);
    }
  }
  void wait_slot(int slot) {
    if (!prep_thread.joinable()) return;
    std::unique_lock<std::mutex> lk(prep_m);
    prep_cv.wait(lk, [&] { return prep_pending[slot] == 0; });
    rethrow_prep_error();
  }
  void wait_prep_all() {
    if (!prep_thread.joinable()) return;
    std::unique_lock<std::mutex> lk(prep_m);
    prep_cv.wait(lk, [&] { return prep_q.empty() && std::all_of(std::begin(prep_pending), std::end(prep_pending), [](int v) { return v == 0; }); });
    rethrow_prep_error();
  }

  // Host scan preparation + H2D into a device slot (filter.cpp:154-165 for
  // the strided Gauss-Newton subset).
  void set_slot(int i, const smcl_cloud* scan) {
    wait_slot(i);
    set_slot_impl(i, scan, st);
  }
  void set_slot_impl(int i, const smcl_cloud* scan, cudaStream_t us) {
    const long long h2d0 = g_h2d.load();
    ScanSlot& sl = slot_at(i);
    struct Tally {
      long long h0;
      long long& out;
      ~Tally() { out = g_h2d.load() - h0; }
    } tally{h2d0, sl.upload_bytes};
    const int S = static_cast<int>(scan ? scan->n : 0);
    sl.valid = true;
    if (S == 0) {
      sl.full.n = 0;
      sl.gn_alias = true;
      return;
    }
    upload_scan(sl.full, scan->mu, scan->sigma, S, us);
    const int stride = cfg.gn_scan_stride;
    if (stride > 1 && S > 2 * stride) {
      std::vector<double> mu, sg;
      for (int q = 0; q < S; q += stride) {
        mu.insert(mu.end(), scan->mu + 3 * q, scan->mu + 3 * q + 3);
        sg.insert(sg.end(), scan->sigma + 9 * q, scan->sigma + 9 * q + 9);
      }
      upload_scan(sl.gn, mu.data(), sg.data(), static_cast<int>(mu.size() / 3), us);
      sl.gn_alias = false;
    } else {
      sl.gn_alias = true;
    }
    CK(cudaStreamSynchronize(us));  // host staging vectors die here
  }

  // make_scan_cloud (filter.cpp:86-100) on the device into slot i: raw
  // points in, prepared Gaussian scan + fast records out, no host math on the
  // data path. Falls back to the host preparation only for inputs outside the
  // device path's envelope (voxel keys beyond 21 bits, k + 1 > 16).
  void prepare_slot(int i, const double* points, int64_t n, cudaStream_t ps) {
    if (n < 0 || (n > 0 && !points)) throw std::invalid_argument("scan_prepare: null points");
    ScanSlot& sl = slot_at(i);
    const long long h2d0 = g_h2d.load();
    auto empty = [&]() {
      sl.valid = true;
      sl.full.n = 0;
      sl.gn_alias = true;
    };
    if (n < static_cast<int64_t>(cfg.covariance_k) + 1 || n < 5) return empty();
    if (n > (int64_t(1) << 30)) throw std::invalid_argument("scan_prepare: too many points");
    auto host_fallback = [&]() {
      std::vector<double> mu(static_cast<size_t>(n) * 3), sg(static_cast<size_t>(n) * 9);
      int64_t m = 0;
      if (smcl_make_scan_cloud(points, n, &cfg, mu.data(), sg.data(), &m) != SMCL_OK)
        throw std::runtime_error(smcl_last_error());
      smcl_cloud c{};
      c.n = m;
      c.mu = mu.data();
      c.sigma = sg.data();
      set_slot_impl(i, &c, ps);
    };
    if (cfg.covariance_k + 1 > 16) return host_fallback();
    // SMCL_PREP_STATS=1: per-phase host-timed breakdown on stderr (diagnostics only).
    static const bool prep_stats = std::getenv("SMCL_PREP_STATS") != nullptr;
    auto t_prev = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
      if (!prep_stats) return;
      CK(cudaStreamSynchronize(ps));
      const auto t = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[prep] %s %.1f us\n", what, std::chrono::duration<double, std::micro>(t - t_prev).count());
      t_prev = t;
    };
    raw_pts.upload(points, static_cast<size_t>(n) * 3, ps);
    if (!prep_work) prep_work.reset(scan_prep_create());
    lap("upload");
    const int ni = static_cast<int>(n);
    const double* d_down = raw_pts.p;
    int m = ni;
    double b[6];
    bool have_bounds = false;
    if (n > cfg.n_scan_max) {  // downsample_to (gaussian_cloud.cpp:134-144)
      down_pts.ensure(static_cast<size_t>(n) * 3);
      bool overflow = false;
      if (n <= 4096) {  // one block, leaf doubling on the device
        CK(scan_downsample_block(prep_work.get(), raw_pts.p, ni, cfg.scan_voxel_leaf, cfg.n_scan_max, down_pts.p, &m,
                                 &overflow, b, ps));
        have_bounds = true;
      } else {
        double leaf = cfg.scan_voxel_leaf;
        CK(scan_voxel_downsample(prep_work.get(), raw_pts.p, ni, leaf, down_pts.p, &m, &overflow, ps));
        while (!overflow && m > cfg.n_scan_max) {
          leaf *= 2.0;
          CK(scan_voxel_downsample(prep_work.get(), raw_pts.p, ni, leaf, down_pts.p, &m, &overflow, ps));
        }
      }
      if (overflow) return host_fallback();
      d_down = down_pts.p;
      lap("downsample");
    }
    const int k = std::min<int>(cfg.covariance_k, m - 1);
    if (k < 4) return empty();
    if (m > kMaxScan) throw std::invalid_argument("scan exceeds the device scan capacity");
    // kNN grid (point_grid.cpp:10-49 over the downsampled points,
    // gaussian_cloud.cpp:24-32 cell size) — scalars on the host.
    if (!have_bounds) {
      CK(scan_bounds(prep_work.get(), d_down, m, b, ps));
      lap("bounds");
    }
    double ext[3];
    for (int a = 0; a < 3; ++a) ext[a] = std::max(b[3 + a] - b[a], 1e-6);
    const double volume = (ext[0] * ext[1]) * ext[2];
    const double per_cell = std::max(1.0, static_cast<double>(k) / 2.0);
    const double cell = std::max(1e-6, std::cbrt(volume * per_cell / static_cast<double>(m)));
    int dims[3];
    for (int a = 0; a < 3; ++a) {
      const double d = std::floor((b[3 + a] - b[a]) / cell) + 1.0;
      if (!(d < 65535.0)) return host_fallback();
      dims[a] = static_cast<int>(d);
    }
    ScanDev& sd = sl.full;
    sd.n = m;
    sd.mu.ensure(static_cast<size_t>(m) * 3);
    sd.sigma.ensure(static_cast<size_t>(m) * 9);
    sd.rec.ensure(2 * static_cast<size_t>(m));
    scan_l1.ensure(static_cast<size_t>(m));
    CK(cudaMemcpyAsync(sd.mu.p, d_down, sizeof(double) * 3 * m, cudaMemcpyDeviceToDevice, ps));
    const double nv = cfg.sensor_noise_sigma * cfg.sensor_noise_sigma;
    CK(scan_knn_cov_records(prep_work.get(), sd.mu.p, m, k, cfg.epsilon_plane, nv > 0.0 ? nv : 0.0, b, cell, dims,
                            sd.sigma.p, sd.rec.p, &sd.structured, &sd.l1max, ps));
    lap("knn+cov+records");
    const int stride = cfg.gn_scan_stride;
    if (stride > 1 && m > 2 * stride) {  // filter.cpp:154-165 strided GN subset
      const int ng = (m + stride - 1) / stride;
      ScanDev& g = sl.gn;
      g.n = ng;
      g.mu.ensure(static_cast<size_t>(ng) * 3);
      g.sigma.ensure(static_cast<size_t>(ng) * 9);
      g.rec.ensure(2 * static_cast<size_t>(ng));
      scan_l1.ensure(static_cast<size_t>(std::max(m, ng)));
      CK(scan_gather_stride(sd.mu.p, sd.sigma.p, ng, stride, g.mu.p, g.sigma.p, ps));
      CK(scan_records(prep_work.get(), g.mu.p, g.sigma.p, ng, g.rec.p, scan_l1.p, &g.structured, &g.l1max, ps));
      sl.gn_alias = false;
    } else {
      sl.gn_alias = true;
    }
    sl.valid = true;
    sl.upload_bytes = g_h2d.load() - h2d0;
  }

  void step_points(const double* points, int64_t n, const smcl_odom* odo, smcl_frame_result* out) {
    if (n_total == 0) throw std::logic_error("FilterEngine::step: not initialized");
    wait_prep_all();
    prepare_slot(0, points, n, st);
    step_slot(0, odo, out);
  }

  bool use_fast(const ScanDev& sd) const {
    // Fast-path queue entries pack (k, ix, iy, iz) in 16-bit fields.
    const bool small_dims = geom.dims[0] < 65535 && geom.dims[1] < 65535 && geom.dims[2] < 65535;
    const bool can = map_structured && sd.structured && sd.n <= kFastMaxScan && small_dims;
    if (cfg.likelihood_mode == 1) return false;
    if (cfg.likelihood_mode == 2) {
      if (!can) throw std::invalid_argument("likelihood_mode=fast needs plane-model map and scan covariances");
      return true;
    }
    return can;
  }

  GicpParamsDev gicp_params(int scan_size) const {
    GicpParamsDev p;
    p.damping_scale = cfg.damping_scale;
    p.omega_max = cfg.omega_max;
    p.v_max = cfg.v_max;
    p.miss_cost = cfg.miss_cost;
    p.min_matched = static_cast<int>(std::ceil(cfg.min_match_fraction * static_cast<double>(scan_size)));
    p.scan_size = scan_size;
    return p;
  }

  // ------------------------------------------------------------ stages
  // need_cost: the GN pass's raw log-likelihood (the stage API returns it;
  // FilterEngine::step overwrites it with the likelihood pass's, so the step
  // does not compute it).
  void run_likelihood(bool gn, const ScanDev& sd, bool need_cost = true) {
    if (!has_map) throw std::invalid_argument("engine has no map");
    if (sd.n == 0) throw std::invalid_argument("gicp::evaluate: empty scan");
    ScanView sv{sd.n, sd.mu.p, sd.sigma.p, sd.structured ? sd.rec.p : nullptr, sd.l1max};
    if (profiling) gn ? mark_it(gn_iter, I_GN0) : mark(E_LL0);
    fast_used = use_fast(sd);
    if (fast_used) {
      MapFast mf{geom, map_fast.p, map_brick, map_occ.p, map_fast.p + 2 * map_records};
      const GicpParamsDev gp0 = gicp_params(sd.n);
      live_list.ensure(static_cast<size_t>(std::max<int64_t>(n_local, 1)));
      live_count.ensure(1);
      // Likelihood pass of a step right after its GN pass: the GN counts
      // predict the gate (k_ll_split); results do not depend on the prediction.
      const bool predict_gate = !gn && profiling && nm_from_gn && gn_gate_thr > 0;
      if (predict_gate) {
        sub_list.ensure(static_cast<size_t>(std::max<int64_t>(n_local, 1)));
        sub_count.ensure(1);
      }
      launch_gicp_fast(gn, poses.p, n_local, sv, mf, sysf.p, raw_ll.p, nm.p, need_cost, gp0.min_matched, live_list.p,
                       live_count.p, st, predict_gate ? gn_gate_thr : 0, predict_gate ? sub_list.p : nullptr,
                       predict_gate ? sub_count.p : nullptr);
      nm_from_gn = gn && profiling;
      gn_gate_thr = gn ? gp0.min_matched : 0;
    } else {
      MapExact me{geom, cells.p, map_mu.p, map_sigma.p};
      if (gn) sys.ensure(static_cast<size_t>(std::max<int64_t>(n_local, 1)) * kSysStride);
      launch_gicp_exact(gn, poses.p, n_local, sv, me, sys.p, raw_ll.p, nm.p, st);
      nm_from_gn = false;
    }
    CK(cudaGetLastError());
    if (profiling) {  // matched particle-points of this pass, summed over the step's passes (counts only)
      gn ? mark_it(gn_iter, I_GN1) : mark(E_LL1);
      // the GN pass's sum comes out of the solve (d_counts[3]); unsharded, the
      // likelihood pass's is the Bayes update's own count (d_counts[1])
      if (!gn && sharded) launch_match_counts(nullptr, nm.p, n_local, d_counts.p + 4, st, /*zero=*/false);
    }
    const GicpParamsDev gp = gicp_params(sd.n);
    if (gn)
      launch_solve(fast_used ? nullptr : sys.p, fast_used ? sysf.p : nullptr, raw_ll.p, nm.p, n_local, gp, steps.p,
                   ll.p, st, profiling ? d_counts.p + 3 : nullptr);
    else
      // in a step the gate also forms the Bayes update's match counts (d_counts[0..1])
      launch_gate_ll(raw_ll.p, nm.p, n_local, gp, ll.p, st, profiling ? d_counts.p : nullptr);
      gate_counted = profiling;
    CK(cudaGetLastError());
    ll_valid = true;
    if (gn) steps_valid = true;
  }

  void predict(const double* delta, const double* cov, uint64_t frame_seed) {
    PredictParams pp{};
    pp.delta = load_pose(delta);
    bool noiseless = true;
    for (int q = 0; q < 36; ++q)
      if (cov[q] != 0.0) noiseless = false;
    pp.noiseless = noiseless ? 1 : 0;
    if (!noiseless) covariance_sqrt(cov, pp.L);
    pp.frame_seed = frame_seed;
    launch_predict(poses.p, n_local, gbase, pp, st);
    poses_changed();
    CK(cudaGetLastError());
  }

  // Pass scalars on the host (neighbor_search.cpp:71-103): identical
  // SplitMix64 + libm as the reference.
  LshPass make_pass(uint64_t pass_seed, const double* bounds) const {
    const int64_t n = n_total;
    SplitMix64 rng(pass_seed);
    LshPass lp{};
    random_rotation(rng, lp.frame.R);
    for (int a = 0; a < 3; ++a) lp.frame.t[a] = rng.uniform_range(bounds[a], bounds[3 + a]);
    double z[6];
    rng.normal6(z);
    for (int c = 0; c < 6; ++c) lp.noise[c] = cfg.lsh_noise_sigma * z[c];
    lp.alpha = cfg.lsh_alpha;
    lp.sigma_r = cfg.sigma_r;
    lp.sigma_t = cfg.sigma_t;
    const int32_t nb = cfg.lsh_n_buckets > 0
                           ? cfg.lsh_n_buckets
                           : next_prime_at_least(static_cast<int32_t>(std::ceil(cfg.lsh_buckets_factor * static_cast<double>(n))));
    lp.n_buckets = nb;
    lp.idx_bits = std::max(1, static_cast<int>(std::bit_width(static_cast<uint64_t>(n - 1))));
    lp.h_bits = std::max(1, static_cast<int>(std::bit_width(static_cast<uint32_t>(nb - 1))));
    lp.prio_bits = std::max(0, 64 - lp.h_bits - lp.idx_bits);
    lp.prio_seed = mix_seed(pass_seed, 0x70726f6974ull);
    return lp;
  }

  // ---- LSH near-integer guard (lsh.cu): speculate, verify, replay.
  // K3 hashes with CUDA's libm and counts the particles whose cell
  // coordinates sit within the libm-discrepancy bound of an integer. After the
  // pass's (or step's) sync, a nonzero count makes the host rehash this
  // shard's particles with glibc (the reference's arithmetic, lsh_key_host);
  // if any key differs, the pre-pass state is restored from the checkpoint
  // and the neighbour pass (and, in a step, everything after it) is replayed
  // on the corrected keys. The checkpoint costs nothing with reorder (the
  // pre-pass arrays survive in the second buffers and SVGD never writes the
  // post-predict pose buffer, see svgd()); without reorder the lists and
  // log-posteriors are copied aside (172 B per particle).
  DBuf<unsigned> lsh_flagged;
  LshPass last_lp{};
  double last_bounds[6] = {};
  bool ckpt_reorder = false;
  const Pose* ckpt_poses = nullptr;
  unsigned long long guard_flagged_total = 0, guard_replays = 0;
  DBuf<int> guard_flag_dev, guard_flag_all;

  void begin_neighbors(uint64_t pass_seed, const double* bounds) {
    last_lp = make_pass(pass_seed, bounds);
    std::memcpy(last_bounds, bounds, sizeof(last_bounds));
    ckpt_poses = poses.p;
    ckpt_reorder = cfg.reorder_particles != 0;
    if (!ckpt_reorder) {
      const size_t nl = static_cast<size_t>(n_local), kk = static_cast<size_t>(k);
      CK(cudaMemcpyAsync(log_post2.p, log_post.p, sizeof(double) * nl, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(idx2.p, idx.p, sizeof(int32_t) * nl * kk, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(kval2.p, kval.p, sizeof(float) * nl * kk, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(count2.p, count.p, sizeof(int32_t) * nl, cudaMemcpyDeviceToDevice, st));
    }
    lsh_flagged.ensure(1 + kGuardListCap);
    launch_lsh_keys(poses.p, n_local, gbase, last_lp, keys.p, lsh_flagged.p, st);
  }

  // After a sync: flagged = this pass's flag count summed over all shards.
  // Rehashes on the host; patches keys.p and returns true when any shard
  // must replay.
  DBuf<Pose> guard_pose;
  DBuf<uint64_t> guard_key;
  bool guard_mismatch(unsigned long long flagged) {
    if (flagged == 0) return false;
    guard_flagged_total += flagged;
    // This shard's flags: only those particles can hash differently on the
    // host, so only they are gathered and rehashed (a whole-shard download
    // and rehash cost ~50 ms at 1M particles).
    unsigned nloc = 0;
    CK(cudaMemcpyAsync(&nloc, lsh_flagged.p, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    sync();
    int mism = 0;
    if (nloc > 0 && nloc <= static_cast<unsigned>(kGuardListCap)) {
      const int m = static_cast<int>(nloc);
      guard_pose.ensure(static_cast<size_t>(m));
      guard_key.ensure(static_cast<size_t>(m));
      launch_gather_flagged(ckpt_poses, keys.p, lsh_flagged.p + 1, m, guard_pose.p, guard_key.p, st);
      std::vector<unsigned> li(static_cast<size_t>(m));
      std::vector<Pose> hp(static_cast<size_t>(m));
      std::vector<uint64_t> hk(static_cast<size_t>(m));
      CK(cudaMemcpyAsync(li.data(), lsh_flagged.p + 1, sizeof(unsigned) * m, cudaMemcpyDeviceToHost, st));
      guard_pose.download(hp.data(), static_cast<size_t>(m), st);
      guard_key.download(hk.data(), static_cast<size_t>(m), st);
      sync();
      for (int q = 0; q < m; ++q) {
        const uint64_t kh = lsh_key_host(hp[static_cast<size_t>(q)], static_cast<uint64_t>(gbase + li[static_cast<size_t>(q)]),
                                         last_lp);
        if (kh != hk[static_cast<size_t>(q)]) {
          hk[static_cast<size_t>(q)] = kh;
          mism = 1;
        }
      }
      if (mism) {
        guard_key.upload(hk.data(), static_cast<size_t>(m), st);
        launch_scatter_keys(keys.p, lsh_flagged.p + 1, m, guard_key.p, st);
      }
    } else if (nloc > 0) {  // more flags than the list holds: rehash the whole shard
      const size_t nl = static_cast<size_t>(n_local);
      std::vector<Pose> hp(nl);
      std::vector<uint64_t> hk(nl);
      CK(cudaMemcpyAsync(hp.data(), ckpt_poses, sizeof(Pose) * nl, cudaMemcpyDeviceToHost, st));
      keys.download(hk.data(), nl, st);
      sync();
#pragma omp parallel for schedule(static) reduction(| : mism)
      for (int64_t i = 0; i < n_local; ++i) {
        const uint64_t kh = lsh_key_host(hp[static_cast<size_t>(i)], static_cast<uint64_t>(gbase + i), last_lp);
        if (kh != hk[static_cast<size_t>(i)]) {
          hk[static_cast<size_t>(i)] = kh;
          mism = 1;
        }
      }
      if (mism) keys.upload(hk.data(), nl, st);
    }
    if (sharded) {  // every shard replays if any shard must
      guard_flag_dev.ensure(1);
      guard_flag_all.ensure(static_cast<size_t>(world));
      CK(cudaMemcpyAsync(guard_flag_dev.p, &mism, sizeof(int), cudaMemcpyHostToDevice, st));
      allgather(guard_flag_dev.p, guard_flag_all.p, sizeof(int));
      std::vector<int> all(static_cast<size_t>(world));
      guard_flag_all.download(all.data(), all.size(), st);
      sync();
      for (int v : all) mism |= v;
    } else {
      sync();
    }
    return mism != 0;
  }

  // Pre-pass state back in place (the pass's outputs are discarded).
  void restore_pass() {
    log_post.swap(log_post2);
    idx.swap(idx2);
    kval.swap(kval2);
    count.swap(count2);
    if (ckpt_reorder) id.swap(id2);
    if (poses.p != ckpt_poses) (poses2.p == ckpt_poses ? poses.swap(poses2) : poses.swap(poses3));
    poses_changed();
    steps_valid = phis_valid = ll_valid = false;
    ++guard_replays;
  }

  // Global flag count of the last K3 (sharded: summed over shards; stage API only).
  unsigned long long flagged_global() {
    unsigned v = 0;
    CK(cudaMemcpyAsync(&v, lsh_flagged.p, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    sync();
    unsigned long long tot = v;
    if (sharded) {
      guard_flag_dev.ensure(1);
      guard_flag_all.ensure(static_cast<size_t>(world));
      const int vi = static_cast<int>(v);
      CK(cudaMemcpyAsync(guard_flag_dev.p, &vi, sizeof(int), cudaMemcpyHostToDevice, st));
      allgather(guard_flag_dev.p, guard_flag_all.p, sizeof(int));
      std::vector<int> all(static_cast<size_t>(world));
      guard_flag_all.download(all.data(), all.size(), st);
      sync();
      tot = 0;
      for (int x : all) tot += static_cast<unsigned long long>(x);
    }
    return tot;
  }

  // Stage API update_neighbors (neighbor_search.cpp:61-192): K3, the rest of
  // the pass, and the guard's verification / replay.
  void update_neighbors(uint64_t pass_seed, const double* bounds, smcl_neighbor_stats* out) {
    if (!begin_pass_checks(out)) return;
    begin_neighbors(pass_seed, bounds);
    neighbor_rest(out);
    if (guard_mismatch(flagged_global())) {
      restore_pass();
      neighbor_rest(out);
    }
  }

  bool begin_pass_checks(smcl_neighbor_stats* out) {
    join_aux();
    nb_out = nullptr;
    if (out) std::memset(out, 0, sizeof(*out));
    if (n_total == 0) return false;
    if (k != cfg.k_neighbors) throw std::invalid_argument("update_neighbors: graph not initialized for this set");
    return true;
  }

  // The neighbour pass after K3: key exchange, sort, reorder, bucket runs,
  // fused refresh + gather, statistics.
  void neighbor_rest(smcl_neighbor_stats* out) {
    const int64_t n = n_total;
    join_aux();
    nb_out = nullptr;
    if (out) std::memset(out, 0, sizeof(*out));
    const LshPass& lp = last_lp;
    const double* bounds = last_bounds;
    const int32_t nb = static_cast<int32_t>(lp.n_buckets);
    const uint64_t idx_mask = (uint64_t(1) << lp.idx_bits) - 1;
    const int shift = lp.prio_bits + lp.idx_bits;
    // Exchange 1: every rank needs all N keys (global sort, bucket
    // runs) and all N poses (candidates of its own particles).
    const uint64_t* keys_all = keys.p;
    if (sharded) {
      allgather(keys.p, g_keys.p, sizeof(uint64_t) * static_cast<size_t>(n_local));
      keys_all = g_keys.p;
    }
    if (profiling) mark(E_KEYS);
    // The keys are in global index order with the index in the low idx_bits
    // (neighbor_search.cpp:86-103): a stable sort of the upper bits suffices.
    sort_keys(keys_all, skeys.p, n, lp.idx_bits, 64, temp.p, temp_bytes, st);
    if (profiling) mark(E_SORT);
    const double anchor[3] = {0.5 * (bounds[0] + bounds[3]), 0.5 * (bounds[1] + bounds[4]),
                              0.5 * (bounds[2] + bounds[5])};  // the pose mirror's translation origin
    bool mirror_ready = false;
    // with reorder, the inverse permutation comes out of the same sweep
    launch_members(skeys.p, n, idx_mask, shift, member_of.p, head.p, st,
                   cfg.reorder_particles ? new_of_old.p : nullptr);
    const int32_t* members = member_of.p;
    bool segments_done = false;
    if (cfg.reorder_particles) {
      if (sharded) {
        // Cross-shard permutation (particle_set.cpp:7-47 over the global
        // order): every rank owns the new positions [gbase, gbase + n_local)
        // and pulls their old state from whichever shard held it. Poses: the
        // new global order is a permutation of the gathered old one, applied
        // locally by every rank (no second gather). The rest of the state
        // (16 + 8K B per particle) moves by alltoallv, only the particles
        // that change shard; without alltoallv, by all-gather of everything.
        const size_t nl = static_cast<size_t>(n_local), kk = static_cast<size_t>(k);
        all_poses();  // old poses of every particle (cached gather)
        if (comm.alltoallv) {
          migrate_begin();
          // bucket runs depend only on the sorted keys: computed while the host reads the counts
          inclusive_sum_i32(head.p, seg_id.p, n, temp.p, temp_bytes, st);
          launch_segments(head.p, seg_id.p, n, seg_start.p, st);
          segments_done = true;
          migrate_finish();
        } else {
          allgather(log_post.p, g_lp.p, sizeof(double) * nl);
          allgather(id.p, g_id.p, sizeof(int32_t) * nl);
          allgather(count.p, g_count.p, sizeof(int32_t) * nl);
          allgather(idx.p, g_idx.p, sizeof(int32_t) * nl * kk);
          allgather(kval.p, g_kval.p, sizeof(float) * nl * kk);
          launch_reorder(member_of.p + gbase, new_of_old.p, n_local, k, g_poses.p, g_lp.p, g_id.p, g_idx.p, g_kval.p,
                         g_count.p, poses2.p, log_post2.p, id2.p, idx2.p, kval2.p, count2.p, st);
        }
        launch_permute_poses(member_of.p, n, g_poses.p, g_poses2.p, st);
        g_poses.swap(g_poses2);
        if (comm.alltoallv)
          CK(cudaMemcpyAsync(poses2.p, g_poses.p + gbase, sizeof(Pose) * nl, cudaMemcpyDeviceToDevice, st));
      } else {  // the neighbour pass's fp32 pose mirror is written by the same sweep
        pose_mirror.ensure(3 * static_cast<size_t>(n));
        mirror_tmax.ensure(1);
        mirror_ready = launch_reorder(member_of.p, new_of_old.p, n, k, poses.p, log_post.p, id.p, idx.p, kval.p,
                                      count.p, poses2.p, log_post2.p, id2.p, idx2.p, kval2.p, count2.p, st,
                                      pose_mirror.p, mirror_tmax.p, anchor);
      }
      poses.swap(poses2);
      log_post.swap(log_post2);
      id.swap(id2);
      idx.swap(idx2);
      kval.swap(kval2);
      count.swap(count2);
      members = iota.p;
      steps_valid = phis_valid = ll_valid = false;  // storage order changed
      g_poses_valid = sharded;  // sharded: g_poses already holds the permuted global array
    }
    const Pose* poses_all = all_poses();  // after the reorder: candidates read the current storage
    if (profiling) mark(E_REORDER);
    if (!segments_done) {
      inclusive_sum_i32(head.p, seg_id.p, n, temp.p, temp_bytes, st);
      launch_segments(head.p, seg_id.p, n, seg_start.p, st);
    }
    const int32_t* n_seg = seg_id.p + (n - 1);  // number of buckets (device)
    // Sorted positions of this shard's particles, in sorted order.
    const int32_t* owned = nullptr;
    if (sharded) {
      launch_owned_flags(members, n, gbase, n_local, g_flag.p, st);
      inclusive_sum_i32(g_flag.p, new_of_old.p, n, temp.p, temp_bytes, st);
      launch_owned_scatter(g_flag.p, new_of_old.p, n, pos_list.p, st);
      owned = pos_list.p;
    }
    if (profiling) mark(E_SEG);
    // Sorted position of every particle, for the neighbour pass's duplicate
    // test: the identity after a reorder, else the inverse of member_of.
    const int32_t* pos_of = nullptr;
    if (members != iota.p) {
      pos_of_buf.ensure(static_cast<size_t>(n));
      launch_inverse_perm(members, n, pos_of_buf.p, st);
      pos_of = pos_of_buf.p;
    }
    pose_mirror.ensure(3 * static_cast<size_t>(n));
    mirror_tmax.ensure(1);
    launch_refresh_gather(poses_all, n_local, gbase, owned, members, seg_id.p, seg_start.p, n, pos_of, idx.p,
                          kval.p, count.p, k, cfg.lsh_bucket_capacity, cfg.sigma_r, cfg.sigma_t, anchor,
                          pose_mirror.p, mirror_tmax.p, st, mirror_ready);
    CK(cudaGetLastError());
    if (profiling) mark(E_RG);
    // statistics (neighbor_search.cpp:172-190)
    const int hist_len = cfg.lsh_bucket_capacity + 2;
    if (hist_len > SMCL_MAX_HIST) throw std::invalid_argument("lsh_bucket_capacity too large for the statistics");
    cudaStream_t ss = st;
    if (!sharded) {  // overlapped with the rest of the step
      CK(cudaEventRecord(ev_fork, st));
      CK(cudaStreamWaitEvent(aux, ev_fork, 0));
      ss = aux;
    }
    CK(cudaMemsetAsync(nb_hist.p, 0, sizeof(unsigned long long) * (SMCL_MAX_HIST + 1), ss));
    launch_seg_stats(seg_start.p, n_seg, n, cfg.lsh_bucket_capacity, nb_hist.p, nb_hist.p + SMCL_MAX_HIST, ss);
    const int64_t chunks = (n_local + kReduceChunk - 1) / kReduceChunk;
    launch_chunk_sum_kernel(kval.p, count.p, n_local, k, nb_s1.p, nb_s2.p, nb_p1.p, nb_p2.p, ss);
    if (sharded) {  // chunk partials of every shard, combined in global chunk order
      allgather(nb_p1.p, g_part.p, sizeof(double) * static_cast<size_t>(chunks));
      allgather(nb_p2.p, g_part2.p, sizeof(double) * static_cast<size_t>(chunks));
      launch_finish_sum2(g_part.p, g_part2.p, chunks * world, nb_sum.p, ss);
    } else {
      launch_finish_sum2(nb_p1.p, nb_p2.p, chunks, nb_sum.p, ss);
    }
    CK(cudaGetLastError());
    if (out) {  // read back after the call's final sync (finish_nb_stats)
      CK(cudaMemcpyAsync(nb_host->hist, nb_hist.p, sizeof(unsigned long long) * (SMCL_MAX_HIST + 1),
                         cudaMemcpyDeviceToHost, ss));
      CK(cudaMemcpyAsync(nb_host->sums, nb_sum.p, sizeof(double) * 2, cudaMemcpyDeviceToHost, ss));
      CK(cudaMemcpyAsync(&nb_host->n_seg, n_seg, sizeof(int32_t), cudaMemcpyDeviceToHost, ss));
      g_d2h += static_cast<long long>(sizeof(unsigned long long) * (SMCL_MAX_HIST + 1) + 2 * sizeof(double) +
                                      sizeof(int32_t));
      nb_out = out;
      nb_buckets = nb;
      nb_hist_len = hist_len;
    }
    if (!sharded) {
      CK(cudaEventRecord(ev_join, aux));
      aux_pending = true;
    }
  }

  void svgd(bool fused_apply) {
    SvgdParams sp{cfg.sigma_r, cfg.sigma_t, cfg.repulsion_gain};
    // Exchange 2: neighbours' poses and Gauss-Newton steps.
    const Pose* pa = all_poses();
    const double* sa = all_steps();
    if (fused_apply) {  // into whichever spare buffer does not hold the post-predict checkpoint
      DBuf<Pose>& dst = poses2.p != ckpt_poses ? poses2 : poses3;
      launch_svgd(pa, sa, n_local, gbase, idx.p, count.p, k, sp, nullptr, dst.p, st);
      poses.swap(dst);
      poses_changed();
    } else {
      launch_svgd(pa, sa, n_local, gbase, idx.p, count.p, k, sp, phis.p, nullptr, st);
      phis_valid = true;
    }
    CK(cudaGetLastError());
  }

  // Global argmax (value, index; ties -> lowest index) of log_post into
  // scal[slot], scal_i[slot_i]: per-shard partial, all-gathered, merged.
  void global_argmax(int slot, int slot_i) {
    if (sharded) {  // this shard's (value, index) as one 16-byte pair: one all-gather
      launch_argmax(log_post.p, n_local, gbase, argv.p, argi.p, arg_pair.p,
                    reinterpret_cast<long long*>(arg_pair.p + 1), st);
      allgather(arg_pair.p, g_argv.p, 2 * sizeof(double));
      launch_merge_pairs(g_argv.p, world, scal.p + slot, scal_i.p + slot_i, st);
    } else {
      launch_argmax(log_post.p, n_local, gbase, argv.p, argi.p, scal.p + slot, scal_i.p + slot_i, st);
    }
  }

  // p_out (optional): exp of the normalised log-posterior, the smoothing
  // pass's input, written by the same sweep.
  // rep_parts (unsharded): also leave the argmax partials of the result in
  // argv/argi for representative_enqueue; returns whether it did.
  // numer (unsharded): apply the Bayes numerator (k_bayes_numer) in the
  // argmax sweep first.
  struct Numer {
    double beta, fill;
    const unsigned long long* matched;
  };
  bool gate_counted = false;  // this step's gate already formed d_counts[0..1]
  bool normalize(double floor_v, const unsigned long long* skip_if_zero = nullptr, double* p_out = nullptr,
                 bool rep_parts = false, const Numer* numer = nullptr) {
    const int64_t n = n_local;
    if (n == 0) return false;
    const int64_t chunks_local = (n + kReduceChunk - 1) / kReduceChunk;
    if (!sharded) {  // three launches: argmax partials, chunk sums (max from the partials), finish + apply
      if (numer)
        launch_numer_argmax_partials(log_post.p, ll.p, nm.p, n, gbase, numer->beta, numer->matched, numer->fill,
                                     argv.p, argi.p, st);
      else
        launch_argmax_partials(log_post.p, n, gbase, argv.p, argi.p, st);
      launch_chunk_sum_exp_parts(log_post.p, n, argv.p, argmax_partials(n), scal.p + 2, partial.p, st);
      launch_apply_lse_fin(log_post.p, n, partial.p, chunks_local, scal.p + 2, floor_v, skip_if_zero, scal.p + 3,
                           p_out, gbase, rep_parts ? argv.p : nullptr, rep_parts ? argi.p : nullptr, st);
      CK(cudaGetLastError());
      return rep_parts;
    }
    if (numer) launch_bayes_numer(log_post.p, ll.p, nm.p, n, numer->beta, numer->matched, numer->fill, st);
    global_argmax(2, 0);
    launch_chunk_sum_exp(log_post.p, n, scal.p + 2, partial.p, st);
    const int64_t chunks = (n + kReduceChunk - 1) / kReduceChunk;
    if (sharded) {  // reduce.hpp order: every chunk partial, in global chunk order
      allgather(partial.p, g_part.p, sizeof(double) * static_cast<size_t>(chunks));
      launch_finish_lse(g_part.p, chunks * world, scal.p + 2, scal.p + 3, st);
    } else {
      launch_finish_lse(partial.p, chunks, scal.p + 2, scal.p + 3, st);
    }
    launch_apply_lse(log_post.p, n, scal.p + 3, floor_v, st, skip_if_zero);
    if (p_out) launch_exp(log_post.p, p_out, n, st);
    CK(cudaGetLastError());
    return false;
  }

  // (matched particles, sum of n_matched) over all shards: exact integers.
  void global_match_counts(unsigned long long* cnt) {
    launch_match_counts(ll.p, nm.p, n_local, d_counts.p, st);
    if (sharded) {
      allgather(d_counts.p, g_counts.p, 2 * sizeof(unsigned long long));
      std::vector<unsigned long long> all(2 * static_cast<size_t>(world));
      g_counts.download(all.data(), all.size(), st);
      sync();
      cnt[0] = cnt[1] = 0;
      for (int r = 0; r < world; ++r) {
        cnt[0] += all[2 * static_cast<size_t>(r)];
        cnt[1] += all[2 * static_cast<size_t>(r) + 1];
      }
      return;
    }
    d_counts.download(cnt, 2, st);
    sync();
  }

  // Returns observation_rejected.
  bool bayes(double beta, double floor_v) {
    if (!(beta >= 0.0)) throw std::invalid_argument("bayes_update: beta must be >= 0");
    const int64_t n = n_local;
    if (n == 0) return false;
    unsigned long long cnt[2];
    global_match_counts(cnt);
    last_nm_sum = cnt[1];
    if (cnt[0] == 0) {
      launch_fill(log_post.p, n, -std::log(static_cast<double>(n_total)), st);
      return true;
    }
    launch_bayes_numer(log_post.p, ll.p, nm.p, n, beta, nullptr, 0.0, st);
    normalize(floor_v);
    return false;
  }

  // bayes() without the host round trip (the step's form): the match counts
  // stay in d_counts[0..1], the uniform reset and the skipped normalization of
  // a rejected observation are decided on the device; the caller reads the
  // counts with its end-of-step sync.
  void bayes_async(double beta, double floor_v, double* p_out = nullptr) {
    if (!(beta >= 0.0)) throw std::invalid_argument("bayes_update: beta must be >= 0");
    const int64_t n = n_local;
    if (n == 0) return;
    if (!gate_counted) launch_match_counts(ll.p, nm.p, n_local, d_counts.p, st);
    gate_counted = false;
    if (sharded) {
      allgather(d_counts.p, g_counts.p, 2 * sizeof(unsigned long long));
      launch_sum_pairs(g_counts.p, world, d_counts.p, st);
    }
    // numerator, normalisation and (the step's smoothing follows) its
    // exp(log_post), fused where unsharded
    const Numer numer{beta, -std::log(static_cast<double>(n_total)), d_counts.p};
    normalize(floor_v, d_counts.p, p_out, false, &numer);
  }

  // p_ready: pbuf already holds exp(log_post) (bayes_async's normalisation).
  // rep_parts: leave the representative's argmax partials (see normalize);
  // returns whether they were left.
  bool smooth(int iters, double floor_v, bool p_ready = false, bool rep_parts = false) {
    if (iters < 0) throw std::invalid_argument("smooth: iters must be >= 0");
    const int64_t n = n_local;
    if (n == 0 || iters == 0) return false;
    if (!p_ready) launch_exp(log_post.p, pbuf.p, n, st);
    for (int r = 0; r < iters; ++r) {
      // Exchange 3: neighbours' probabilities every round.
      const double* p_all = pbuf.p;
      if (sharded) {
        allgather(pbuf.p, g_p.p, sizeof(double) * static_cast<size_t>(n));
        p_all = g_p.p;
      }
      // the last round writes log(q) straight into log_post (posterior.cpp:94)
      const bool last = r + 1 == iters;
      // alternate sweep directions: each round starts on the L2-resident rows
      static const bool no_rev = std::getenv("SMCL_SMOOTH_NOREV") != nullptr;  // A/B
      launch_smooth_round(p_all, last ? log_post.p : qbuf.p, n, idx.p, kval.p, count.p, k, st, last,
                          !no_rev && (r & 1) != 0);
      pbuf.swap(qbuf);
    }
    CK(cudaGetLastError());
    return normalize(floor_v, nullptr, nullptr, rep_parts);
  }

  void representative(int64_t* index, double* pose, double* value) {
    representative_enqueue();
    sync();
    representative_read(index, pose, value);
  }
  // Value, index, pose and id of the winner gathered on the device into one
  // staging record, read back into pinned memory (no host round trip until
  // the caller's sync).
  // rep_stage[15] (sharded: summed over shards): the last K3's hash-guard flag count.
  // parts_ready: argv/argi hold the argmax partials of the current
  // log-posterior (left by the step's final normalisation, unsharded).
  void representative_enqueue(bool parts_ready = false) {
    if (n_local == 0) throw std::invalid_argument("representative: empty or mismatched particle set");
    lsh_flagged.ensure(1);
    if (parts_ready && !sharded)
      launch_max_of_partials(argv.p, argi.p, apply_fin_blocks(n_local), scal.p + 4, scal_i.p + 1, st);
    else
      global_argmax(4, 1);
    rep_stage.ensure(16);
    if (sharded) {  // the owner rank publishes the winner's pose and id (one slot per rank)
      double* mine = g_rep.p + 14 * static_cast<size_t>(rank);
      launch_rep_local(scal.p + 4, scal_i.p + 1, n_local, rank, true, poses.p, id.p, lsh_flagged.p,
                       reinterpret_cast<Pose*>(mine), nullptr, nullptr, st);
      allgather(mine, g_rep.p, 14 * sizeof(double));
      launch_rep_select(scal.p + 4, scal_i.p + 1, n_local, world, g_rep.p, rep_stage.p, st);
    } else {
      launch_rep_local(scal.p + 4, scal_i.p + 1, n_local, 0, false, poses.p, id.p, lsh_flagged.p, nullptr, nullptr,
                       rep_stage.p, st);
    }
    CK(cudaMemcpyAsync(step_host->rep, rep_stage.p, sizeof(double) * 16, cudaMemcpyDeviceToHost, st));
    g_d2h += sizeof(double) * 16;
  }
  void representative_read(int64_t* index, double* pose, double* value) {  // after a sync
    const double* h = step_host->rep;
    *value = h[0];
    long long ix;
    std::memcpy(&ix, &h[1], sizeof(ix));
    *index = ix;
    rep_id = static_cast<int32_t>(h[14]);
    if (pose) {
      Pose p;
      for (int q = 0; q < 9; ++q) p.R[q] = h[2 + q];
      for (int a = 0; a < 3; ++a) p.t[a] = h[11 + a];
      store_pose(p, pose);
    }
  }

  void init_uniform(int64_t n, const double* b, bool full_rotation, uint64_t seed) {
    if (n < 1) throw std::invalid_argument("init_uniform: n_particles must be >= 1");
    for (int a = 0; a < 3; ++a)
      if (b[3 + a] - b[a] <= 0.0) throw std::invalid_argument("init_uniform: degenerate bounds");
    if (cfg.k_neighbors < 1 || cfg.k_neighbors > kMaxK)
      throw std::invalid_argument("k_neighbors must be in [1, 32] on this device build");
    set_shape(n);
    alloc_particles(n_local, cfg.k_neighbors);
    InitParams ip{};
    ip.stream = mix_seed(seed, k_stream_init);
    for (int a = 0; a < 3; ++a) {
      ip.bmin[a] = b[a];
      ip.bmax[a] = b[3 + a];
    }
    ip.log_post0 = -std::log(static_cast<double>(n));
    ip.full_rotation = full_rotation ? 1 : 0;
    launch_init_uniform(poses.p, log_post.p, id.p, idx.p, kval.p, count.p, n_local, gbase, k, ip, st);
    poses_changed();
    CK(cudaGetLastError());
    sync();
  }

  void step_slot(int slot_i, const smcl_odom* odo, smcl_frame_result* out) {
    if (n_total == 0) throw std::logic_error("FilterEngine::step: not initialized");
    if (!has_map) throw std::invalid_argument("engine has no map");
    wait_slot(slot_i);
    ScanSlot& sl = slot_at(slot_i);
    if (!sl.valid) throw std::invalid_argument("scan slot not uploaded");
    static const bool host_timing = std::getenv("SMCL_HOST_TIMING") != nullptr;  // diagnostics: host time around the GPU work
    const auto h0 = std::chrono::steady_clock::now();
    profiling = true;
    struct ProfilingOff {  // cleared on every exit path (a throwing stage must not leave the step's events armed)
      bool& f;
      bool& nvtx;
      ~ProfilingOff() {
        f = false;
        if (nvtx) nvtxRangePop();  // the open stage range
        nvtx = false;
        nvtxRangePop();  // the step range
      }
    } profiling_off{profiling, nvtx_open};
    nvtxRangePushA("smcl::step");
    const long long launches0 = launch_count();
    const long long d2h0 = g_d2h.load();
    smcl_frame_result r;
    std::memset(&r, 0, sizeof(r));
    std::memset(&prof, 0, sizeof(prof));
    prof_times_pending = false;
    nm_from_gn = false;  // set again by this step's GN pass (the likelihood gate's prediction)
    gate_counted = false;
    r.n_particles = n_total;
    const bool empty = sl.full.n == 0;
    r.scan_empty = empty ? 1 : 0;
    CK(cudaMemsetAsync(d_counts.p, 0, sizeof(unsigned long long) * 6, st));

    mark(E_START);
    {
      double delta[12], cov[36];
      if (odo->valid) {
        std::memcpy(delta, odo->delta, sizeof(delta));
        std::memcpy(cov, odo->cov, sizeof(cov));
      } else {
        store_pose(pose_identity(), delta);
        std::memset(cov, 0, sizeof(cov));
        for (int d = 0; d < 3; ++d) {
          cov[d * 7] = cfg.diffusion_sigma_rot * cfg.diffusion_sigma_rot;
          cov[(d + 3) * 7] = cfg.diffusion_sigma_trans * cfg.diffusion_sigma_trans;
        }
      }
      predict(delta, cov, mix_seed(cfg.seed, k_stream_predict, static_cast<uint64_t>(frame)));
    }
    const auto h1 = std::chrono::steady_clock::now();
    mark(E_PRED);
    const double bounds[6] = {map_bounds.min[0], map_bounds.min[1], map_bounds.min[2],
                              map_bounds.max[0], map_bounds.max[1], map_bounds.max[2]};
    int64_t ix;
    double v;
    begin_pass_checks(&r.neighbor_stats);
    begin_neighbors(mix_seed(cfg.seed, k_stream_neighbors, static_cast<uint64_t>(frame)), bounds);  // K3
    double t_like = 0.0, t_upd = 0.0, t_gn = 0.0, t_solve = 0.0, t_svgd = 0.0;
    const ScanDev& gn_scan = sl.gn_view();
    // Everything after K3, up to the end-of-frame readback and sync; run a
    // second time only if the hash guard finds a key to correct.
    std::chrono::steady_clock::time_point h_sync;
    auto run_from_keys = [&]() {
      bool p_ready = false;  // pbuf = exp(log_post) from the Bayes normalisation
      neighbor_rest(&r.neighbor_stats);
      mark(E_NB);
      if (!empty) {
        for (int it = 0; it < cfg.n_svgd_iters; ++it) {  // filter.cpp:166-180
          gn_iter = it;
          run_likelihood(true, gn_scan, /*need_cost=*/false);
          mark_it(it, I_SOLVE);
          mark_it(it, I_SV0);
          svgd(true);
          mark_it(it, I_SVGD);
        }
        run_likelihood(false, sl.full);
        mark(E_BAYES);
        // rejection flag read at the end of the step; exp(log_post) for the smoothing rides along
        bayes_async(cfg.beta, cfg.log_post_floor, cfg.smooth_iters > 0 ? pbuf.p : nullptr);
        p_ready = cfg.smooth_iters > 0;
      } else {
        mark(E_LL0);
        mark(E_LL1);
        mark(E_BAYES);
      }
      mark(E_SMOOTH);  // posterior smoothing starts
      const bool rep_parts = smooth(cfg.smooth_iters, cfg.log_post_floor, p_ready, /*rep_parts=*/true);
      mark(E_END);
      representative_enqueue(rep_parts);
      join_aux();
      CK(cudaMemcpyAsync(step_host->cnt, d_counts.p, sizeof(unsigned long long) * 6, cudaMemcpyDeviceToHost, st));
      g_d2h += sizeof(unsigned long long) * 6;
      sync();  // the step's one end-of-frame host synchronisation
      h_sync = std::chrono::steady_clock::now();
    };
    run_from_keys();
    // step_host->rep[15]: this pass's hash-guard flags, summed over all shards
    if (guard_mismatch(static_cast<unsigned long long>(step_host->rep[15]))) {
      restore_pass();
      CK(cudaMemsetAsync(d_counts.p, 0, sizeof(unsigned long long) * 6, st));
      run_from_keys();
    }
    representative_read(&ix, r.representative, &v);
    unsigned long long cnt[6];
    std::memcpy(cnt, step_host->cnt, sizeof(cnt));
    const int32_t rid = rep_id;
    if (!empty) {  // bayes_async: global (matched particles, sum of n_matched)
      r.observation_rejected = cnt[0] == 0 ? 1 : 0;
      last_nm_sum = cnt[1];
    }
    finish_nb_stats();
    if (!empty)
      for (int it = 0; it < cfg.n_svgd_iters; ++it) {
        t_gn += since_it(it, I_GN0, I_GN1);
        t_solve += since_it(it, I_GN1, I_SOLVE);
        t_svgd += since_it(it, I_SV0, I_SVGD);
      }
    static const bool timeline = std::getenv("SMCL_STEP_TIMELINE") != nullptr;  // diagnostics: event offsets
    if (timeline) {
      static const char* names[E_COUNT] = {"start", "pred", "keys", "sort", "reorder", "seg", "rg", "nb",
                                           "ll0", "ll1", "bayes", "smooth", "end"};
      std::fprintf(stderr, "[timeline]");
      for (int e = 1; e < E_COUNT; ++e) std::fprintf(stderr, " %s=%.3f", names[e], since(E_START, static_cast<Ev>(e)));
      static const char* inames[I_COUNT] = {"gn0", "gn1", "solve", "sv0", "svgd"};
      for (int it = 0; it < (empty ? 0 : cfg.n_svgd_iters); ++it)
        for (int e = 0; e < I_COUNT; ++e) std::fprintf(stderr, " %s%d=%.3f", inames[e], it, since_it_ev(ev[E_START], it, static_cast<ItEv>(e)));
      std::fprintf(stderr, "\n");
    }
    t_like = t_gn + t_solve;
    t_upd = t_svgd;
    const double t_ll = since(E_LL0, E_BAYES);
    r.mean_n_matched = empty ? 0.0 : static_cast<double>(cnt[1]) / static_cast<double>(n_total);
    r.rep_index = ix;
    r.rep_log_post = v;
    r.rep_id = rid;
    r.predict_ms = since(E_START, E_PRED);
    r.neighbor_ms = since(E_PRED, E_NB);
    r.likelihood_ms = t_like + t_ll;
    r.update_ms = t_upd;
    r.posterior_ms = since(E_BAYES, E_END);
    r.total_ms = since(E_START, E_END);
    // per-kernel profile
    // per-kernel stage times: read from the events on the first
    // smcl_last_step_profile call (fill_prof_times), not on every step
    prof.predict_ms = r.predict_ms;
    prof.gn_kernel_ms = t_gn;
    prof.solve_ms = t_solve;
    prof.svgd_ms = t_svgd;
    prof.total_ms = r.total_ms;
    prof_times_pending = true;
    prof_empty = empty;
    prof.gn_points = empty ? 0 : static_cast<int64_t>(gn_scan.n) * n_total * cfg.n_svgd_iters;
    prof.ll_points = empty ? 0 : static_cast<int64_t>(sl.full.n) * n_total;
    prof.gn_matched = static_cast<int64_t>(cnt[3]);
    prof.ll_matched = static_cast<int64_t>(sharded ? cnt[5] : (empty ? 0 : cnt[1]));
    prof.fast_path = fast_used ? 1 : 0;
    prof.n_svgd_iters = cfg.n_svgd_iters;
    prof.kernel_launches = launch_count() - launches0;
    prof.d2h_bytes = g_d2h.load() - d2h0;
    prof.h2d_bytes = sl.upload_bytes;
    *out = r;
    ++frame;
    if (host_timing) {
      const auto h2 = std::chrono::steady_clock::now();
      auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
      std::fprintf(stderr, "[host] enter->predict launched %.1f us, sync return->exit %.1f us\n", us(h0, h1),
                   us(h_sync, h2));
    }
  }

  void step(const smcl_cloud* scan, const smcl_odom* odo, smcl_frame_result* out) {
    if (n_total == 0) throw std::logic_error("FilterEngine::step: not initialized");
    set_slot(0, scan);  // host scan prep + H2D (inside the caller's e2e timing)
    step_slot(0, odo, out);
  }
};

// ---------------------------------------------------------------- C ABI
namespace {
smcl_engine* make_engine(const smcl_cloud* map, const smcl_config* cfg, int device) {
  if (!cfg) throw std::invalid_argument("config must not be null");
  auto e = std::make_unique<smcl_engine>();
  e->cfg = *cfg;
  if (device >= 0) {
    CK(cudaSetDevice(device));
    e->device = device;
  } else {
    CK(cudaGetDevice(&e->device));
  }
  CK(cudaStreamCreateWithFlags(&e->st, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&e->aux, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming));
  CK(cudaMallocHost(reinterpret_cast<void**>(&e->nb_host), sizeof(smcl_engine::NbHost)));
  CK(cudaMallocHost(reinterpret_cast<void**>(&e->step_host), sizeof(smcl_engine::StepHost)));
  for (int q = 0; q < SMCL_MAX_SCAN_SLOTS; ++q) e->slots.push_back(std::make_unique<smcl_engine::ScanSlot>());
  e->k = cfg->k_neighbors;
  if (map) e->setup_map(map);
  return e.release();
}
inline void use_dev(const smcl_engine* h) {
  if (!h) throw std::invalid_argument("null engine handle");
  CK(cudaSetDevice(h->device));
}
}  // namespace

extern "C" {

int smcl_abi_version(void) { return SMCL_ABI_VERSION; }
const char* smcl_last_error(void) { return g_last_error.c_str(); }

void smcl_config_default(smcl_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->n_particles = 10000;
  c->k_neighbors = 20;
  c->sigma_r = 5.0;
  c->sigma_t = 2.5;
  c->repulsion_gain = 1.0;
  c->lsh_alpha = 0.1;
  c->lsh_noise_sigma = 0.5;
  c->lsh_buckets_factor = 2.0;
  c->lsh_n_buckets = 0;
  c->lsh_bucket_capacity = 64;
  c->reorder_particles = 1;
  c->smooth_iters = 10;
  c->nnf_resolution = 0.1;
  c->nnf_max_query_dist = 1.0;
  c->nnf_padding = 0.5;
  c->beta = 2.0;
  c->n_svgd_iters = 1;
  c->gn_scan_stride = 1;
  c->damping_scale = 1e-3;
  c->omega_max = 0.5;
  c->v_max = 1.0;
  c->min_match_fraction = 0.5;
  c->miss_cost = 25.0;
  c->log_post_floor = -80.0;
  c->covariance_k = 10;
  c->n_scan_max = 1000;
  c->epsilon_plane = 1e-3;
  c->scan_voxel_leaf = 0.05;
  c->sensor_noise_sigma = 0.01;
  c->diffusion_sigma_rot = 0.02;
  c->diffusion_sigma_trans = 0.5;
  c->full_rotation = 1;
  c->likelihood_mode = 0;
  c->seed = 1;
}

int smcl_device_count(int* out) {
  return guard([&] { CK(cudaGetDeviceCount(out)); });
}

int smcl_create(const smcl_cloud* map, const smcl_config* cfg, int device, smcl_engine** out) {
  return guard([&] { *out = make_engine(map, cfg, device); });
}

int smcl_create_sharded(const smcl_cloud* map, const smcl_config* cfg, int device, const smcl_comm* comm,
                        smcl_engine** out) {
  return guard([&] {
    if (!comm || comm->world < 1 || comm->rank < 0 || comm->rank >= comm->world || !comm->allgather)
      throw std::invalid_argument("smcl_create_sharded: invalid communicator");
    std::unique_ptr<smcl_engine> e(make_engine(map, cfg, device));
    e->comm = *comm;
    e->rank = comm->rank;
    e->world = comm->world;
    e->sharded = comm->world > 1;
    *out = e.release();
  });
}

// ---------------------------------------------------------------- loopback collectives
namespace {
struct LoopShared {
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<const void*> send;
  std::vector<std::vector<uint64_t>> send_bytes;  // alltoallv: per rank, bytes to each destination
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};
struct LoopRank {
  std::shared_ptr<LoopShared> shared;
  int rank;
};
// Every rank posts its send pointer, then copies all ranks' buffers into its
// own recv on its own stream; host barriers order the phases (no device-side
// waiting between kernels of different ranks).
int loopback_allgather(void* ctx, const void* send, void* recv, uint64_t bytes, void* stream) {
  auto* lr = static_cast<LoopRank*>(ctx);
  LoopShared& sh = *lr->shared;
  auto st = static_cast<cudaStream_t>(stream);
  if (cudaStreamSynchronize(st) != cudaSuccess) return 1;
  sh.send[static_cast<size_t>(lr->rank)] = send;
  sh.barrier();
  for (int r = 0; r < sh.world; ++r) {
    char* dst = static_cast<char*>(recv) + static_cast<size_t>(r) * bytes;
    const void* src = sh.send[static_cast<size_t>(r)];
    if (src == dst) continue;  // in place
    if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return 1;
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) return 1;
  sh.barrier();  // no rank reuses its send buffer before every rank has read it
  return 0;
}
// alltoallv: every rank posts its packed send buffer and per-destination
// sizes; each rank then copies the chunk addressed to it out of every peer's
// buffer (the chunk's offset = the peer's bytes to lower ranks).
int loopback_alltoallv(void* ctx, const void* send, const uint64_t* send_bytes, void* recv, const uint64_t* recv_bytes,
                       void* stream) {
  auto* lr = static_cast<LoopRank*>(ctx);
  LoopShared& sh = *lr->shared;
  auto st = static_cast<cudaStream_t>(stream);
  const size_t w = static_cast<size_t>(sh.world), me = static_cast<size_t>(lr->rank);
  if (cudaStreamSynchronize(st) != cudaSuccess) return 1;
  sh.send[me] = send;
  sh.send_bytes[me].assign(send_bytes, send_bytes + w);
  sh.barrier();
  int rc = 0;
  uint64_t roff = 0;
  for (size_t s = 0; s < w && rc == 0; ++s) {
    const std::vector<uint64_t>& sb = sh.send_bytes[s];
    uint64_t soff = 0;
    for (size_t d = 0; d < me; ++d) soff += sb[d];
    if (sb[me] != recv_bytes[s]) rc = 1;  // sender and receiver disagree on the chunk size
    else if (sb[me] && cudaMemcpyAsync(static_cast<char*>(recv) + roff, static_cast<const char*>(sh.send[s]) + soff,
                                       sb[me], cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      rc = 1;
    roff += recv_bytes[s];
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) rc = 1;
  sh.barrier();  // always reached by every rank: no deadlock on a failed rank
  return rc;
}
}  // namespace

int smcl_comm_loopback_create(int32_t world, smcl_comm* comms) {
  return guard([&] {
    if (world < 1) throw std::invalid_argument("loopback: world must be >= 1");
    auto sh = std::make_shared<LoopShared>();
    sh->world = world;
    sh->send.assign(static_cast<size_t>(world), nullptr);
    sh->send_bytes.assign(static_cast<size_t>(world), {});
    for (int r = 0; r < world; ++r) {
      comms[r].ctx = new LoopRank{sh, r};
      comms[r].rank = r;
      comms[r].world = world;
      comms[r].allgather = loopback_allgather;
      comms[r].alltoallv = loopback_alltoallv;
    }
  });
}

void smcl_comm_loopback_destroy(smcl_comm* comms) {
  if (!comms) return;
  const int world = comms[0].world;
  for (int r = 0; r < world; ++r) {
    delete static_cast<LoopRank*>(comms[r].ctx);
    comms[r].ctx = nullptr;
  }
}

int smcl_destroy(smcl_engine* h) {
  return guard([&] { delete h; });
}

int smcl_init_uniform(smcl_engine* h, const double bounds[6]) {
  return guard([&] {
    use_dev(h);
    h->init_uniform(h->cfg.n_particles, bounds, h->cfg.full_rotation != 0, h->cfg.seed);
    h->frame = 0;
  });
}

int smcl_init_uniform_seeded(smcl_engine* h, int64_t n, const double bounds[6], int full_rotation, uint64_t seed) {
  return guard([&] {
    use_dev(h);
    h->init_uniform(n, bounds, full_rotation != 0, seed);
  });
}

int smcl_step(smcl_engine* h, const smcl_cloud* scan, const smcl_odom* odo, smcl_frame_result* out) {
  return guard([&] {
    use_dev(h);
    if (!odo || !out) throw std::invalid_argument("smcl_step: null odometry or result");
    h->step(scan, odo, out);
  });
}

int smcl_scan_upload(smcl_engine* h, int slot, const smcl_cloud* scan) {
  return guard([&] {
    use_dev(h);
    h->set_slot(slot, scan);
    h->sync();
  });
}

int smcl_step_slot(smcl_engine* h, int slot, const smcl_odom* odo, smcl_frame_result* out) {
  return guard([&] {
    use_dev(h);
    if (!odo || !out) throw std::invalid_argument("smcl_step: null odometry or result");
    h->step_slot(slot, odo, out);
  });
}

int smcl_scan_prepare(smcl_engine* h, int slot, const double* points, int64_t n) {
  return guard([&] {
    use_dev(h);
    h->wait_prep_all();
    h->prepare_slot(slot, points, n, h->st);
    h->sync();
  });
}

int smcl_scan_prepare_async(smcl_engine* h, int slot, const double* points, int64_t n) {
  return guard([&] {
    use_dev(h);
    h->prepare_async(slot, points, n);
  });
}

int smcl_scan_get(smcl_engine* h, int slot, double* mu_out, double* sigma_out, int64_t* n_out) {
  return guard([&] {
    use_dev(h);
    h->wait_slot(slot);
    if (!n_out) throw std::invalid_argument("smcl_scan_get: null count");
    auto& sl = h->slot_at(slot);
    if (!sl.valid) throw std::invalid_argument("smcl_scan_get: empty slot");
    *n_out = sl.full.n;
    if (sl.full.n > 0 && mu_out) sl.full.mu.download(mu_out, static_cast<size_t>(sl.full.n) * 3, h->st);
    if (sl.full.n > 0 && sigma_out) sl.full.sigma.download(sigma_out, static_cast<size_t>(sl.full.n) * 9, h->st);
    h->sync();
  });
}

int smcl_step_points(smcl_engine* h, const double* points, int64_t n, const smcl_odom* odo, smcl_frame_result* out) {
  return guard([&] {
    use_dev(h);
    if (!odo || !out) throw std::invalid_argument("smcl_step: null odometry or result");
    h->step_points(points, n, odo, out);
  });
}

int smcl_timer_start(smcl_engine* h) {
  return guard([&] {
    use_dev(h);
    if (!h->timer[0]) CK(cudaEventCreate(&h->timer[0]));
    if (!h->timer[1]) CK(cudaEventCreate(&h->timer[1]));
    CK(cudaEventRecord(h->timer[0], h->st));
  });
}

int smcl_timer_stop(smcl_engine* h, double* ms) {
  return guard([&] {
    use_dev(h);
    CK(cudaEventRecord(h->timer[1], h->st));
    CK(cudaEventSynchronize(h->timer[1]));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, h->timer[0], h->timer[1]));
    *ms = f;
  });
}

int smcl_last_step_counts(smcl_engine* h, smcl_step_profile* out) {
  return guard([&] {
    if (!h) throw std::invalid_argument("null engine handle");
    *out = h->prof;  // stage times not read: only the fields the step itself filled
    out->hash_guard_flagged = static_cast<int64_t>(h->guard_flagged_total);
    out->hash_guard_replays = static_cast<int64_t>(h->guard_replays);
  });
}

int smcl_last_step_profile(smcl_engine* h, smcl_step_profile* out) {
  return guard([&] {
    if (!h) throw std::invalid_argument("null engine handle");
    h->fill_prof_times();
    *out = h->prof;
    // engine-lifetime totals, current also after stage-API passes
    out->hash_guard_flagged = static_cast<int64_t>(h->guard_flagged_total);
    out->hash_guard_replays = static_cast<int64_t>(h->guard_replays);
  });
}

int64_t smcl_frame_index(const smcl_engine* h) { return h ? h->frame : -1; }
int64_t smcl_num_particles(const smcl_engine* h) { return h ? h->n_total : -1; }

int smcl_get_particles(smcl_engine* h, smcl_particles_view* v) {
  return guard([&] {
    use_dev(h);
    const size_t n = static_cast<size_t>(h->n_local), k = static_cast<size_t>(h->k);
    if (v->n != h->n_local || v->k != h->k) throw std::invalid_argument("get_particles: view shape mismatch");
    std::vector<Pose> ps(n);
    h->poses.download(ps.data(), n, h->st);
    h->log_post.download(v->log_post, n, h->st);
    h->id.download(v->id, n, h->st);
    h->idx.download(v->idx, n * k, h->st);
    h->kval.download(v->kval, n * k, h->st);
    h->count.download(v->count, n, h->st);
    h->sync();
    for (size_t i = 0; i < n; ++i) store_pose(ps[i], v->poses + 12 * i);
  });
}

int smcl_set_particles(smcl_engine* h, const smcl_particles_view* v) {
  return guard([&] {
    use_dev(h);
    if (v->n < 0 || v->k < 1 || v->k > kMaxK) throw std::invalid_argument("set_particles: bad shape");
    h->set_shape(v->n * h->world);  // a sharded engine receives its own shard
    h->alloc_particles(v->n, v->k);
    h->cfg.k_neighbors = v->k;
    const size_t n = static_cast<size_t>(v->n), k = static_cast<size_t>(v->k);
    std::vector<Pose> ps(n);
    for (size_t i = 0; i < n; ++i) ps[i] = load_pose(v->poses + 12 * i);
    h->poses.upload(ps.data(), n, h->st);
    h->poses_changed();
    h->log_post.upload(v->log_post, n, h->st);
    h->id.upload(v->id, n, h->st);
    h->idx.upload(v->idx, n * k, h->st);
    h->kval.upload(v->kval, n * k, h->st);
    h->count.upload(v->count, n, h->st);
    h->sync();
  });
}

int smcl_get_nnf(smcl_engine* h, int32_t dims[3], double origin[3], double* resolution, int32_t* cells) {
  return guard([&] {
    if (!h || !h->has_map) throw std::invalid_argument("engine has no map");
    for (int a = 0; a < 3; ++a) {
      dims[a] = h->geom.dims[a];
      origin[a] = h->geom.origin[a];
    }
    if (resolution) *resolution = h->geom.res;
    if (cells) {
      if (h->h_cells.size() != static_cast<size_t>(h->n_cells)) {
        h->h_cells.resize(static_cast<size_t>(h->n_cells));
        h->cells.download(h->h_cells.data(), h->h_cells.size(), h->st);
        h->sync();
      }
      std::memcpy(cells, h->h_cells.data(), h->h_cells.size() * sizeof(int32_t));
    }
  });
}

int smcl_predict(smcl_engine* h, const double delta[12], const double cov[36], uint64_t frame_seed) {
  return guard([&] {
    use_dev(h);
    h->predict(delta, cov, frame_seed);
    h->sync();
  });
}

int smcl_update_neighbors(smcl_engine* h, uint64_t pass_seed, const double bounds[6], smcl_neighbor_stats* stats) {
  return guard([&] {
    use_dev(h);
    h->update_neighbors(pass_seed, bounds, stats);
    h->join_aux();
    h->sync();
    h->finish_nb_stats();
  });
}

int smcl_evaluate_all(smcl_engine* h, const smcl_cloud* scan, double* step_out, double* ll_out, int32_t* nm_out,
                      double* H_out, double* b_out) {
  return guard([&] {
    use_dev(h);
    if (!scan || scan->n == 0) throw std::invalid_argument("gicp::evaluate: empty scan");
    h->upload_scan(h->scan_tmp, scan->mu, scan->sigma, static_cast<int>(scan->n), h->st);
    h->run_likelihood(true, h->scan_tmp);
    const size_t n = static_cast<size_t>(h->n_local);
    if (step_out) h->steps.download(step_out, n * 6, h->st);
    if (ll_out) h->ll.download(ll_out, n, h->st);
    if (nm_out) h->nm.download(nm_out, n, h->st);
    if (H_out || b_out) {
      std::vector<double> sys(n * kSysStride);
      if (h->fast_used) {  // widen the fp32 record (lower triangle of H, b), mirror H
        std::vector<float> f(n * kSysF);
        h->sysf.download(f.data(), f.size(), h->st);
        h->sync();
        constexpr int off[27] = SMCL_FAST_SYS_OFF;
        for (size_t i = 0; i < n; ++i) {
          double* r = &sys[i * kSysStride];
          for (int q = 0; q < kSysStride; ++q) r[q] = 0.0;
          for (int q = 0; q < 27; ++q) r[off[q]] = static_cast<double>(f[i * kSysF + q]);
          for (int a = 0; a < 6; ++a)
            for (int c = a + 1; c < 6; ++c) r[a * 6 + c] = r[c * 6 + a];
        }
      } else {
        h->sys.download(sys.data(), sys.size(), h->st);
        h->sync();
      }
      for (size_t i = 0; i < n; ++i) {
        if (H_out) std::memcpy(H_out + 36 * i, &sys[i * kSysStride], 36 * sizeof(double));
        if (b_out) std::memcpy(b_out + 6 * i, &sys[i * kSysStride + 36], 6 * sizeof(double));
      }
    }
    h->sync();
  });
}

int smcl_evaluate_likelihoods(smcl_engine* h, const smcl_cloud* scan, double* ll_out, int32_t* nm_out) {
  return guard([&] {
    use_dev(h);
    if (!scan || scan->n == 0) throw std::invalid_argument("gicp::evaluate: empty scan");
    h->upload_scan(h->scan_tmp, scan->mu, scan->sigma, static_cast<int>(scan->n), h->st);
    h->run_likelihood(false, h->scan_tmp);
    const size_t n = static_cast<size_t>(h->n_local);
    if (ll_out) h->ll.download(ll_out, n, h->st);
    if (nm_out) h->nm.download(nm_out, n, h->st);
    h->sync();
  });
}

int smcl_compute_phis(smcl_engine* h, const double* steps, double* phi_out) {
  return guard([&] {
    use_dev(h);
    const size_t n = static_cast<size_t>(h->n_local);
    if (steps) {
      h->steps.upload(steps, n * 6, h->st);
      h->steps_valid = true;
    }
    if (!h->steps_valid) throw std::logic_error("compute_phis: no Gauss-Newton steps on the device");
    h->svgd(false);
    if (phi_out) h->phis.download(phi_out, n * 6, h->st);
    h->sync();
  });
}

int smcl_apply_updates(smcl_engine* h, const double* phis) {
  return guard([&] {
    use_dev(h);
    const size_t n = static_cast<size_t>(h->n_local);
    if (phis) {
      h->phis.upload(phis, n * 6, h->st);
      h->phis_valid = true;
    }
    if (!h->phis_valid) throw std::logic_error("apply_updates: one phi per particle required");
    launch_apply(h->poses.p, h->phis.p, h->n_local, h->st);
    h->poses_changed();
    CK(cudaGetLastError());
    h->sync();
  });
}

int smcl_bayes_update(smcl_engine* h, const double* ll, const int32_t* nm, double beta, double floor_v,
                      int32_t* rejected) {
  return guard([&] {
    use_dev(h);
    const size_t n = static_cast<size_t>(h->n_local);
    if ((ll == nullptr) != (nm == nullptr)) throw std::invalid_argument("bayes_update: size mismatch");
    if (ll) {
      h->ll.upload(ll, n, h->st);
      h->nm.upload(nm, n, h->st);
      h->ll_valid = true;
    }
    if (!h->ll_valid) throw std::logic_error("bayes_update: no likelihoods on the device");
    const bool rej = h->bayes(beta, floor_v);
    if (rejected) *rejected = rej ? 1 : 0;
    h->sync();
  });
}

int smcl_normalize_log_post(smcl_engine* h, double floor_v) {
  return guard([&] {
    use_dev(h);
    h->normalize(floor_v);
    h->sync();
  });
}

int smcl_smooth(smcl_engine* h, int32_t iters, double floor_v) {
  return guard([&] {
    use_dev(h);
    h->smooth(iters, floor_v);
    h->sync();
  });
}

int smcl_representative(smcl_engine* h, int64_t* index, double pose[12], double* log_post) {
  return guard([&] {
    use_dev(h);
    h->representative(index, pose, log_post);
  });
}

// ---------------------------------------------------------------- batch math
int smcl_se3_exp_batch(const double* xi, int64_t n, double* poses_out) {
  return guard([&] {
    DBuf<double> dx;
    DBuf<Pose> dp;
    dx.upload(xi, static_cast<size_t>(n) * 6, nullptr);
    dp.ensure(static_cast<size_t>(n));
    launch_exp_batch(dx.p, n, dp.p, nullptr);
    CK(cudaGetLastError());
    std::vector<Pose> h(static_cast<size_t>(n));
    dp.download(h.data(), h.size(), nullptr);
    CK(cudaDeviceSynchronize());
    for (int64_t i = 0; i < n; ++i) store_pose(h[static_cast<size_t>(i)], poses_out + 12 * i);
  });
}

int smcl_se3_log_batch(const double* poses, int64_t n, double* xi_out) {
  return guard([&] {
    std::vector<Pose> h(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) h[static_cast<size_t>(i)] = load_pose(poses + 12 * i);
    DBuf<Pose> dp;
    DBuf<double> dx;
    dp.upload(h.data(), h.size(), nullptr);
    dx.ensure(static_cast<size_t>(n) * 6);
    launch_log_batch(dp.p, n, dx.p, nullptr);
    CK(cudaGetLastError());
    dx.download(xi_out, static_cast<size_t>(n) * 6, nullptr);
    CK(cudaDeviceSynchronize());
  });
}

int smcl_kernel_batch(const double* a, const double* b, int64_t n, double sigma_r, double sigma_t, double* k_out) {
  return guard([&] {
    std::vector<Pose> ha(static_cast<size_t>(n)), hb(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      ha[static_cast<size_t>(i)] = load_pose(a + 12 * i);
      hb[static_cast<size_t>(i)] = load_pose(b + 12 * i);
    }
    DBuf<Pose> da, db;
    DBuf<double> dk;
    da.upload(ha.data(), ha.size(), nullptr);
    db.upload(hb.data(), hb.size(), nullptr);
    dk.ensure(static_cast<size_t>(n));
    launch_kernel_batch(da.p, db.p, n, sigma_r, sigma_t, dk.p, nullptr);
    CK(cudaGetLastError());
    dk.download(k_out, static_cast<size_t>(n), nullptr);
    CK(cudaDeviceSynchronize());
  });
}

int smcl_lsh_hash_batch(const double* poses, int64_t n, const double frame[12], const double noise[6], double alpha,
                        double sigma_r, double sigma_t, uint64_t* out) {
  return guard([&] {
    std::vector<Pose> h(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) h[static_cast<size_t>(i)] = load_pose(poses + 12 * i);
    LshPass lp{};
    lp.frame = load_pose(frame);
    std::memcpy(lp.noise, noise, sizeof(lp.noise));
    lp.alpha = alpha;
    lp.sigma_r = sigma_r;
    lp.sigma_t = sigma_t;
    DBuf<Pose> dp;
    DBuf<uint64_t> dout;
    DBuf<unsigned char> damb;
    dp.upload(h.data(), h.size(), nullptr);
    dout.ensure(static_cast<size_t>(n));
    damb.ensure(static_cast<size_t>(n));
    launch_hash_batch(dp.p, n, lp, dout.p, damb.p, nullptr);
    CK(cudaGetLastError());
    dout.download(out, static_cast<size_t>(n), nullptr);
    std::vector<unsigned char> amb(static_cast<size_t>(n));
    damb.download(amb.data(), amb.size(), nullptr);
    CK(cudaDeviceSynchronize());
    for (int64_t i = 0; i < n; ++i)  // near-integer guard: the reference's (glibc) hash
      if (amb[static_cast<size_t>(i)]) out[i] = lsh_hash_host(h[static_cast<size_t>(i)], lp);
  });
}

int smcl_solve_step_batch(const double* H, const double* b, const double* lambda, int64_t n, double omega_max,
                          double v_max, double* step_out) {
  return guard([&] {
    for (int64_t i = 0; i < n; ++i)
      if (lambda[i] < 0.0) throw std::invalid_argument("solve_step: lambda must be >= 0");
    DBuf<double> dH, db, dl, dout;
    dH.upload(H, static_cast<size_t>(n) * 36, nullptr);
    db.upload(b, static_cast<size_t>(n) * 6, nullptr);
    dl.upload(lambda, static_cast<size_t>(n), nullptr);
    dout.ensure(static_cast<size_t>(n) * 6);
    launch_solve_batch(dH.p, db.p, dl.p, n, omega_max, v_max, dout.p, nullptr);
    CK(cudaGetLastError());
    dout.download(step_out, static_cast<size_t>(n) * 6, nullptr);
    CK(cudaDeviceSynchronize());
  });
}

}  // extern "C"
