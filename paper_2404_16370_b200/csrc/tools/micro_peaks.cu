// Microbenchmarks for the roofline denominators MEASURED_PEAKS.json does not
// carry: FP32 and FP64 FMA throughput, and the random 32-byte
// record gather bandwidth of the likelihood kernels, from an L2-resident table
// (the corridor map's 49 MB of NNF records) and from an HBM-sized table (the
// outdoor map's 7 GB), for three ways of issuing the gather (two 16-byte
// loads, one 256-bit load, two 16-byte cp.async). Prints one JSON object.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_peaks micro_peaks.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));             \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

template <typename T, int ILP>
__global__ void k_fma(T* out, int iters, T a, T b) {
  T v[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) v[j] = static_cast<T>(threadIdx.x + j);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < ILP; ++j) v[j] = fma(v[j], a, b);
  T s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += v[j];
  if (s == static_cast<T>(-1.2345)) out[0] = s;
}

// Each thread gathers `per_thread` random 32-byte records (two 16-byte loads,
// the K1/K2 record layout) from a table of n_rec records.
__global__ void k_gather(const float4* __restrict__ rec, uint64_t n_rec, int per_thread, uint64_t seed,
                         float* __restrict__ out) {
  uint64_t s = seed ^ (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull;
  float acc = 0.f;
  for (int i = 0; i < per_thread; i += 8) {
    float4 r[16];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s ^= s << 13;
      s ^= s >> 7;
      s ^= s << 17;
      const uint64_t c = s % n_rec;
      r[2 * u] = __ldg(rec + 2 * c);
      r[2 * u + 1] = __ldg(rec + 2 * c + 1);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += r[u].x + r[u].w;
  }
  if (acc == -1.2345f) out[0] = acc;
}

// Same access, one 256-bit load per record (sm_100 LDG.256).
__global__ void k_gather256(const double* __restrict__ rec, uint64_t n_rec, int per_thread, uint64_t seed,
                            float* __restrict__ out) {
  uint64_t s = seed ^ (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull;
  double acc = 0.0;
  for (int i = 0; i < per_thread; i += 8) {
    double r[8][4];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s ^= s << 13;
      s ^= s >> 7;
      s ^= s << 17;
      const uint64_t c = s % n_rec;
      asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                   : "=d"(r[u][0]), "=d"(r[u][1]), "=d"(r[u][2]), "=d"(r[u][3])
                   : "l"(rec + 4 * c));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += r[u][0] + r[u][3];
  }
  if (acc == -1.2345) out[0] = static_cast<float>(acc);
}

// Same access through cp.async (two 16-byte async copies per record into a
// per-thread shared-memory stage), as the likelihood kernels issue it.
__global__ void k_gather_cpasync(const float4* __restrict__ rec, uint64_t n_rec, int per_thread, uint64_t seed,
                                 float* __restrict__ out) {
  __shared__ float4 stage[128 * 16];  // launched with 128 threads
  uint64_t s = seed ^ (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull;
  float acc = 0.f;
  for (int i = 0; i < per_thread; i += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s ^= s << 13;
      s ^= s >> 7;
      s ^= s << 17;
      const uint64_t c = s % n_rec;
      const unsigned d0 = static_cast<unsigned>(__cvta_generic_to_shared(&stage[(2 * u) * 128 + threadIdx.x]));
      const unsigned d1 = static_cast<unsigned>(__cvta_generic_to_shared(&stage[(2 * u + 1) * 128 + threadIdx.x]));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d0), "l"(rec + 2 * c) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d1), "l"(rec + 2 * c + 1) : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += stage[(2 * u) * 128 + threadIdx.x].x + stage[(2 * u + 1) * 128 + threadIdx.x].w;
  }
  if (acc == -1.2345f) out[0] = acc;
}

// Same access through the bulk-copy (TMA) engine: one 32-byte
// cp.async.bulk per record into shared memory, completion counted by a
// per-thread mbarrier (expect-tx of the 8 records' bytes).
__global__ void k_gather_bulk(const float4* __restrict__ rec, uint64_t n_rec, int per_thread, uint64_t seed,
                              float* __restrict__ out) {
  __shared__ __align__(16) float4 stage[128 * 16];  // launched with 128 threads
  __shared__ __align__(8) unsigned long long bar[128];
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[threadIdx.x]));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t s = seed ^ (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull;
  float acc = 0.f;
  unsigned phase = 0;
  for (int i = 0; i < per_thread; i += 8) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(8 * 32) : "memory");
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s ^= s << 13;
      s ^= s >> 7;
      s ^= s << 17;
      const uint64_t c = s % n_rec;
      const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(&stage[(threadIdx.x * 8 + u) * 2]));
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 32, [%2];" ::"r"(d),
                   "l"(rec + 2 * c), "r"(b)
                   : "memory");
    }
    asm volatile(
        "{\n .reg .pred P1;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra WAIT_%=;\n}" ::"r"(b),
        "r"(phase)
        : "memory");
    phase ^= 1u;
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += stage[(threadIdx.x * 8 + u) * 2].x;
  }
  if (acc == -1.2345f) out[0] = acc;
}

int main() {
  int dev = 0, n_sm = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float* out;
  CK(cudaMalloc(&out, 16));
  auto time_ms = [&](auto launch) -> float {
    launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5.f;
  };
  const int blocks = n_sm * 8, threads = 256, iters = 4096;
  const float ms32 = time_ms([&] { k_fma<float, 8><<<blocks, threads>>>(out, iters, 1.0000001f, 1e-7f); });
  const double f32 = 2.0 * blocks * threads * 8.0 * iters / (ms32 * 1e-3) / 1e12;
  const float ms64 = time_ms([&] {
    k_fma<double, 8><<<blocks, threads>>>(reinterpret_cast<double*>(out), iters / 4, 1.0000001, 1e-7);
  });
  const double f64 = 2.0 * blocks * threads * 8.0 * (iters / 4) / (ms64 * 1e-3) / 1e12;
  std::printf("{\"fp32_fma_tflops\": %.2f, \"fp64_fma_tflops\": %.2f", f32, f64);
  const uint64_t tables[2] = {uint64_t(49) << 20, uint64_t(7) << 30};  // bytes
  const char* names[2] = {"l2_resident_49MB", "hbm_7GB"};
  for (int t = 0; t < 2; ++t) {
    const uint64_t n_rec = tables[t] / 32;
    float4* rec = nullptr;
    if (cudaMalloc(&rec, n_rec * 32) != cudaSuccess) {
      std::printf(", \"gather_%s_gbs\": null", names[t]);
      cudaGetLastError();
      continue;
    }
    CK(cudaMemset(rec, 0, n_rec * 32));
    const int gblocks = n_sm * 8, gthreads = 256, per = 256;
    const float ms = time_ms([&] { k_gather<<<gblocks, gthreads>>>(rec, n_rec, per, 12345ull, out); });
    const double gbs = 32.0 * gblocks * gthreads * per / (ms * 1e-3) / 1e9;
    std::printf(", \"gather_%s_gbs\": %.1f", names[t], gbs);
    const float ms2 = time_ms([&] {
      k_gather256<<<gblocks, gthreads>>>(reinterpret_cast<const double*>(rec), n_rec, per, 12345ull, out);
    });
    std::printf(", \"gather256_%s_gbs\": %.1f", names[t], 32.0 * gblocks * gthreads * per / (ms2 * 1e-3) / 1e9);
    const float ms3 = time_ms([&] { k_gather_cpasync<<<2 * gblocks, 128>>>(rec, n_rec, per, 12345ull, out); });
    std::printf(", \"gather_cpasync_%s_gbs\": %.1f", names[t], 32.0 * gblocks * gthreads * per / (ms3 * 1e-3) / 1e9);
    const float ms4 = time_ms([&] { k_gather_bulk<<<2 * gblocks, 128>>>(rec, n_rec, per, 12345ull, out); });
    std::printf(", \"gather_bulk_%s_gbs\": %.1f", names[t], 32.0 * gblocks * gthreads * per / (ms4 * 1e-3) / 1e9);
    CK(cudaFree(rec));
  }
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  std::printf(", \"sm_count\": %d, \"note\": \"random 32-byte record gathers, 8 records in flight per thread, %d "
              "CTAs x 256 threads: gather_ = two 16-B __ldg per record, gather256_ = one 256-bit ld.global.nc.v4.f64, "
              "gather_cpasync_ = two 16-B cp.async.cg into shared memory, gather_bulk_ = one 32-B "
              "cp.async.bulk (TMA) per record\"}\n",
              n_sm, n_sm * 8);
  return 0;
}
