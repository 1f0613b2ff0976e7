// K5: measured FP32 and MUFU/XU pipe peaks on this
// B200, the roofline denominators MEASURED_PEAKS.json does not carry (it has
// HBM copy bandwidth and cuBLAS bf16 only).  Standalone: nvcc -o k5 this.cu,
// run on the GPU box, prints one JSON object (tools/k5_peaks.sh writes it to
// profiles/peaks_fp32_xu.json, which bench.py reads).
//
// Every kernel runs NC independent dependency chains per thread (enough ILP
// to hide the 4-cycle FMA latency and the MUFU latency at full occupancy) in
// a grid of 148 SMs x CTAS_PER_SM x 256 threads, timed with CUDA events over
// REP launches after a warm-up.  The chains' results are stored behind a
// runtime-false predicate so the compiler keeps every operation.
//   ffma_reg   a = fma(a, b, c), b, c loop-invariant registers (3-register form)
//   ffma_imm   a = fma(a, 1.0001, 0.5) (immediate form)
//   ffma_mix   the two alternating (what compiled code mixes)
//   ex2        a = ex2.approx(a') with a' = a * k (one FMUL per MUFU, not counted)
//   lg2        a = lg2.approx(|a| + 1)
//   rcp        a = rcp.approx(a + 1)
//   rsqrt      a = rsqrt.approx(|a| + 1)
//   ex2_lg2    alternating ex2(lg2(x)) (the SQ evaluation's mix)
// FLOPs: an FFMA counts 2.  MUFU ops count 1 each.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)

constexpr int NC = 8;          // independent chains per thread
constexpr int ITERS = 4096;    // loop trips per launch
constexpr int UNROLL = 8;

__device__ __forceinline__ float ex2a(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float lg2a(float x) { float y; asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rcpa(float x) { float y; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rsqa(float x) { float y; asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

template <int MODE>
__global__ void __launch_bounds__(256) k_chain(float* out, float b, float c, int flag) {
  float a[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) a[i] = (threadIdx.x + i) * 1e-3f + 0.5f;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        if constexpr (MODE == 0) a[i] = fmaf(a[i], b, c);
        if constexpr (MODE == 1) a[i] = fmaf(a[i], 1.0001f, 0.5f);
        if constexpr (MODE == 2) a[i] = (u & 1) ? fmaf(a[i], b, c) : fmaf(a[i], 0.9999f, -0.25f);
        if constexpr (MODE == 3) a[i] = ex2a(a[i] * -0.5f);
        if constexpr (MODE == 4) a[i] = lg2a(fabsf(a[i]) + 1.f);
        if constexpr (MODE == 5) a[i] = rcpa(a[i] + 1.f);
        if constexpr (MODE == 6) a[i] = rsqa(fabsf(a[i]) + 1.f);
        if constexpr (MODE == 7) a[i] = (u & 1) ? ex2a(a[i] * -0.5f) : lg2a(fabsf(a[i]) + 1.f);
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NC; ++i) s += a[i];
  if (flag) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

struct Res { const char* name; double ops_per_s; double ops_per_clk_sm; double ms; };

template <int MODE>
Res run(const char* name, int sms, int clk_khz, float* out) {
  const int cps = 8, T = 256;   // 2048 threads per SM (full occupancy at <= 32 regs)
  dim3 grid(sms * cps), block(T);
  for (int w = 0; w < 3; ++w) k_chain<MODE><<<grid, block>>>(out, 1.0001f, 0.5f, 0);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int REP = 10;
  CK(cudaEventRecord(e0));
  for (int r = 0; r < REP; ++r) k_chain<MODE><<<grid, block>>>(out, 1.0001f, 0.5f, 0);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double ops = (double)REP * grid.x * T * (double)ITERS * UNROLL * NC * (MODE <= 2 ? 2.0 : 1.0);
  const double rate = ops / (ms * 1e-3);
  return Res{name, rate, rate / (sms * (clk_khz * 1e3)), ms / REP};
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));   // kHz (max)
  float* out = nullptr;
  CK(cudaMalloc(&out, (size_t)sms * 8 * 256 * sizeof(float)));
  std::vector<Res> rs;
  for (int round = 0; round < 2; ++round) {   // best of two rounds
    std::vector<Res> r = {run<0>("ffma_reg", sms, clk, out), run<1>("ffma_imm", sms, clk, out),
                          run<2>("ffma_mix", sms, clk, out), run<3>("ex2", sms, clk, out),
                          run<4>("lg2", sms, clk, out),       run<5>("rcp", sms, clk, out),
                          run<6>("rsqrt", sms, clk, out),     run<7>("ex2_lg2", sms, clk, out)};
    if (rs.empty()) rs = r;
    else
      for (size_t i = 0; i < r.size(); ++i)
        if (r[i].ops_per_s > rs[i].ops_per_s) rs[i] = r[i];
  }
  std::printf("{\n \"sms\": %d,\n \"sm_max_mhz_attr\": %.0f,\n \"kernels\": {\n", sms, clk / 1e3);
  for (size_t i = 0; i < rs.size(); ++i)
    std::printf("  \"%s\": {\"rate\": %.6e, \"unit\": \"%s\", \"per_clk_per_sm_at_max_clock\": %.2f, \"ms\": %.4f}%s\n",
                rs[i].name, rs[i].ops_per_s, i < 3 ? "FLOP/s" : "ops/s", rs[i].ops_per_clk_sm, rs[i].ms,
                i + 1 < rs.size() ? "," : "");
  std::printf(" }\n}\n");
  CK(cudaFree(out));
  return 0;
}
