// fp64 peak microbenchmarks for the roofline denominators of the near-field
// and direct-sum kernels ("fp64 pipe ... measure it").
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_peak tools/fp64_peak.cu
//   ./tools/fp64_peak > profiles/fp64_peak.json
//
// dfma: every thread runs 16 independent DFMA chains (enough ILP to cover the
//       ~9-cycle dependent latency), grid = SMs x 8 CTAs x 256 threads.
// dmma: every warp issues mma.sync m8n8k4 f64 (DMMA.8x8x4, the instruction
//       the near kernel uses) on 8 independent accumulators.
// Each is timed with CUDA events after a warm-up launch; FLOPs = 2 per DFMA,
// 2*8*8*4 = 512 per DMMA.  The clock (nvidia-smi) is read around the run.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int kChains = 16;

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;  // never true; keeps the chains live
}

constexpr int kAcc = 8;

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.5;
  double c[kAcc][2];
#pragma unroll
  for (int i = 0; i < kAcc; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kAcc; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kAcc; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  double* out;
  CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));

  // ---- DFMA
  const int threads = 256, ctas = sms * 8, iters = 20000;
  dfma_kernel<<<ctas, threads>>>(out, 100, 0.999999, 1e-7);
  CK(cudaDeviceSynchronize());
  float best_dfma = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    dfma_kernel<<<ctas, threads>>>(out, iters, 0.999999, 1e-7);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best_dfma) best_dfma = ms;
  }
  double dfma_flops = 2.0 * kChains * (double)iters * threads * ctas;
  double dfma_tf = dfma_flops / (best_dfma * 1e-3) / 1e12;

  // ---- DMMA
  const int dthreads = 128, dctas = sms * 4, diters = 20000;
  dmma_kernel<<<dctas, dthreads>>>(out, 100);
  CK(cudaDeviceSynchronize());
  float best_dmma = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    dmma_kernel<<<dctas, dthreads>>>(out, diters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best_dmma) best_dmma = ms;
  }
  double warps = dctas * (dthreads / 32.0);
  double dmma_flops = 512.0 * kAcc * (double)diters * warps;
  double dmma_tf = dmma_flops / (best_dmma * 1e-3) / 1e12;

  printf("{\"sms\": %d, \"attr_clock_mhz\": %.0f,\n"
         " \"dfma\": {\"tflops\": %.3f, \"ms\": %.3f, \"flops\": %.6e, \"per_sm_per_clk_at_attr_clock\": %.2f,\n"
         "          \"how\": \"%d CTAs x %d threads, %d independent DFMA chains x %d iters, best of 5\"},\n"
         " \"dmma\": {\"tflops\": %.3f, \"ms\": %.3f, \"flops\": %.6e, \"per_sm_per_clk_at_attr_clock\": %.2f,\n"
         "          \"how\": \"%d CTAs x %d threads, mma.sync m8n8k4 f64 on %d accumulators x %d iters, best of 5\"}}\n",
         sms, clk_khz / 1e3,
         dfma_tf, best_dfma, dfma_flops, dfma_flops / (best_dfma * 1e-3) / sms / (clk_khz * 1e3),
         ctas, threads, kChains, iters,
         dmma_tf, best_dmma, dmma_flops, dmma_flops / (best_dmma * 1e-3) / sms / (clk_khz * 1e3),
         dctas, dthreads, kAcc, diters);
  return 0;
}
