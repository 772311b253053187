// Roofline denominator for the MUFU-bound KDE kernels: measured
// MUFU.EX2 throughput of this device at its current clocks (MEASURED_PEAKS
// only carries HBM and bf16 tensor peaks). A grid of 148 x k CTAs, each
// warp issuing long chains of independent ex2.approx.ftz.f32.
#include <cuda_runtime.h>

#include "../../include/fsgg_probe.h"
#include "common.cuh"

namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) ex2_probe_kernel(float* out, int iters, float seed) {
  float v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = seed * (threadIdx.x + c) * 1e-9f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = fsgg::ex2_approx(-v[c]);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  if (s == 12345.f) out[blockIdx.x] = s;  // keep the chains alive
}

}  // namespace

extern "C" int fsgg_probe_ex2_throughput(int device, double* ex2_per_second,
                                         double* sm_clock_mhz) {
  try {
    FSGG_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    FSGG_CUDA(cudaGetDeviceProperties(&prop, device));
    float* out = nullptr;
    FSGG_CUDA(cudaMalloc(&out, 4096 * sizeof(float)));
    const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
    cudaEvent_t a, b;
    FSGG_CUDA(cudaEventCreate(&a));
    FSGG_CUDA(cudaEventCreate(&b));
    ex2_probe_kernel<<<blocks, threads>>>(out, 64, 1.f);  // warm-up
    FSGG_CUDA(cudaEventRecord(a));
    for (int r = 0; r < 5; ++r) ex2_probe_kernel<<<blocks, threads>>>(out, iters, 1.f);
    FSGG_CUDA(cudaEventRecord(b));
    FSGG_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    FSGG_CUDA(cudaEventElapsedTime(&ms, a, b));
    const double ops = 5.0 * blocks * threads * double(iters) * kChains;
    if (ex2_per_second) *ex2_per_second = ops / (ms * 1e-3);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, device);
    if (sm_clock_mhz) *sm_clock_mhz = clk_khz / 1000.0;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    return 0;
  } catch (const fsgg::Error& e) {
    return e.code;
  }
}
