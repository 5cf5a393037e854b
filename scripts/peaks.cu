// peaks.cu -- measured B200 ceilings for the resources the section kernels
// actually use (the chi state lives in shared memory, not HBM):
//
//   smem_ld_gbs      LDS.128, conflict-free, all SMs (bytes read / s)
//   smem_ldst_gbs    LDS.128 + STS.128 pairs (bytes read + written / s)
//   fp64_gflops      DFMA, 8 independent chains per thread (2 flop / DFMA)
//   issue_ginst      warp instructions / s at the issue limit: the best of
//                    FP32 FMA chains and an FMA+LOP3 mix (8 independent
//                    chains per thread; one instruction per SMSP per clock)
//   lop3_ginst, imad_ginst  the integer pipe (half rate on B200)
//
// Each is the best of 5 timed launches (CUDA events) after a warm-up, at full
// occupancy (grid = SMs x resident blocks).  Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/peaks scripts/peaks.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <algorithm>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                        \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

constexpr int kSmemWords = 8192;   // 16-B words; each block uses half (64 KB)

__global__ void __launch_bounds__(1024) smem_ld(int iters, uint32_t *sink) {
  extern __shared__ uint4 buf[];
  const int n = kSmemWords / 2;    // 64 KB per block: two blocks per SM
  for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  uint32_t a = 0, b = 0, c = 0, d = 0;
  int idx = threadIdx.x;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      uint32_t x0, x1, x2, x3;
      const uint32_t addr = (uint32_t)__cvta_generic_to_shared(buf + ((idx + u * 1024) & (n - 1)));
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "r"(addr));
      a ^= x0; b ^= x1; c ^= x2; d ^= x3;
    }
    idx += 32;
  }
  if ((a ^ b ^ c ^ d) == 0x12345678u) sink[0] = a;
}

__global__ void __launch_bounds__(1024) smem_ldst(int iters, uint32_t *sink) {
  extern __shared__ uint4 buf[];
  const int n = kSmemWords / 2;
  for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  int idx = threadIdx.x;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = (idx + u * 1024) & (n - 1);
      const uint32_t addr = (uint32_t)__cvta_generic_to_shared(buf + j);
      uint32_t x0, x1, x2, x3;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "r"(addr));
      x0 ^= 1u;
      asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};"
                   :: "r"(addr), "r"(x0), "r"(x1), "r"(x2), "r"(x3) : "memory");
    }
    idx += 32;    // conflict-free rows; slot values are irrelevant (bandwidth only)
  }
  __syncthreads();
  if (buf[threadIdx.x].x == 0x12345678u) sink[0] = 1;
}

__global__ void __launch_bounds__(512) fp64_fma(int iters, double *sink) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = 1.0 + 1e-9 * (threadIdx.x + c);
  const double m = 0.999999999, k = 1e-9;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], m, k);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 12345.0) sink[0] = s;
}

__global__ void __launch_bounds__(1024) lop3_issue(int iters, uint32_t *sink) {
  uint32_t x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * (c + 1);
  const uint32_t y = blockIdx.x | 0x55u, z = 0x0f0f0f0fu;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y), "r"(z));
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s ^= x[c];
  if (s == 0x12345678u) sink[0] = s;
}

__global__ void __launch_bounds__(1024) imad_issue(int iters, uint32_t *sink) {
  uint32_t x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * (c + 1);
  const uint32_t y = blockIdx.x | 3u, z = 0x9e3779b9u;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s ^= x[c];
  if (s == 0x12345678u) sink[0] = s;
}

// FP32 FMA chains: full-rate on Blackwell (128 lanes/clk/SM = 4 warp
// instructions / clk / SM), so this one is bound by instruction issue
__global__ void __launch_bounds__(1024) ffma_issue(int iters, float *sink) {
  float x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = 1.0f + 1e-6f * (threadIdx.x + c);
  const float m = 0.9999999f, k = 1e-7f;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(m), "f"(k));
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 12345.0f) sink[0] = s;
}

// alternating FP32 FMA and LOP3 chains (two pipes): issue-bound mix
__global__ void __launch_bounds__(1024) mix_issue(int iters, float *sink) {
  float x[4];
  uint32_t y[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) { x[c] = 1.0f + 1e-6f * (threadIdx.x + c); y[c] = threadIdx.x * (c + 1); }
  const float m = 0.9999999f, k = 1e-7f;
  const uint32_t a = blockIdx.x | 0x55u, b = 0x0f0f0f0fu;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(m), "f"(k));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[c]) : "r"(a), "r"(b));
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) s += x[c] + (float)(y[c] & 1u);
  if (s == 12345.0f) sink[0] = s;
}

template <typename F>
static float best_ms(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  uint32_t *sink;
  double *dsink;
  CK(cudaMalloc(&sink, 64));
  CK(cudaMalloc(&dsink, 64));
  const size_t smem = (size_t)kSmemWords / 2 * 16;   // 64 KB
  CK(cudaFuncSetAttribute(smem_ld, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(smem_ldst, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, smem_ld, 1024, smem));
  const int it_s = 4096;
  const float t_ld = best_ms([&] { smem_ld<<<sms * per, 1024, smem>>>(it_s, sink); });
  CK(cudaGetLastError());
  const double b_ld = (double)sms * per * 1024 * it_s * 8 * 16;
  int per2 = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, smem_ldst, 1024, smem));
  const float t_ls = best_ms([&] { smem_ldst<<<sms * per2, 1024, smem>>>(it_s, sink); });
  CK(cudaGetLastError());
  const double b_ls = (double)sms * per2 * 1024 * it_s * 4 * 32;
  int per3 = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per3, fp64_fma, 512, 0));
  const int it_f = 8192;
  const float t_f = best_ms([&] { fp64_fma<<<sms * per3, 512>>>(it_f, dsink); });
  CK(cudaGetLastError());
  const double fl = (double)sms * per3 * 512 * it_f * 8 * 2;
  int per4 = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per4, lop3_issue, 1024, 0));
  const int it_i = 8192;
  const float t_i = best_ms([&] { lop3_issue<<<sms * per4, 1024>>>(it_i, sink); });
  CK(cudaGetLastError());
  const double wi = (double)sms * per4 * 32 * it_i * 8;
  int per5 = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per5, imad_issue, 1024, 0));
  const float t_m = best_ms([&] { imad_issue<<<sms * per5, 1024>>>(it_i, sink); });
  CK(cudaGetLastError());
  const double wm = (double)sms * per5 * 32 * it_i * 8;
  float *fsink;
  CK(cudaMalloc(&fsink, 64));
  int per6 = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per6, ffma_issue, 1024, 0));
  const float t_ff = best_ms([&] { ffma_issue<<<sms * per6, 1024>>>(it_i, fsink); });
  CK(cudaGetLastError());
  const double wf = (double)sms * per6 * 32 * it_i * 8;
  int per7 = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per7, mix_issue, 1024, 0));
  const float t_mx = best_ms([&] { mix_issue<<<sms * per7, 1024>>>(it_i, fsink); });
  CK(cudaGetLastError());
  const double wx = (double)sms * per7 * 32 * it_i * 8;
  const double issue = std::max(wf / t_ff, wx / t_mx) / 1e6;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_max_mhz\": %.0f, "
         "\"smem_ld_gbs\": %.1f, \"smem_ldst_gbs\": %.1f, \"fp64_gflops\": %.1f, "
         "\"issue_ginst\": %.1f, \"lop3_ginst\": %.1f, \"imad_ginst\": %.1f, "
         "\"ffma_ginst\": %.1f, \"mix_ginst\": %.1f, "
         "\"per_sm_per_clk\": {\"smem_ld_bytes\": %.1f, \"smem_ldst_bytes\": %.1f, "
         "\"dfma_warp_inst\": %.3f, \"lop3_warp_inst\": %.3f, \"imad_warp_inst\": %.3f, "
         "\"issue_warp_inst\": %.3f}}\n",
         prop.name, sms, clk_khz / 1e3, b_ld / t_ld / 1e6, b_ls / t_ls / 1e6, fl / t_f / 1e6,
         issue, wi / t_i / 1e6, wm / t_m / 1e6, wf / t_ff / 1e6, wx / t_mx / 1e6,
         b_ld / (t_ld * 1e-3) / sms / (clk_khz * 1e3), b_ls / (t_ls * 1e-3) / sms / (clk_khz * 1e3),
         fl / 2 / (t_f * 1e-3) / sms / (clk_khz * 1e3) / 32.0,
         wi / (t_i * 1e-3) / sms / (clk_khz * 1e3), wm / (t_m * 1e-3) / sms / (clk_khz * 1e3),
         issue * 1e9 / sms / (clk_khz * 1e3));
  return 0;
}
