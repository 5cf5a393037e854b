// peaks.cu -- measured B200 ceilings for the resources the section kernels
// actually use (the chi state lives in shared memory, not HBM):
//
//   smem_ld_gbs      LDS.128, conflict-free, all SMs (bytes read / s)
//   smem_ldst_gbs    LDS.128 + STS.128 pairs (bytes read + written / s)
//   fp64_gflops      DFMA, 8 independent chains per thread (2 flop / DFMA)
//   ffma_ginst, mix_ginst  warp instructions / s of FP32 FMA chains and an
//                    FMA+LOP3 mix (8 independent chains per thread): the
//                    issue limit, one instruction per SMSP per clock
//   lop3_ginst, imad_ginst  the integer pipe (half rate on B200)
//   l2_rw_gbs        L2-resident float4 read + write streams, one block per SM
//
// Each is the best of 5 timed launches (CUDA events) after a warm-up, at full
// occupancy (grid = SMs x resident blocks).  Heavy FP loads can pull the SM
// clock below its maximum, so every kernel also reports the clock it ran at
// (clock64 / globaltimer per block) and its rate per SM per clock; the
// ceilings a kernel running at clock f is held to are per_sm_per_clk x SMs x
// f (issue_ipc_per_sm, ..._at_max_clock).  Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/peaks scripts/peaks.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <algorithm>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                        \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

// per-block elapsed SM cycles and ns (thread 0, between two barriers): the
// clock the SMs actually ran at during the measurement (heavy FP loads can
// drop below the maximum), so rates are also reported per SM per clock
struct Tm { unsigned long long c0, t0; };
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ Tm tstart() {
  __syncthreads();
  return Tm{(unsigned long long)clock64(), gtimer()};
}
__device__ __forceinline__ void tstop(Tm t, unsigned long long *cyc, unsigned long long *ns) {
  __syncthreads();
  if (threadIdx.x == 0) {
    cyc[blockIdx.x] = (unsigned long long)clock64() - t.c0;
    ns[blockIdx.x] = gtimer() - t.t0;
  }
}

constexpr int kSmemWords = 8192;   // 16-B words; each block uses half (64 KB)

__global__ void __launch_bounds__(1024) smem_ld(int iters, uint32_t *sink, unsigned long long *cyc, unsigned long long *ns) {
  extern __shared__ uint4 buf[];
  const int n = kSmemWords / 2;    // 64 KB per block: two blocks per SM
  for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = make_uint4(i, i * 3, i * 5, i * 7);
  uint32_t a = 0, b = 0, c = 0, d = 0;
  int idx = threadIdx.x;
  const Tm tm = tstart();
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
  tstop(tm, cyc, ns);
  if ((a ^ b ^ c ^ d) == 0x12345678u) sink[0] = a;
}

__global__ void __launch_bounds__(1024) smem_ldst(int iters, uint32_t *sink, unsigned long long *cyc, unsigned long long *ns) {
  extern __shared__ uint4 buf[];
  const int n = kSmemWords / 2;
  for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = make_uint4(i, i * 3, i * 5, i * 7);
  int idx = threadIdx.x;
  const Tm tm = tstart();
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
  tstop(tm, cyc, ns);
  if (buf[threadIdx.x].x == 0x12345678u) sink[0] = 1;
}

// L2-resident read + write: every block streams its own slice of a buffer
// that fits in L2 (the block-per-shot chi lives in such a buffer; DESIGN
// §3), float4 loads 4 deep per thread, then stores; bytes read + written
__global__ void __launch_bounds__(512) l2_rw(int iters, uint4 *buf, size_t slice_u4, uint32_t *sink,
                                             unsigned long long *cyc, unsigned long long *ns) {
  uint4 *mine = buf + (size_t)blockIdx.x * slice_u4;
  const Tm tm = tstart();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (size_t i = threadIdx.x; i + 3 * blockDim.x < slice_u4; i += 4 * blockDim.x) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcg(mine + i + u * blockDim.x);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        v[u].x ^= 1u;
        __stcg(mine + i + u * blockDim.x, v[u]);
      }
    }
  }
  tstop(tm, cyc, ns);
  if (mine[threadIdx.x].y == 0x12345678u) sink[0] = 1;
}

__global__ void __launch_bounds__(512) fp64_fma(int iters, double *sink, unsigned long long *cyc, unsigned long long *ns) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = 1.0 + 1e-9 * (threadIdx.x + c);
  const double m = 0.999999999, k = 1e-9;
const Tm tm = tstart();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], m, k);
  }
  tstop(tm, cyc, ns);
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 12345.0) sink[0] = s;
}

__global__ void __launch_bounds__(1024) lop3_issue(int iters, uint32_t *sink, unsigned long long *cyc, unsigned long long *ns) {
  uint32_t x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * (c + 1);
  const uint32_t y = blockIdx.x | 0x55u, z = 0x0f0f0f0fu;
const Tm tm = tstart();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y), "r"(z));
  }
  tstop(tm, cyc, ns);
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s ^= x[c];
  if (s == 0x12345678u) sink[0] = s;
}

__global__ void __launch_bounds__(1024) imad_issue(int iters, uint32_t *sink, unsigned long long *cyc, unsigned long long *ns) {
  uint32_t x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * (c + 1);
  const uint32_t y = blockIdx.x | 3u, z = 0x9e3779b9u;
const Tm tm = tstart();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
  }
  tstop(tm, cyc, ns);
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s ^= x[c];
  if (s == 0x12345678u) sink[0] = s;
}

constexpr int kIssueUnroll = 16;

// FP32 FMA chains: full-rate on Blackwell (128 lanes/clk/SM = 4 warp
// instructions / clk / SM), so this one is bound by instruction issue
__global__ void __launch_bounds__(1024) ffma_issue(int iters, float *sink, unsigned long long *cyc, unsigned long long *ns) {
  float x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = 1.0f + 1e-6f * (threadIdx.x + c);
  const float m = 0.9999999f, k = 1e-7f;
const Tm tm = tstart();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    // kIssueUnroll x 8 FMAs per trip: the loop's own counter/compare/branch
    // (3 instructions) stay below 3 % of what is issued
#pragma unroll
    for (int u = 0; u < kIssueUnroll; ++u)
#pragma unroll
      for (int c = 0; c < 8; ++c) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(m), "f"(k));
  }
  tstop(tm, cyc, ns);
  float s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 12345.0f) sink[0] = s;
}

// alternating FP32 FMA and LOP3 chains (two pipes): issue-bound mix
__global__ void __launch_bounds__(1024) mix_issue(int iters, float *sink, unsigned long long *cyc, unsigned long long *ns) {
  float x[4];
  uint32_t y[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) { x[c] = 1.0f + 1e-6f * (threadIdx.x + c); y[c] = threadIdx.x * (c + 1); }
  const float m = 0.9999999f, k = 1e-7f;
  const uint32_t a = blockIdx.x | 0x55u, b = 0x0f0f0f0fu;
const Tm tm = tstart();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < kIssueUnroll; ++u)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(m), "f"(k));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[c]) : "r"(a), "r"(b));
      }
  }
  tstop(tm, cyc, ns);
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

struct Res {
  double rate;       // units / s (wall, CUDA events)
  double mhz;        // SM clock during the last launch (clock64 / globaltimer)
  double per_sm_clk; // units per SM per clock at that clock
};

static unsigned long long *g_cyc, *g_ns;
static int g_sms;

// units = total work units of one launch of `blocks` blocks
template <typename F>
static Res measure(F launch, double units, int blocks) {
  const float ms = best_ms(launch);
  std::vector<unsigned long long> c(blocks), n(blocks);
  cudaMemcpy(c.data(), g_cyc, blocks * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(n.data(), g_ns, blocks * 8, cudaMemcpyDeviceToHost);
  double sc = 0, sn = 0;
  for (int i = 0; i < blocks; ++i) { sc += (double)c[i]; sn += (double)n[i]; }
  Res r;
  r.rate = units / (ms * 1e-3);
  r.mhz = sn > 0 ? 1e3 * sc / sn : 0.0;
  r.per_sm_clk = r.mhz > 0 ? r.rate / g_sms / (r.mhz * 1e6) : 0.0;
  return r;
}

static void emit(const char *name, Res r, double scale, bool last = false) {
  printf("\"%s\": {\"rate\": %.1f, \"sm_mhz\": %.0f, \"per_sm_per_clk\": %.3f}%s", name,
         r.rate * scale, r.mhz, r.per_sm_clk, last ? "" : ", ");
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  g_sms = sms;
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  uint32_t *sink;
  double *dsink;
  float *fsink;
  CK(cudaMalloc(&sink, 64));
  CK(cudaMalloc(&dsink, 64));
  CK(cudaMalloc(&fsink, 64));
  CK(cudaMalloc(&g_cyc, 1 << 20));
  CK(cudaMalloc(&g_ns, 1 << 20));
  unsigned long long *cy = g_cyc, *ns = g_ns;
  const size_t smem = (size_t)kSmemWords / 2 * 16;   // 64 KB
  CK(cudaFuncSetAttribute(smem_ld, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(smem_ldst, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per = 0;
  const int it_s = 4096, it_f = 8192, it_i = 8192;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, smem_ld, 1024, smem));
  const int b1 = sms * per;
  const Res ld = measure([&] { smem_ld<<<b1, 1024, smem>>>(it_s, sink, cy, ns); },
                         (double)b1 * 1024 * it_s * 8 * 16, b1);
  CK(cudaGetLastError());
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, smem_ldst, 1024, smem));
  const int b2 = sms * per;
  const Res ls = measure([&] { smem_ldst<<<b2, 1024, smem>>>(it_s, sink, cy, ns); },
                         (double)b2 * 1024 * it_s * 4 * 32, b2);
  CK(cudaGetLastError());
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fp64_fma, 512, 0));
  const int b3 = sms * per;
  const Res fp = measure([&] { fp64_fma<<<b3, 512>>>(it_f, dsink, cy, ns); },
                         (double)b3 * 512 * it_f * 8 * 2, b3);
  CK(cudaGetLastError());
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, lop3_issue, 1024, 0));
  const int b4 = sms * per;
  const Res lo = measure([&] { lop3_issue<<<b4, 1024>>>(it_i, sink, cy, ns); },
                         (double)b4 * 32 * it_i * 8, b4);
  CK(cudaGetLastError());
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, imad_issue, 1024, 0));
  const int b5 = sms * per;
  const Res im = measure([&] { imad_issue<<<b5, 1024>>>(it_i, sink, cy, ns); },
                         (double)b5 * 32 * it_i * 8, b5);
  CK(cudaGetLastError());
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ffma_issue, 1024, 0));
  const int b6 = sms * per;
  const int it_u = it_i / kIssueUnroll;
  const Res ff = measure([&] { ffma_issue<<<b6, 1024>>>(it_u, fsink, cy, ns); },
                         (double)b6 * 32 * it_u * kIssueUnroll * 8, b6);
  CK(cudaGetLastError());
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, mix_issue, 1024, 0));
  const int b7 = sms * per;
  const Res mx = measure([&] { mix_issue<<<b7, 1024>>>(it_u, fsink, cy, ns); },
                         (double)b7 * 32 * it_u * kIssueUnroll * 8, b7);
  CK(cudaGetLastError());
  // L2: 48 MiB in total (below one die's half of the 126 MB L2), one
  // 512-thread block per SM streaming its slice
  uint4 *l2buf;
  const size_t l2_bytes = (size_t)48 << 20;
  CK(cudaMalloc(&l2buf, l2_bytes));
  CK(cudaMemset(l2buf, 0, l2_bytes));
  const size_t slice = l2_bytes / 16 / sms / 2048 * 2048;
  const int it_l2 = 64;
  const Res l2 = measure([&] { l2_rw<<<sms, 512>>>(it_l2, l2buf, slice, sink, cy, ns); },
                         (double)sms * slice * 16 * 2 * it_l2, sms);
  CK(cudaGetLastError());
  // the issue ceiling per SM per clock (best instruction mix), and the
  // rates it implies at the maximum SM clock
  const double ipc = std::max(ff.per_sm_clk, mx.per_sm_clk);
  const double fmax = clk_khz / 1e3;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_max_mhz\": %.0f, ", prop.name, sms, fmax);
  emit("smem_ld_gbs", ld, 1e-9);
  emit("smem_ldst_gbs", ls, 1e-9);
  emit("fp64_gflops", fp, 1e-9);
  emit("lop3_ginst", lo, 1e-9);
  emit("imad_ginst", im, 1e-9);
  emit("ffma_ginst", ff, 1e-9);
  emit("mix_ginst", mx, 1e-9);
  emit("l2_rw_gbs", l2, 1e-9);
  printf("\"issue_ipc_per_sm\": %.3f, \"issue_ginst_at_max_clock\": %.1f, "
         "\"smem_ldst_gbs_at_max_clock\": %.1f, \"fp64_gflops_at_max_clock\": %.1f}\n",
         ipc, ipc * sms * fmax * 1e-3, ls.per_sm_clk * sms * fmax * 1e-3,
         fp.per_sm_clk * sms * fmax * 1e-3);
  return 0;
}
