// dsmem.cu -- thread-block-cluster / distributed-shared-memory costs on this
// B200, the numbers behind DESIGN.md §9's "clusters do not pay" for the
// large-chi form: pointer-chase latency of a local vs a remote (other CTA of
// the cluster) shared-memory load, remote read bandwidth with every thread of
// both CTAs streaming the partner's buffer, and the cost of cluster.sync().
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dsmem scripts/dsmem.cu
// Prints one JSON object (cycles at the SM clock; bandwidth per SM).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

namespace cg = cooperative_groups;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                          \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

constexpr int kWords = 8192;    // u32 chase ring: 32 KB per CTA (static shared memory)

// pointer chase through a permutation in (local or the partner CTA's)
// shared memory: one thread per cluster, dependent loads
__global__ void __cluster_dims__(2, 1, 1) chase(int iters, int remote, unsigned long long *out) {
  __shared__ uint32_t ring[kWords];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < kWords; i += blockDim.x)
    ring[i] = (uint32_t)((i * 4099 + 17) & (kWords - 1));   // odd multiplier: one cycle
  cl.sync();
  if (cl.block_rank() == 0 && threadIdx.x == 0) {
    const uint32_t *r = remote ? cl.map_shared_rank(ring, 1) : ring;
    uint32_t j = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) j = r[j];
    const long long t1 = clock64();
    out[0] = (unsigned long long)(t1 - t0);
    out[1] = j;
  }
  cl.sync();
}

// the same chase through global memory with L1 bypassed (.cg: L2 hits)
__global__ void chase_l2(int iters, const uint32_t *ring, unsigned long long *out) {
  uint32_t j = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) j = __ldcg(ring + j);
  const long long t1 = clock64();
  out[0] = (unsigned long long)(t1 - t0);
  out[1] = j;
}

// every thread of both CTAs streams the partner's 32 KB buffer (uint4 loads)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(1024)
stream(int iters, unsigned long long *cyc, uint32_t *sink) {
  __shared__ uint4 buf[2048];   // 32 KB
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_uint4(i, i + 1, i + 2, i + 3);
  cl.sync();
  const uint4 *r = cl.map_shared_rank(buf, cl.block_rank() ^ 1);
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) {
      const uint4 v = r[i];
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 0x12345678u) sink[0] = acc;
  cl.sync();
}

// cost of a cluster barrier (all threads of both CTAs)
__global__ void __cluster_dims__(2, 1, 1) csync(int iters, unsigned long long *cyc) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) cl.sync();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  unsigned long long *d, h[2];
  uint32_t *sink;
  CK(cudaMalloc(&d, 1 << 20));
  CK(cudaMalloc(&sink, 64));
  const int it_c = 1 << 16;
  double lat[2];
  for (int remote = 0; remote < 2; ++remote) {
    chase<<<2, 256>>>(it_c, remote, d);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    chase<<<2, 256>>>(it_c, remote, d);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
    lat[remote] = (double)h[0] / it_c;
  }
  double lat_l2 = 0;
  {
    uint32_t hr[kWords];
    for (int i = 0; i < kWords; ++i) hr[i] = (uint32_t)((i * 4099 + 17) & (kWords - 1));
    uint32_t *dr;
    CK(cudaMalloc(&dr, sizeof(hr)));
    CK(cudaMemcpy(dr, hr, sizeof(hr), cudaMemcpyHostToDevice));
    chase_l2<<<1, 1>>>(it_c, dr, d);
    CK(cudaDeviceSynchronize());
    chase_l2<<<1, 1>>>(it_c, dr, d);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
    lat_l2 = (double)h[0] / it_c;
  }
  // bandwidth: one cluster (2 SMs) and all clusters at once
  const int it_s = 256;
  double bw1 = 0, bwall = 0;
  const int sms = prop.multiProcessorCount;
  for (int pass = 0; pass < 2; ++pass) {
    const int blocks = pass == 0 ? 2 : (sms / 2) * 2;
    stream<<<blocks, 1024>>>(it_s, d, sink);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    stream<<<blocks, 1024>>>(it_s, d, sink);
    CK(cudaDeviceSynchronize());
    unsigned long long c[512];
    CK(cudaMemcpy(c, d, blocks * 8, cudaMemcpyDeviceToHost));
    double mx = 0;
    for (int b = 0; b < blocks; ++b) mx = c[b] > mx ? (double)c[b] : mx;
    const double bytes_per_sm = (double)it_s * 2048 * 16;
    (pass == 0 ? bw1 : bwall) = bytes_per_sm / mx;   // bytes per clock per SM
  }
  const int it_y = 4096;
  csync<<<2, 512>>>(it_y, d);
  CK(cudaDeviceSynchronize());
  csync<<<2, 512>>>(it_y, d);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
  printf("{\"gpu\": \"%s\", \"smem_local_chase_cycles\": %.1f, \"dsmem_remote_chase_cycles\": %.1f, "
         "\"l2_chase_cycles\": %.1f, "
         "\"dsmem_read_bytes_per_clk_per_sm_one_cluster\": %.1f, "
         "\"dsmem_read_bytes_per_clk_per_sm_all_sms\": %.1f, \"cluster_sync_cycles\": %.1f}\n",
         prop.name, lat[0], lat[1], lat_l2, bw1, bwall, (double)h[0] / it_y);
  return 0;
}
