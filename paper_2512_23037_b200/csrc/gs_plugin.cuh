// gs_plugin.cuh -- batched kernels of the reference backend plugin API.
// Part of gs_kernels.cu (one translation unit; included inside namespace gs).
#pragma once

// @region plugin kernels + host
// ------------------------------------------------ kernel plugin API kernels
// batched equivalents of ref _kernels.pyx / _kernels_py.py

__global__ void anticommute_kernel(const u64 *xs, const u64 *zs, u32 rows, u32 batch,
                                   const u64 *qx, const u64 *qz, u64 *out) {
  const u32 lane = threadIdx.x & 31u;
  const u64 b = (u64)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= batch) return;
  const u64 X = qx[b], Zq = qz[b];
  u64 lo = 0, hi = 0;
  for (u32 base = 0; base < rows; base += 32) {
    const u32 r = base + lane;
    bool a = false;
    if (r < rows) a = ((__popcll(xs[b * rows + r] & Zq) + __popcll(zs[b * rows + r] & X)) & 1) != 0;
    const u32 bits = __ballot_sync(FULL, a);
    if (base < 64) lo |= (u64)bits << base;
    else hi |= (u64)bits << (base - 64);
  }
  if (lane == 0) { out[2 * b] = lo; out[2 * b + 1] = hi; }
}

__global__ void conj_gate_kernel(u64 *xs, u64 *zs, u8 *ph, u32 rows, u32 batch,
                                 const u32 *code, const u64 *m1s, const u64 *m2s) {
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (u64)rows * batch) return;
  const u64 b = i / rows;
  const u64 m1 = m1s[b], m2 = m2s[b];
  u64 x = xs[i], z = zs[i];
  const bool x1 = (x & m1) != 0, z1 = (z & m1) != 0;
  const bool x2 = (x & m2) != 0, z2 = (z & m2) != 0;
  bool flip = false;
  switch (code[b]) {
    case 0: return;
    case 1: flip = z1; break;
    case 2: flip = x1 ^ z1; break;
    case 3: flip = x1; break;
    case 4: flip = x1 && z1; if (x1 != z1) { x ^= m1; z ^= m1; } break;
    case 5: flip = x1 && z1; if (x1) z ^= m1; break;
    case 6: flip = x1 && !z1; if (x1) z ^= m1; break;
    case 7: flip = z1 && !x1; if (x1) z ^= m1; break;
    case 8: flip = x1 || z1; if (x1) z ^= m1; break;
    case 9: flip = x1 && z2 && !(x2 ^ z1); if (x1) x ^= m2; if (z2) z ^= m1; break;
    case 10: flip = x1 && x2 && (z1 ^ z2); if (x1) z ^= m2; if (x2) z ^= m1; break;
    case 11: if (x1 != x2) x ^= (m1 | m2); if (z1 != z2) z ^= (m1 | m2); break;
    default: return;
  }
  xs[i] = x; zs[i] = z;
  if (flip) ph[i] ^= 2;
}

__global__ void mul_rows_kernel(u64 *xs, u64 *zs, u8 *ph, u32 rows, u32 batch, const u8 *sel,
                                const u64 *pxs, const u64 *pzs, const u32 *pes) {
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (u64)rows * batch || !sel[i]) return;
  const u64 b = i / rows;
  const u64 px = pxs[b], pz = pzs[b];
  const u64 xj = xs[i], zj = zs[i], x3 = xj ^ px, z3 = zj ^ pz;
  const long long e = (long long)ph[i] + pes[b] + __popcll(px & pz) + 2 * __popcll(zj & px) +
                      __popcll(xj & zj) - __popcll(x3 & z3);
  xs[i] = x3; zs[i] = z3;
  ph[i] = (u8)(e & 3);
}

__global__ void parity_pm_kernel(const u64 *idx, size_t count, u64 mask, double *out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = 1.0 - 2.0 * (double)(__popcll(idx[i] & mask) & 1);
}
