// gs_kernels.cu -- B200 (sm_100a) shot-parallel generalized-stabilizer sampler.
//
// One warp simulates one shot at a time (persistent grid, atomic shot queue).
// The per-shot state is the static-frame state of compiler.py:
//   sig  : 2n tableau sign bits (destab word, stab word)    [ref tableau.py]
//   c    : u64 coset offset of the amplitude support        [ref state.py]
//   A    : dense complex128 amplitudes over 2^k coordinates [ref state.py]
//   rec  : measurement record bits (shared memory)
// Everything shot-invariant (x/z tableau trajectory, pivot rows, coordinate
// basis, draw offsets) was folded into the op stream on the host.
//
// Per-element arithmetic mirrors the reference's numpy forms:
//   complex product  (fma(ar,br,-(ai*bi)), fma(ar,bi,ai*br))
//   |v|^2            hypot(re,im)^2                              np.abs()**2
//   prune            hypot > 1e-12                        ref state.py:298
//   renormalise      v * (1/sqrt(sum |v|^2))                ref state.py:311
// so amplitudes agree with the reference to rounding of the (differently
// ordered) sums only.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <math.h>
#include <algorithm>
#include <string>
#include <vector>

#include "../../include/gstab_sm100.h"

// @region helpers
typedef unsigned long long u64;
typedef unsigned int u32;
typedef unsigned char u8;

#define FULL 0xffffffffu

namespace gs {

enum { OP_END = 0, OP_T = 1, OP_MEAS = 2, OP_NOISE = 3, OP_FEEDBACK = 4,
       OP_DETECTOR = 5, OP_OBSERVABLE = 6, OP_GROW_LIMIT = 7 };
enum { T_DIAG = 0, T_BUTTERFLY = 1, T_GROW = 2 };
enum { TF_FUSE = 16 };   // T flag: apply together with the next BUTTERFLY op
enum { M_DET = 0, M_PIVOT_SPAN = 1, M_PIVOT_NOSPAN = 2 };
enum { MF_RECORD = 16, MF_FLIP = 32, MF_RESET = 64, MF_COMPACT = 128 };
enum { NK_DEP1 = 0, NK_DEP2 = 1, NK_XERR = 2, NK_ZERR = 3 };
enum { ST_RUNNING = 0, ST_PRESERVED = 1, ST_DISCARDED = 2, ST_OVERFLOW = 3,
       ST_CORRUPT = 4, ST_UNSUPPORTED = 5 };
enum { MODE_COUNTERS = 0, MODE_RECORDS = 1, MODE_DUMP = 2 };

constexpr int kWinWords = 64;          // noise fire window: 2048 locations
constexpr int kWinBytes = kWinWords * 4;
constexpr double kPrune2 = 1e-24;   // (1e-12)^2, ref state.py:24
constexpr int kEntryBytes = 24;        // SURVEY §8(d) state-touch model

struct DevProg {
  const u64 *ops, *tables, *locs;
  u32 n, nmeas, max_dim, nobs, rec_words32, nlocs;
  u32 nnoise, nwords;
  u64 noise_off, wordpc_off;
  u64 geo_off, acc_off;   // Philox fire schedule: gap table, thinning table
  u32 geo_len, noise_uniform;
  float geo_ilq;          // 1 / log(1 - p_max), the gap search's first guess
};

struct DevRun {
  u64 master, shot_begin, shot_count, cap;
  u32 flags;
  const u64 *seeds;
};

struct DevOut {
  long long *counters;
  u8 *status;
  int *aux;
  u64 *rec;
  u64 *obs;
  u64 *sig;
  u64 *cvec;
  double2 *amps;
  u32 *dim;
  double2 *gchi;        // global chi scratch (per warp) when not in smem
  u32 *grec;            // global record scratch (per warp) when not in smem
  u32 mode;
  u32 warp_bytes;       // dynamic smem bytes per warp
  u32 rec_in_smem;
  u32 chi_off;          // wide kernel: byte offset of chi in the warp's smem slice
  u64 *witness;         // optional: global indices of preserved shots with a
  u32 *witness_count;   //   flipped observable (paper §V-B witnesses)
  u32 witness_cap;
};

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)),
                      __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double2 cneg(double2 a) { return make_double2(-a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double r) {
  return make_double2(__dmul_rn(a.x, r), __dmul_rn(a.y, r));
}
// |v|^2 as one fma; the reference's hypot(v)^2 and hypot(v) > 1e-12 agree
// with these except within an ulp of the threshold
__device__ __forceinline__ double abs2(double2 v) {
  return __fma_rn(v.x, v.x, __dmul_rn(v.y, v.y));
}
__device__ __forceinline__ double2 prune(double2 v) {
  return abs2(v) > kPrune2 ? v : make_double2(0.0, 0.0);
}
__device__ __forceinline__ u32 par64(u64 x) { return __popcll(x) & 1u; }
// 1/sqrt(sum |v|^2) of ref state.py:311; exactly 1 when the sum is 1
__device__ __forceinline__ double inv_sqrt_norm(double s) {
  return s == 1.0 ? 1.0 : 1.0 / sqrt(s);
}
__device__ __forceinline__ u32 par32(u32 x) { return __popc(x) & 1u; }
__device__ __forceinline__ double dbits(u64 w) { return __longlong_as_double((long long)w); }
// _I_POWERS of ref state.py:28 (signed zeros included)
__device__ __forceinline__ double2 ipow(u32 e) {
  switch (e & 3u) {
    case 0: return make_double2(1.0, 0.0);
    case 1: return make_double2(0.0, 1.0);
    case 2: return make_double2(-1.0, 0.0);
    default: return make_double2(-0.0, -1.0);
  }
}
// insert `bit` at position pos of jp
__device__ __forceinline__ u32 ins_bit(u32 jp, u32 pos, u32 bit) {
  u32 low = jp & ((1u << pos) - 1u);
  return ((jp >> pos) << (pos + 1)) | (bit << pos) | low;
}
// butterfly sum over the warp (every lane gets the same bits); inline (an
// out-of-line copy needs divergence checks around its shuffles: A/B 53.2M
// vs 52.1M shots/s in the section design)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ u32 warp_sum_u32(u32 v) { return __reduce_add_sync(FULL, v); }
__device__ __forceinline__ u64 warp_or64(u64 v) {
  u32 lo = __reduce_or_sync(FULL, (u32)v);
  u32 hi = __reduce_or_sync(FULL, (u32)(v >> 32));
  return ((u64)hi << 32) | lo;
}

// ---------------------------------------------------------------- RNG

__device__ __forceinline__ u32 bswap32(u32 x) { return __byte_perm(x, 0, 0x0123); }
__device__ __forceinline__ u32 rotl(u32 x, int r) { return __funnelshift_l(x, x, r); }

// derive_seed: first 8 bytes (LE) of SHA-1(LE64 master || LE64 shot)
// (ref sampler.py:37-42); single 64-byte block.
__device__ __noinline__ u64 sha1_seed(u64 master, u64 shot) {
  u32 w[16];
  w[0] = bswap32((u32)master);
  w[1] = bswap32((u32)(master >> 32));
  w[2] = bswap32((u32)shot);
  w[3] = bswap32((u32)(shot >> 32));
  w[4] = 0x80000000u;
#pragma unroll
  for (int i = 5; i < 15; ++i) w[i] = 0;
  w[15] = 128;
  u32 a = 0x67452301u, b = 0xEFCDAB89u, c = 0x98BADCFEu, d = 0x10325476u,
      e = 0xC3D2E1F0u;
#pragma unroll
  for (int i = 0; i < 80; ++i) {
    u32 wi;
    if (i < 16) {
      wi = w[i];
    } else {
      wi = rotl(w[(i - 3) & 15] ^ w[(i - 8) & 15] ^ w[(i - 14) & 15] ^ w[i & 15], 1);
      w[i & 15] = wi;
    }
    u32 f, k;
    if (i < 20) { f = (b & c) | (~b & d); k = 0x5A827999u; }
    else if (i < 40) { f = b ^ c ^ d; k = 0x6ED9EBA1u; }
    else if (i < 60) { f = (b & c) | (b & d) | (c & d); k = 0x8F1BBCDCu; }
    else { f = b ^ c ^ d; k = 0xCA62C1D6u; }
    u32 t = rotl(a, 5) + f + e + k + wi;
    e = d; d = c; c = rotl(b, 30); b = a; a = t;
  }
  u32 h0 = 0x67452301u + a, h1 = 0xEFCDAB89u + b;
  return ((u64)bswap32(h1) << 32) | bswap32(h0);
}

__device__ __forceinline__ u64 splitmix(u64 seed, u32 k) {
  u64 z = seed + (u64)(k + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Philox4x32-10, key = master seed, counter = (c0, c1, shot lo, shot hi)
__device__ __forceinline__ uint4 philox4(u32 c0, u32 c1, u64 shot, u64 master) {
  u32 c2 = (u32)shot, c3 = (u32)(shot >> 32);
  u32 k0 = (u32)master, k1 = (u32)(master >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    u32 lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    u32 lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    u32 n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return make_uint4(c0, c1, c2, c3);
}

// static draw k (measurements, MPP flips): block (k>>1, 0, shot), even k
// takes words (0,1), odd k words (2,3)
__device__ __forceinline__ u64 philox_u64(u64 master, u64 shot, u32 k) {
  const uint4 x = philox4(k >> 1, 0u, shot, master);
  return (k & 1u) ? (((u64)x.w << 32) | x.z) : (((u64)x.y << 32) | x.x);
}

// Philox-mode noise: candidate j of the shot's Bernoulli(p_max) location
// process (oracle GeoNoise).  Block (j, 1, shot): words 0-1 >> 11 = gap draw
// m, words 2-3 >> 11 = letter pick; gap = max{g : m < T[g]} (binary search
// of the host gap table); the candidate sits at start + gap.
struct GeoCand {
  u64 pick;
  u32 pos;
};
// The search starts from the float guess log(u)/log(1-p_max) (`ilq` =
// 1/log(T[1] 2^-53)) and narrows to a 3-entry window before bisecting, so a
// gap costs ~4 table loads instead of log2(tlen); the table decides (exact).
__device__ __noinline__ GeoCand geo_candidate(const u64 *__restrict__ T, u32 tlen, float ilq,
                                              u64 master, u64 shot, u32 j, u32 start) {
  const uint4 x = philox4(j, 1u, shot, master);
  const u64 m = ((((u64)x.y) << 32) | x.x) >> 11;
  GeoCand c;
  c.pick = ((((u64)x.w) << 32) | x.z) >> 11;
  const u32 G = tlen - 1;
  // answer = max{g <= G : m < T[g]}; invariant: m < T[lo], answer <= hi
  const float gf = __logf(((float)m + 0.5f) * 0x1.0p-53f) * ilq;
  u32 g = gf >= (float)G ? G : (gf > 0.f ? (u32)gf : 0u);
  u32 lo = 0, hi = G;
  if (m < __ldg(T + g)) {
    lo = g;
    if (g + 3 <= G && !(m < __ldg(T + g + 3))) hi = g + 2;
  } else {
    hi = g - 1;                      // g >= 1: T[0] = 2^53 > m
    if (g >= 3 && m < __ldg(T + g - 3)) lo = g - 3;
  }
  while (lo < hi) {
    const u32 mid = (lo + hi + 1) >> 1;
    if (m < __ldg(T + mid)) lo = mid; else hi = mid - 1;
  }
  c.pos = start + lo;
  return c;
}
// thinning of candidate j at a location with p < p_max: block (j, 2, shot)
__device__ __noinline__ bool geo_accept(u64 master, u64 shot, u32 j, u64 thr) {
  const uint4 x = philox4(j, 2u, shot, master);
  return (((((u64)x.y) << 32) | x.x) >> 11) < thr;
}

__device__ __noinline__ u64 draw53(u64 seed, u64 master, u64 shot, u32 k, bool philox) {
  return (philox ? philox_u64(master, shot, k) : splitmix(seed, k)) >> 11;
}

struct Rng {
  u64 seed, master, shot;
  bool philox;
  __device__ __forceinline__ u64 m53(u32 k) const {
    return draw53(seed, master, shot, k, philox);
  }
  __device__ __forceinline__ double uniform(u32 k) const {
    return (double)m53(k) * 0x1.0p-53;
  }
};

// ---------------------------------------------------------------- chi storage
//
// Per shot the chi map is a dense complex128 array over the 2^k coordinates
// of the static basis (zero = absent reference entry, so partner lookups
// are O(1)); positions >= 2^k are don't-care until a GROW initialises them.

#ifndef GS_KN
#define GS_KN 4u                // narrow (lane-per-shot) chi dimension limit
#endif
constexpr u32 kNarrowBytes = (1u << GS_KN) * 32u * 16u;   // An[2^KN][32] double2
constexpr u32 kCntBytes = 64;                              // per-warp counters

__device__ __forceinline__ bool nonzero(double2 v) { return v.x != 0.0 || v.y != 0.0; }

__device__ __forceinline__ u32 lanemask_lt(u32 lane) { return (1u << lane) - 1u; }

// @region sweeps
// ---------------------------------------------------------------- wide sweeps
//
// Warp-cooperative passes over a dense chi array A[0, 2^k): lane l takes
// coordinates l, l+32, ... (pair / group indices for the T sweeps), one
// group in flight per lane -- measured on the B200, more per lane (unrolled
// rounds, 8-element groups of three fused gates) was slower every time
// (profiles/README.md).  Inlined into wide_kernel (+1.4 % over out-of-line
// copies once each section kernel has its own code).  Per-lane partial
// results (nonzero count, sum of |v|^2 of the written entries = the chi
// norm the next deterministic measurement needs); callers reduce across
// the warp.

struct SumNz {
  double sum;
  u32 nz;
};

// A[i] with a renormalisation still pending (ps != 1): the reference would
// have stored v * ps (ref state.py:311), so every reader applies it first --
// the same rounding, one pass later
__device__ __forceinline__ double2 ldps(const double2 *__restrict__ A, u32 i, double ps) {
  const double2 v = A[i];
  return ps != 1.0 ? cscale(v, ps) : v;
}
// prune at |v| <= 1e-12 (ref state.py:298), accumulating |v|^2 of the kept
__device__ __forceinline__ double2 prune_acc(double2 v, double &sum, u32 &nz) {
  const double q = abs2(v);
  if (q > kPrune2) {
    sum = __dadd_rn(sum, q);
    nz += 1;
    return v;
  }
  return make_double2(0.0, 0.0);
}

// The T sweeps are the hottest code (about half of all instructions): chi
// is addressed as shared memory when it lives there (LDS/STS instead of
// generic loads), and the per-coordinate sign (-1)^s of the b-term is applied
// to the product b*v by flipping sign bits -- cmul(-b, v) == -cmul(b, v)
// bit for bit, since fma(-x, y, -z) == -fma(x, y, z).
template <bool kS>
__device__ __forceinline__ double2 *chi_ptr(double2 *A) {
  if (!kS) return A;
  extern __shared__ __align__(16) u8 smem_dyn[];
  return reinterpret_cast<double2 *>(smem_dyn + (reinterpret_cast<u8 *>(A) - smem_dyn));
}
__device__ __forceinline__ double2 neg_if(double2 v, u32 s) {
  const long long m = (long long)s << 63;
  return make_double2(__longlong_as_double(__double_as_longlong(v.x) ^ m),
                      __longlong_as_double(__double_as_longlong(v.y) ^ m));
}

// T with beta in span: new[j] = a v_j + b_j v_{j^cb} (ref state.py:127-129,
// 294-306: a-term then b-term); no renormalisation pending (caller)
template <bool kS>
__device__ __forceinline__ SumNz sweep_butterfly(double2 *A_, u32 half, u32 cb, u32 dc, u32 dmask,
                                              double2 a, double2 bx0) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = threadIdx.x & 31u;
  const u32 hb = 31 - __clz(cb);
  SumNz r;
  r.sum = 0.0;
  r.nz = 0;
  const u32 jl = ins_bit(lane, hb, 0);
  const u32 pl = dc ^ par32(jl & dmask), pcb = par32(cb & dmask);
#pragma unroll 1
  for (u32 m = lane; m < half; m += 32) {
    const u32 jr = ins_bit(m & ~31u, hb, 0);
    const u32 j0 = jr | jl, j1 = j0 ^ cb;
    const double2 v0 = A[j0], v1 = A[j1];
    const u32 s0 = pl ^ par32(jr & dmask), s1 = s0 ^ pcb;
    A[j0] = prune_acc(cadd(cmul(a, v0), neg_if(cmul(bx0, v1), s1)), r.sum, r.nz);
    A[j1] = prune_acc(cadd(cmul(a, v1), neg_if(cmul(bx0, v0), s0)), r.sum, r.nz);
  }
  return r;
}

// Two consecutive T gates with partner vectors cb1 != cb2 (compiler flag
// TF_FUSE): one pass over the 4-element groups {x, x^cb1, x^cb2,
// x^cb1^cb2}; gate 1 on the cb1 pairs, prune, gate 2 on the cb2 pairs,
// prune -- exactly the two single-gate passes' arithmetic, half the memory
// traffic and index work.  Groups are enumerated by inserting zeros at the
// pivot bits h1 = top(cb1) and h2 = top(cb2 reduced by cb1).
struct Gate {
  double2 a, bx0;
  u32 cb, dc, dmask;
};
struct SumNz2 {
  double sum;
  u32 nz, nz1;
};
template <bool kS>
__device__ __forceinline__ SumNz2 sweep_butterfly2(double2 *A_, u32 quarter, Gate g1, Gate g2) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = threadIdx.x & 31u;
  const u32 h1 = 31 - __clz(g1.cb);
  const u32 cr = ((g2.cb >> h1) & 1u) ? (g2.cb ^ g1.cb) : g2.cb;
  const u32 h2 = 31 - __clz(cr);
  const u32 plo = min(h1, h2), phi = max(h1, h2);
  SumNz2 r;
  r.sum = 0.0;
  r.nz = 0;
  r.nz1 = 0;
  double dummy = 0.0;
  // sign parities: the zero-insertion J is bitwise linear, so for
  // m = 32r + lane, par(J(m) & mask) = par(J(32r) & mask) ^ par(J(lane) & mask)
  // (a per-round and a per-lane term); the group members differ by cb1, cb2
  const u32 jl = ins_bit(ins_bit(lane, plo, 0), phi, 0);
  const u32 l1 = g1.dc ^ par32(jl & g1.dmask), l2 = g2.dc ^ par32(jl & g2.dmask);
  const u32 a1 = par32(g1.cb & g1.dmask), b1 = par32(g2.cb & g1.dmask);
  const u32 a2 = par32(g1.cb & g2.dmask), b2 = par32(g2.cb & g2.dmask);
#pragma unroll 1
  for (u32 m = lane; m < quarter; m += 32) {
    const u32 jr = ins_bit(ins_bit(m & ~31u, plo, 0), phi, 0);
    const u32 x0 = jr | jl;
    const u32 x1 = x0 ^ g1.cb, x2 = x0 ^ g2.cb, x3 = x1 ^ g2.cb;
    const double2 v0 = A[x0], v1 = A[x1], v2 = A[x2], v3 = A[x3];
    const u32 p1 = l1 ^ par32(jr & g1.dmask), p2 = l2 ^ par32(jr & g2.dmask);
    // gate 1: pairs (x0, x1), (x2, x3)
    const u32 s0 = p1, s1 = p1 ^ a1, s2 = p1 ^ b1, s3 = p1 ^ a1 ^ b1;
    const double2 u0 = prune_acc(cadd(cmul(g1.a, v0), neg_if(cmul(g1.bx0, v1), s1)), dummy, r.nz1);
    const double2 u1 = prune_acc(cadd(cmul(g1.a, v1), neg_if(cmul(g1.bx0, v0), s0)), dummy, r.nz1);
    const double2 u2 = prune_acc(cadd(cmul(g1.a, v2), neg_if(cmul(g1.bx0, v3), s3)), dummy, r.nz1);
    const double2 u3 = prune_acc(cadd(cmul(g1.a, v3), neg_if(cmul(g1.bx0, v2), s2)), dummy, r.nz1);
    // gate 2: pairs (x0, x2), (x1, x3)
    const u32 t0 = p2, t1 = p2 ^ a2, t2 = p2 ^ b2, t3 = p2 ^ a2 ^ b2;
    A[x0] = prune_acc(cadd(cmul(g2.a, u0), neg_if(cmul(g2.bx0, u2), t2)), r.sum, r.nz);
    A[x2] = prune_acc(cadd(cmul(g2.a, u2), neg_if(cmul(g2.bx0, u0), t0)), r.sum, r.nz);
    A[x1] = prune_acc(cadd(cmul(g2.a, u1), neg_if(cmul(g2.bx0, u3), t3)), r.sum, r.nz);
    A[x3] = prune_acc(cadd(cmul(g2.a, u3), neg_if(cmul(g2.bx0, u1), t1)), r.sum, r.nz);
  }
  (void)dummy;
  return r;
}

// T with a new basis vector: A[j] = a v_j, A[size+j] = b_j v_j
template <bool kS>
__device__ __forceinline__ SumNz sweep_grow(double2 *A_, u32 size, u32 dc, u32 dmask, double2 a,
                                         double2 bx0) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = threadIdx.x & 31u;
  SumNz r;
  r.sum = 0.0;
  r.nz = 0;
#pragma unroll 1
  for (u32 j = lane; j < size; j += 32) {
    const double2 v = A[j];
    A[j] = prune_acc(cmul(a, v), r.sum, r.nz);
    A[size + j] = prune_acc(neg_if(cmul(bx0, v), dc ^ par32(j & dmask)), r.sum, r.nz);
  }
  return r;
}

// diagonal phase: A[j] *= (dc ^ par(j & mask)) ? f1 : f0  (T with beta = 0,
// fired noise Paulis)
template <bool kS>
__device__ __forceinline__ void sweep_phase(double2 *A_, u32 size, u32 dc, u32 mask,
                                         double2 f0, double2 f1, double ps) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = threadIdx.x & 31u;
#pragma unroll 1
  for (u32 j = lane; j < size; j += 32)
    A[j] = cmul(ldps(A, j, ps), (dc ^ par32(j & mask)) ? f1 : f0);
}

// beta = 0 measurement weights: (sum over +1 eigen-entries, sum over -1)
template <bool kS>
__device__ __forceinline__ double2 sweep_det_sums(double2 *A_, u32 size, u32 dmask, u32 neg0,
                                               double ps) {
  const double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = threadIdx.x & 31u;
  double sp = 0.0, sm = 0.0;
#pragma unroll 1
  for (u32 j = lane; j < size; j += 32) {
    const double a2 = abs2(ldps(A, j, ps));
    if (neg0 ^ par32(j & dmask)) sm = __dadd_rn(sm, a2); else sp = __dadd_rn(sp, a2);
  }
  return make_double2(sp, sm);
}

// keep the chosen eigen-entries, scaled by rs; zero the others
template <bool kS>
__device__ __forceinline__ SumNz sweep_filter(double2 *A_, u32 size, u32 dmask, u32 neg0,
                                           u32 want_neg, double rs, double ps) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = threadIdx.x & 31u;
  SumNz r;
  r.sum = 0.0;
  r.nz = 0;
#pragma unroll 1
  for (u32 j = lane; j < size; j += 32) {
    const double2 v = ldps(A, j, ps);
    if ((neg0 ^ par32(j & dmask)) == want_neg) {
      const double2 w = cscale(v, rs);
      A[j] = w;
      r.sum = __dadd_rn(r.sum, abs2(w));
      r.nz += nonzero(w);
    } else {
      A[j] = make_double2(0.0, 0.0);
    }
  }
  return r;
}

// in-place compaction dropping coordinate isq: A[jp] = rs * A[src(jp)],
// src(jp) = j0 | ((tau ^ par(j0 & mask)) << isq), j0 = jp with a 0 inserted
// at isq; src(jp) >= jp, so reads of a round finish before its writes
template <bool kS>
__device__ __forceinline__ SumNz sweep_compact(double2 *A_, u32 half, u32 isq, u32 mask, u32 tau,
                                            double rs, double ps) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = threadIdx.x & 31u;
  SumNz r;
  r.sum = 0.0;
  r.nz = 0;
#pragma unroll 1
  for (u32 b0 = 0; b0 < half; b0 += 32) {
    const u32 jp = b0 + lane;
    double2 v = make_double2(0.0, 0.0);
    if (jp < half) {
      const u32 j0 = ins_bit(jp, isq, 0);
      v = ldps(A, j0 | ((tau ^ par32(j0 & mask)) << isq), ps);
    }
    __syncwarp();
    if (jp < half) {
      const double2 w = cscale(v, rs);
      A[jp] = w;
      r.sum = __dadd_rn(r.sum, abs2(w));
      r.nz += nonzero(w);
    }
    __syncwarp();
  }
  return r;
}

// pivot measurement (ref state.py:178-208): w(m) = rep + sg * xi * part.
// span: pairs (rep, rep^cb), rep = j0 | ((ct ^ par(j0 & tmask)) << isq);
// no span: every entry, entries with ct ^ par(m & tmask) are `part` only.
// pass 1 returns the per-lane sum of |w+|^2; pass 2 writes prune(w_sg) to
// the rep slot and returns (sum |w|^2, nonzeros).
struct PivotGeo {
  u32 npairs, isq, tmask, ct, cb, dc, dmask;
  bool span;
};
__device__ __forceinline__ void pivot_terms(const double2 *__restrict__ A, const PivotGeo &g,
                                            double2 xpp, u32 m, double2 &vr, double2 &pr,
                                            u32 &dst, double ps) {
  const double2 xpm = cneg(xpp);
  if (g.span) {
    const u32 j0 = ins_bit(m, g.isq, 0);
    const u32 rep = j0 | ((g.ct ^ par32(j0 & g.tmask)) << g.isq);
    const u32 part = rep ^ g.cb;
    vr = ldps(A, rep, ps);
    pr = cmul((g.dc ^ par32(part & g.dmask)) ? xpm : xpp, ldps(A, part, ps));
    dst = rep;
  } else {
    const double2 v = ldps(A, m, ps);
    if (g.ct ^ par32(m & g.tmask)) {
      vr = make_double2(0.0, 0.0);
      pr = cmul((g.dc ^ par32(m & g.dmask)) ? xpm : xpp, v);
    } else {
      vr = v;
      pr = make_double2(-0.0, -0.0);   // v + (-0) == v exactly
    }
    dst = m;
  }
}
template <bool kS>
__device__ __forceinline__ double sweep_pivot_p(double2 *A_, PivotGeo g, double2 xpp, double ps) {
  const double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = threadIdx.x & 31u;
  double sp = 0.0;
#pragma unroll 1
  for (u32 m = lane; m < g.npairs; m += 32) {
    double2 vr, pr;
    u32 d_;
    pivot_terms(A, g, xpp, m, vr, pr, d_, ps);
    sp = __dadd_rn(sp, abs2(cadd(vr, pr)));
  }
  return sp;
}
template <bool kS>
__device__ __forceinline__ SumNz sweep_pivot_w(double2 *A_, PivotGeo g, double2 xpp, bool plus,
                                            double ps) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = threadIdx.x & 31u;
  SumNz r;
  r.sum = 0.0;
  r.nz = 0;
#pragma unroll 1
  for (u32 m = lane; m < g.npairs; m += 32) {
    double2 vr, pr;
    u32 dst;
    pivot_terms(A, g, xpp, m, vr, pr, dst, ps);
    A[dst] = prune_acc(plus ? cadd(vr, pr) : csub(vr, pr), r.sum, r.nz);
  }
  return r;
}

// apply a pending renormalisation in place: A[j] = ps * A[j]
template <bool kS>
__device__ __forceinline__ void sweep_scale(double2 *A_, u32 size, double ps) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = threadIdx.x & 31u;
#pragma unroll 1
  for (u32 j = lane; j < size; j += 32) A[j] = cscale(A[j], ps);
}

// ---------------------------------------------------------------- kernels
//
// Execution model: breadth-first SECTIONS.  k is static per op
// (shot-invariant basis, compiler.py), so the op stream splits on the host
// into alternating sections of narrow ops (chi dimension k <= GS_KN before
// and after the op) and wide ops (k > GS_KN, GROW_LIMIT).  One launch per
// section runs every live shot of the chunk through it:
//
//  * narrow_kernel: a warp takes 32 shots (one per lane) and walks the
//    section with all lanes at the same pc; chi lives in shared memory as
//    An[j * 32 + lane] (row j uniform across lanes, conflict free); the
//    fixed per-op cost (decode, sign-mask popcounts, static tables) is paid
//    once per 32 shots;
//  * wide_kernel: a warp takes one shot and splits its 2^k coordinates over
//    the lanes (chi in the warp's shared-memory buffer; `sweep_*`).
//
// Shots that survive a section are appended to a global queue (fixed-size
// slots: state words, record bits, chi of dimension <= GS_KN) read by the
// next section's launch.  Each launch keeps only its own code hot, which is
// what the instruction cache needs (B200: 32 KB L1.5).
// GS_WIDE_ONLY runs the whole program as one wide section (A/B, tests).

#ifndef GS_NARROW_BLOCKS
#define GS_NARROW_BLOCKS 5   // <= 102 registers: 20 warps/SM (A/B: 47.4M vs 46.4M at 4)
#endif
#ifndef GS_WIDE_BLOCKS
#define GS_WIDE_BLOCKS 3   // <= 168 registers (no spills); shared memory holds 12-13 warps/SM anyway
#endif

__host__ __device__ __forceinline__ bool op_is_wide(u32 kind, u32 k, u32 fl) {
  return kind == OP_GROW_LIMIT || k > GS_KN ||
         (kind == OP_T && (fl & 3u) == T_GROW && k + 1 > GS_KN);
}

// action of a fired error E = X^ex Z^ez on the static frame:
// alpha ^= beta, v *= i^xi (-1)^{delta.alpha}; `dm` = delta in coordinates
struct ErrAct {
  u64 beta, delt;
  u32 xi, dm;
};
__device__ __noinline__ ErrAct compose_error(const u64 *__restrict__ tables, u64 ex, u64 ez,
                                             u64 qmask, u64 off, u64 sig_lo, u64 sig_hi) {
  ErrAct r;
  r.beta = 0; r.delt = 0; r.xi = 0; r.dm = 0;
#pragma unroll 1
  for (u64 rem = ex | ez; rem; rem &= rem - 1) {
    const u32 q = __ffsll((long long)rem) - 1;
    const u32 slot = __popcll(qmask & ((1ull << q) - 1ull));
    const u64 *tb = tables + off + 10ull * slot;
    const u64 xb_ = __ldg(tb + 0), xd_ = __ldg(tb + 1);
    const u64 xw64 = __ldg(tb + 4);
    const u32 xx = (((u32)xw64 & 3u) + 2u * (par64(sig_lo & __ldg(tb + 2)) ^ par64(sig_hi & __ldg(tb + 3)))) & 3u;
    const u64 zb_ = __ldg(tb + 5), zd_ = __ldg(tb + 6);
    const u64 zw64 = __ldg(tb + 9);
    const u32 zx = (((u32)zw64 & 3u) + 2u * (par64(sig_lo & __ldg(tb + 7)) ^ par64(sig_hi & __ldg(tb + 8)))) & 3u;
    const u32 xdm = (u32)(xw64 >> 8), zdm = (u32)(zw64 >> 8);
    const bool hx = (ex >> q) & 1, hz = (ez >> q) & 1;
    u64 lb, ld; u32 lxi, ldm;
    if (hx && hz) {   // Y = i X Z
      lb = xb_ ^ zb_; ld = xd_ ^ zd_; ldm = xdm ^ zdm;
      lxi = (1u + xx + zx + 2u * par64(xd_ & zb_)) & 3u;
    } else if (hx) {
      lb = xb_; ld = xd_; lxi = xx; ldm = xdm;
    } else {
      lb = zb_; ld = zd_; lxi = zx; ldm = zdm;
    }
    r.xi = (r.xi + lxi + 2u * par64(r.delt & lb)) & 3u;
    r.beta ^= lb; r.delt ^= ld; r.dm ^= ldm;
  }
  return r;
}

// letter of a fired location from its pick draw u (ref noise.py:68-100)
__device__ __forceinline__ void noise_letter(u32 nk, u32 qa, u32 qb, double u, u64 &ex, u64 &ez) {
  if (nk == NK_DEP1) {
    int code = 1 + (int)(u * 3.0);
    code = code > 3 ? 3 : code;
    ex |= (u64)(code != 3) << qa;
    ez |= (u64)(code != 1) << qa;
  } else if (nk == NK_DEP2) {
    int pick = 1 + (int)(u * 15.0);
    pick = pick > 15 ? 15 : pick;
    const int ca = pick & 3, cbq = pick >> 2;
    if (ca) { ex |= (u64)(ca != 3) << qa; ez |= (u64)(ca != 1) << qa; }
    if (cbq) { ex |= (u64)(cbq != 3) << qb; ez |= (u64)(cbq != 1) << qb; }
  } else if (nk == NK_XERR) {
    ex |= 1ull << qa;
  } else {
    ez |= 1ull << qa;
  }
}

// owning noise instruction of location l: its index sits in bits 50..63 of
// the location word when the program has < 2^14 noise instructions
// (compiler.OWNER_LIMIT), else bisect: last m with loc0(m) <= l
__device__ __forceinline__ const u64 *noise_owner(const DevProg &P, u32 l) {
  if (P.nnoise <= (1u << 14))
    return P.tables + P.noise_off + 4ull * (u32)(__ldg(P.locs + 2ull * l) >> 50);
  u32 lo = 0, hi = P.nnoise;
  while (hi - lo > 1) {
    const u32 mid = (lo + hi) >> 1;
    if ((u32)__ldg(P.tables + P.noise_off + 4ull * mid + 1) <= l) lo = mid; else hi = mid;
  }
  return P.tables + P.noise_off + 4ull * lo;
}

// queue slot layout (u64 words): state, then record bits (u32 words), then
// the chi rows [0, 2^GS_KN)
enum { Q_SL = 0, Q_LO, Q_HI, Q_C, Q_OBS, Q_MB, Q_PICK, Q_SEED, Q_CNTK, Q_GEO, Q_FIRE, Q_HDR = 12 };

struct DevSec {
  u32 pc0, k0, nm0;        // first op, its chi dimension, first noise instr. with ipc >= pc0
  u32 pc_end;              // narrow: stop before this op (0xFFFFFFFF: at the first wide op)
  u64 first, count;        // fresh shots (q_in == nullptr): run-local indices [first, first+count)
  const u64 *q_in;         // else: queue slots and their number
  const u32 *n_in;
  u64 *q_out;              // survivors at the section end (nullptr: last section)
  u32 *n_out;
  unsigned long long *work; // atomic work counter
};

// record words of a slot, rounded to 16 B so the chi rows are double2-aligned
__host__ __device__ __forceinline__ u32 rec_u64(u32 rec_words32) { return ((rec_words32 + 3) / 4) * 2; }

__device__ __forceinline__ u32 slot_u64(const DevProg &P) {
  return Q_HDR + rec_u64(P.rec_words32) + 2 * (1u << GS_KN);
}

// per-warp counters in shared memory
enum { WC_TOT = 0, WC_PRES, WC_DISC, WC_OVF, WC_COR, WC_UNS, WC_ERR, WC_MB, WC_N };

__device__ __forceinline__ void flush_counters(const DevOut &O, unsigned long long *wcnt, u32 lane) {
  __syncwarp();
  if (lane < WC_N && wcnt[lane]) {
    static_assert(WC_N == 8, "counter order");
    const int dst[WC_N] = {GS_C_TOTAL, GS_C_PRESERVED, GS_C_DISCARDED, GS_C_OVERFLOW,
                           GS_C_CORRUPT, GS_C_UNSUPPORTED, GS_C_ERROR_SHOTS, GS_C_MODEL_BYTES};
    atomicAdd((unsigned long long *)O.counters + dst[lane], wcnt[lane]);
  }
}

// ---------------------------------------------------------------- narrow

template <bool kPhilox>
__global__ void __launch_bounds__(128, GS_NARROW_BLOCKS)
narrow_kernel(DevProg P, DevRun R, DevOut O, DevSec S) {
  extern __shared__ __align__(16) u8 smem[];
  const u32 lane = threadIdx.x & 31u;
  const u32 wib = threadIdx.x >> 5;
  const u32 wpb = blockDim.x >> 5;
  const u64 gw = (u64)blockIdx.x * wpb + wib;
  u8 *mine = smem + (size_t)wib * O.warp_bytes;
  unsigned long long *wcnt = reinterpret_cast<unsigned long long *>(mine);
  double2 *An = reinterpret_cast<double2 *>(mine + kCntBytes);
  // record bits, one column per lane: word w of lane l at recb[w * 32 + l]
  u32 *recb = O.rec_in_smem ? reinterpret_cast<u32 *>(mine + kCntBytes + kNarrowBytes)
                            : O.grec + gw * (u64)P.rec_words32 * 32u;
  const u32 n = P.n;
  const u64 *__restrict__ ops = P.ops;
  const u64 *__restrict__ tables = P.tables;
  const u64 *__restrict__ locs = P.locs;
  const double2 Z = make_double2(0.0, 0.0);
  constexpr bool philox = kPhilox;   // RNG mode is a template parameter
  const u32 sign_bytes = 2u * ((2u * n + 7u) / 8u);
  const u32 SU = slot_u64(P);
#define AN(j) An[(j) * 32u + lane]

  if (lane < WC_N) wcnt[lane] = 0;
  __syncwarp();
  const u64 total = S.q_in ? (u64)*S.n_in : S.count;

#pragma unroll 1
  for (;;) {
    // @region narrow: batch setup
    u64 base = 0;
    if (lane == 0) base = atomicAdd(S.work, 32ull);
    base = __shfl_sync(FULL, base, 0);
    if (base >= total) break;
    const u64 idx = base + lane;
    const bool valid = idx < total;
    // this lane's shot (ref sampler.py:169-255 state: tableau signs, coset
    // offset, record, observables)
    u64 sl = 0, shot = 0, seed = 0;
    u64 s_lo = 0, s_hi = 0, sc = 0, sobs = 0, smb = 0;
    u32 scnt = 1, sk = S.k0;
    int sst = valid ? ST_RUNNING : ST_PRESERVED, saux = -1;
    // Philox fire schedule of this shot
    u32 sgj = 0, sgpos = 0xFFFFFFFFu, sfire = 0xFFFFFFFFu;
    u64 sgpick = 0;
    if (!S.q_in) {
      sl = S.first + idx;
      shot = R.shot_begin + sl;
      if (valid && !philox) seed = R.seeds ? R.seeds[sl] : sha1_seed(R.master, shot);
#pragma unroll 1
      for (u32 w = 0; w < P.rec_words32; ++w) recb[w * 32u + lane] = 0;
      AN(0) = make_double2(1.0, 0.0);
      if (philox && valid && P.geo_len > 1 && P.nlocs) {
        const GeoCand gc = geo_candidate(tables + P.geo_off, P.geo_len, P.geo_ilq, R.master, shot, 0u, 0u);
        sgpos = gc.pos;
        sgpick = gc.pick;
        sgj = 1;
        sfire = sgpos < P.nlocs ? 0u : 0xFFFFFFFFu;
      }
    } else if (valid) {
      const u64 *q = S.q_in + idx * SU;
      sl = q[Q_SL];
      shot = R.shot_begin + sl;
      s_lo = q[Q_LO]; s_hi = q[Q_HI]; sc = q[Q_C]; sobs = q[Q_OBS]; smb = q[Q_MB];
      sgpick = q[Q_PICK]; seed = q[Q_SEED];
      scnt = (u32)q[Q_CNTK];
      sgj = (u32)q[Q_GEO]; sgpos = (u32)(q[Q_GEO] >> 32);
      sfire = (u32)q[Q_FIRE];
      const u32 *qr = reinterpret_cast<const u32 *>(q + Q_HDR);
#pragma unroll 1
      for (u32 w = 0; w < P.rec_words32; ++w) recb[w * 32u + lane] = qr[w];
      const double2 *qc = reinterpret_cast<const double2 *>(q + Q_HDR + rec_u64(P.rec_words32));
#pragma unroll 1
      for (u32 j = 0; j < (1u << S.k0); ++j) AN(j) = qc[j];
    }
    __syncwarp();

    u32 pc = S.pc0, nm = S.nm0;
    u32 exit_k = 0;
#pragma unroll 1
    for (;;) {
      if (!__any_sync(FULL, sst == ST_RUNNING)) break;
      const u64 h = __ldg(ops + pc);
      const u32 kind = (u32)(h & 0xff), len = (u32)((h >> 8) & 0xff);
      const u32 k = (u32)((h >> 16) & 0xff), fl = (u32)((h >> 24) & 0xff);
      const u32 instr = (u32)(h >> 32);
      if (pc == S.pc_end || op_is_wide(kind, k, fl)) { exit_k = k; break; }   // section end
      // ============================== narrow op, lane per shot
      // @region narrow: noise
      // apply E to this lane's shot (ref state.py:88-102)
      auto lane_error = [&](u64 ex, u64 ez, const u64 *nrec, u32 size) {
        const ErrAct e = compose_error(tables, ex, ez, __ldg(nrec + 2), __ldg(nrec + 3), s_lo, s_hi);
        const double2 php = ipow(e.xi);
        const double2 phm = cneg(php);
        const u32 dcn = par64(e.delt & sc);
#pragma unroll 1
        for (u32 j = 0; j < size; ++j) AN(j) = cmul(AN(j), (dcn ^ par32(j & e.dm)) ? phm : php);
        sc ^= e.beta;
        smb += 2ull * kEntryBytes * scnt + sign_bytes;
      };
      const u64 *op = ops + pc;
      const u32 size = 1u << k;
      // ---- noise instructions inserted before this op
      if (!philox) {
#pragma unroll 1
        for (; nm < P.nnoise; ++nm) {
          const u64 *nrec = tables + P.noise_off + 4ull * nm;
          const u64 nw0 = __ldg(nrec);
          if ((u32)nw0 > pc) break;
          if (sst != ST_RUNNING) continue;
          const u32 nloc = (u32)(nw0 >> 32), loc0 = (u32)__ldg(nrec + 1);
          u64 ex = 0, ez = 0;
#pragma unroll 1
          for (u32 l = loc0; l < loc0 + nloc; ++l) {
            const u64 lw = __ldg(locs + 2ull * l), thr = __ldg(locs + 2ull * l + 1);
            const u32 d = (u32)lw;
            if ((splitmix(seed, d) >> 11) < thr) {
              const u32 nk = (u32)(lw >> 48) & 3;
              const double u = nk <= NK_DEP2 ? (double)(splitmix(seed, d + 1) >> 11) * 0x1.0p-53 : 0.0;
              noise_letter(nk, (u32)(lw >> 32) & 0xff, (u32)(lw >> 40) & 0xff, u, ex, ez);
            }
          }
          if (ex | ez) lane_error(ex, ez, nrec, size);
        }
      } else {
        if (sst == ST_RUNNING && pc >= sfire) {
          sfire = 0xFFFFFFFFu;
          while (sgpos < P.nlocs) {
            const u64 *nrec = noise_owner(P, sgpos);
            const u64 nw0 = __ldg(nrec);
            const u32 ipc = (u32)nw0, nloc = (u32)(nw0 >> 32);
            if (ipc > pc) { sfire = ipc; break; }
            const u32 loc0 = (u32)__ldg(nrec + 1);
            u64 ex = 0, ez = 0;
            while (sgpos < loc0 + nloc) {
              const u32 l = sgpos;
              bool ok = true;
              if (!P.noise_uniform) ok = geo_accept(R.master, shot, sgj - 1, __ldg(tables + P.acc_off + l));
              if (ok) {
                const u64 lw = __ldg(locs + 2ull * l);
                noise_letter((u32)(lw >> 48) & 3, (u32)(lw >> 32) & 0xff, (u32)(lw >> 40) & 0xff,
                             (double)sgpick * 0x1.0p-53, ex, ez);
              }
              const GeoCand gc = geo_candidate(tables + P.geo_off, P.geo_len, P.geo_ilq, R.master, shot, sgj, l + 1);
              sgpos = gc.pos;
              sgpick = gc.pick;
              ++sgj;
            }
            if (ex | ez) lane_error(ex, ez, nrec, size);
          }
        }
      }
      pc += len;
      if (sst != ST_RUNNING) continue;
      sk = k;

      // @region narrow: T
      if (kind == OP_T) {
        s_lo ^= __ldg(op + 1);
        s_hi ^= __ldg(op + 2);
        const u32 flip = par64(s_lo & __ldg(op + 3)) ^ par64(s_hi & __ldg(op + 4));
        const u64 delta = __ldg(op + 5);
        const u64 w6 = __ldg(op + 6);
        const u32 cb = (u32)w6, dmask = (u32)(w6 >> 32);
        const double2 a = make_double2(dbits(__ldg(op + 7)), dbits(__ldg(op + 8)));
        const double2 bxs = make_double2(dbits(__ldg(op + 9)), dbits(__ldg(op + 10)));
        smb += __ldg(op + 11);
        const double2 bx0 = flip ? cneg(bxs) : bxs;
        const double2 bx1 = cneg(bx0);
        const u32 dc = par64(delta & sc);
        const u32 tcase = fl & 3u;
        if (tcase == T_DIAG) {
          // beta == 0: pure phase per entry (ref state.py:120-126)
          const double2 f0 = cadd(a, bx0), f1 = cadd(a, bx1);
#pragma unroll 1
          for (u32 j = 0; j < size; ++j) AN(j) = cmul(AN(j), (dc ^ par32(j & dmask)) ? f1 : f0);
          smb += 32ull * scnt;
          continue;
        }
        // beta != 0: pair merge + prune (ref state.py:127-129, 294-306)
        const u32 cin = scnt;
        u32 nz = 0;
        if (tcase == T_BUTTERFLY) {
          const u32 hb = 31 - __clz(cb);
#pragma unroll 1
          for (u32 m = 0; m < (size >> 1); ++m) {
            const u32 j0 = ins_bit(m, hb, 0), j1 = j0 ^ cb;
            const double2 v0 = AN(j0), v1 = AN(j1);
            const u32 s0 = dc ^ par32(j0 & dmask), s1 = dc ^ par32(j1 & dmask);
            const double2 n0 = prune(cadd(cmul(a, v0), cmul(s1 ? bx1 : bx0, v1)));
            const double2 n1 = prune(cadd(cmul(a, v1), cmul(s0 ? bx1 : bx0, v0)));
            AN(j0) = n0;
            AN(j1) = n1;
            nz += nonzero(n0) + nonzero(n1);
          }
        } else {
#pragma unroll 1
          for (u32 j = 0; j < size; ++j) {
            const double2 v = AN(j);
            const u32 sj = dc ^ par32(j & dmask);
            const double2 n0 = prune(cmul(a, v));
            const double2 n1 = prune(cmul(sj ? bx1 : bx0, v));
            AN(j) = n0;
            AN(size + j) = n1;
            nz += nonzero(n0) + nonzero(n1);
          }
          sk = k + 1;
        }
        scnt = nz;
        smb += (u64)kEntryBytes * (cin + nz);
        if ((u64)nz > R.cap) { sst = ST_OVERFLOW; saux = (int)instr; }
        else if (nz == 0) { sst = ST_CORRUPT; saux = (int)instr; }
        continue;
      }

      // @region narrow: meas
      if (kind == OP_MEAS) {
        s_lo ^= __ldg(op + 1);
        s_hi ^= __ldg(op + 2);
        const u32 mcase = fl & 3u;
        const u32 xi0 = (((fl >> 2) & 3u) + 2u * (par64(s_lo & __ldg(op + 3)) ^ par64(s_hi & __ldg(op + 4)))) & 3u;
        const u64 delta = __ldg(op + 5);
        const u64 w6 = __ldg(op + 6), w7 = __ldg(op + 7);
        const u32 dmask = (u32)w6, tmask = (u32)(w6 >> 32);
        const u32 cb = (u32)w7, t = (u32)(w7 >> 32) & 0xff, isq = (u32)(w7 >> 40) & 0xff;
        const u64 vec = __ldg(op + 8);
        const u64 w13 = __ldg(op + 13);
        const u32 slot = (u32)w13, udraw = (u32)(w13 >> 32);
        smb += __ldg(op + 17);
        const u32 dc = par64(delta & sc);
        // u < P+ with u in [0, 1-2^-53]: P+ >= 1 or P+ <= 0 decide without
        // drawing (exact); otherwise draw u (ref sampler.py:262, state.py:168)
        auto pick_plus = [&](double pplus) -> bool {
          if (pplus >= 1.0) return true;
          if (pplus <= 0.0) return false;
          return (double)draw53(seed, R.master, shot, udraw, philox) * 0x1.0p-53 < pplus;
        };
        const u32 cin = scnt;
        bool plus;
        u32 nz = 0;
        if (mcase == M_DET) {
          // beta == 0: filter by eigenvalue (ref state.py:162-176)
          const u32 neg0 = (xi0 >> 1) ^ dc;
          double sp = 0.0, sm = 0.0;
#pragma unroll 1
          for (u32 j = 0; j < size; ++j) {
            const double a2 = abs2(AN(j));
            if (neg0 ^ par32(j & dmask)) sm = __dadd_rn(sm, a2); else sp = __dadd_rn(sp, a2);
          }
          plus = pick_plus(sp);
          const double chosen = plus ? sp : __dsub_rn(1.0, sp);
          if (chosen < 1e-12) { sst = ST_CORRUPT; saux = (int)instr; continue; }
          const u32 want_neg = plus ? 0u : 1u;
          const double rs = inv_sqrt_norm(plus ? sp : sm);
          if (fl & MF_COMPACT) {
            const u32 tau = want_neg ^ neg0;
#pragma unroll 1
            for (u32 jp = 0; jp < (size >> 1); ++jp) {
              const u32 j0 = ins_bit(jp, isq, 0);
              const double2 v = cscale(AN(j0 | ((tau ^ par32(j0 & dmask)) << isq)), rs);
              AN(jp) = v;
              nz += nonzero(v);
            }
            if (tau) sc ^= vec;
            sk = k - 1;
          } else {
#pragma unroll 1
            for (u32 j = 0; j < size; ++j) {
              const bool keep = (neg0 ^ par32(j & dmask)) == want_neg;
              const double2 v = keep ? cscale(AN(j), rs) : Z;
              AN(j) = v;
              nz += nonzero(v);
            }
          }
        } else {
          // beta != 0: pair-merge + tableau pivot (ref state.py:178-208)
          const double2 xpp = ipow(xi0);
          const double2 xpm = cneg(xpp);
          const u32 ct = (u32)(sc >> t) & 1u;
          const bool span = mcase == M_PIVOT_SPAN;
          const u32 npairs = span ? (size >> 1) : size;
          double sp = 0.0;
#pragma unroll 1
          for (u32 m = 0; m < npairs; ++m) {
            double2 wpv;
            if (span) {
              const u32 j0 = ins_bit(m, isq, 0);
              const u32 rep = j0 | ((ct ^ par32(j0 & tmask)) << isq);
              const u32 part = rep ^ cb;
              wpv = cadd(AN(rep), cmul((dc ^ par32(part & dmask)) ? xpm : xpp, AN(part)));
            } else {
              const double2 v = AN(m);
              wpv = (ct ^ par32(m & tmask)) ? cadd(Z, cmul((dc ^ par32(m & dmask)) ? xpm : xpp, v)) : v;
            }
            sp = __dadd_rn(sp, abs2(wpv));
          }
          const double pp = __dmul_rn(0.5, sp);
          plus = pick_plus(pp);
          const double chosen = plus ? pp : __dsub_rn(1.0, pp);
          if (chosen < 1e-12) { sst = ST_CORRUPT; saux = (int)instr; continue; }
          double sk2 = 0.0;
#pragma unroll 1
          for (u32 m = 0; m < npairs; ++m) {
            double2 w;
            u32 dst;
            if (span) {
              const u32 j0 = ins_bit(m, isq, 0);
              const u32 rep = j0 | ((ct ^ par32(j0 & tmask)) << isq);
              const u32 part = rep ^ cb;
              const double2 prod = cmul((dc ^ par32(part & dmask)) ? xpm : xpp, AN(part));
              w = plus ? cadd(AN(rep), prod) : csub(AN(rep), prod);
              dst = rep;
            } else {
              const double2 v = AN(m);
              if (ct ^ par32(m & tmask)) {
                const double2 prod = cmul((dc ^ par32(m & dmask)) ? xpm : xpp, v);
                w = plus ? cadd(Z, prod) : csub(Z, prod);
              } else {
                w = v;
              }
              dst = m;
            }
            w = prune(w);
            AN(dst) = w;
            sk2 = __dadd_rn(sk2, abs2(w));
            nz += nonzero(w);
          }
          if (nz == 0) { sst = ST_CORRUPT; saux = (int)instr; continue; }
          const double rs = inv_sqrt_norm(sk2);
          if (span) {
#pragma unroll 1
            for (u32 jp = 0; jp < (size >> 1); ++jp) {
              const u32 j0 = ins_bit(jp, isq, 0);
              AN(jp) = cscale(AN(j0 | ((ct ^ par32(j0 & tmask)) << isq)), rs);
            }
            sk = k - 1;
          } else {
#pragma unroll 1
            for (u32 j = 0; j < size; ++j) AN(j) = cscale(AN(j), rs);
          }
          if (ct) sc ^= vec;
          // tableau sign update of the pivot (ref tableau.py:176-200)
          const u32 v = (u32)(s_hi >> t) & 1u;
          if (v) { s_lo ^= __ldg(op + 9); s_hi ^= __ldg(op + 10); }
          s_lo ^= __ldg(op + 11);
          s_hi ^= __ldg(op + 12);
          s_lo = (s_lo & ~(1ull << t)) | ((u64)v << t);
          s_hi = (s_hi & ~(1ull << t)) | ((u64)(plus ? 0u : 1u) << t);
        }
        scnt = nz;
        smb += (u64)kEntryBytes * (cin + nz);
        const u32 bout = plus ? 0u : 1u;
        u32 rb = bout;
        if ((fl & MF_FLIP) && draw53(seed, R.master, shot, udraw + 1, philox) < __ldg(op + 14)) rb ^= 1u;
        if ((fl & MF_RECORD) && rb) recb[(slot >> 5) * 32u + lane] |= 1u << (slot & 31);
        if ((fl & MF_RESET) && bout) { s_lo ^= __ldg(op + 15); s_hi ^= __ldg(op + 16); }
        continue;
      }

      // @region narrow: feedback/detector/end
      if (kind == OP_FEEDBACK) {
        const u32 idx = (u32)__ldg(op + 1);
        if ((recb[(idx >> 5) * 32u + lane] >> (idx & 31)) & 1u) {
          s_lo ^= __ldg(op + 2);
          s_hi ^= __ldg(op + 3);
          smb += __ldg(op + 4);
        }
        continue;
      }

      if (kind == OP_DETECTOR || kind == OP_OBSERVABLE) {
        const u64 w1 = __ldg(op + 1);
        const u32 id = (u32)w1, nidx = (u32)(w1 >> 32);
        const u64 off = __ldg(op + 2);
        u32 parity = 0;
#pragma unroll 1
        for (u32 i = 0; i < nidx; ++i) {
          const u32 idx = (u32)__ldg(tables + off + i);
          parity ^= (recb[(idx >> 5) * 32u + lane] >> (idx & 31)) & 1u;
        }
        if (kind == OP_DETECTOR) {
          if ((R.flags & GS_POSTSELECT) && parity) { sst = ST_DISCARDED; saux = (int)id; }
        } else {
          sobs ^= (u64)parity << id;
        }
        continue;
      }

      if (kind == OP_END) {
        s_lo ^= __ldg(op + 1);
        s_hi ^= __ldg(op + 2);
        smb += __ldg(op + 3);
        sst = ST_PRESERVED;
        continue;
      }
      sst = ST_UNSUPPORTED;  // unknown opcode: fail loudly
      saux = -2;
    }
    __syncwarp();

    // @region narrow: outputs
    // survivors go to the next (wide) section's queue, in lane order
    const u32 run = __ballot_sync(FULL, valid && sst == ST_RUNNING);
    if (run) {
      u32 o = 0;
      if (lane == 0) o = atomicAdd(S.n_out, (u32)__popc(run));
      o = __shfl_sync(FULL, o, 0);
      if ((run >> lane) & 1u) {
        u64 *q = S.q_out + (u64)(o + __popc(run & lanemask_lt(lane))) * SU;
        q[Q_SL] = sl; q[Q_LO] = s_lo; q[Q_HI] = s_hi; q[Q_C] = sc; q[Q_OBS] = sobs;
        q[Q_MB] = smb; q[Q_PICK] = sgpick; q[Q_SEED] = seed;
        q[Q_CNTK] = (u64)scnt;
        q[Q_GEO] = (u64)sgj | ((u64)sgpos << 32);
        q[Q_FIRE] = sfire;
        u32 *qr = reinterpret_cast<u32 *>(q + Q_HDR);
#pragma unroll 1
        for (u32 w = 0; w < P.rec_words32; ++w) qr[w] = recb[w * 32u + lane];
        double2 *qc = reinterpret_cast<double2 *>(q + Q_HDR + rec_u64(P.rec_words32));
#pragma unroll 1
        for (u32 j = 0; j < (1u << exit_k); ++j) qc[j] = AN(j);
      }
    }
    const bool fin = valid && sst != ST_RUNNING;
    {
      const u32 pres = __ballot_sync(FULL, fin && sst == ST_PRESERVED);
      const u32 errb = __ballot_sync(FULL, fin && sst == ST_PRESERVED && sobs != 0);
      const u32 disc = __ballot_sync(FULL, fin && sst == ST_DISCARDED);
      const u32 ovf = __ballot_sync(FULL, fin && sst == ST_OVERFLOW);
      const u32 cor = __ballot_sync(FULL, fin && sst == ST_CORRUPT);
      const u32 uns = __ballot_sync(FULL, fin && sst == ST_UNSUPPORTED);
      const u32 val = __ballot_sync(FULL, fin);
      u64 mb = fin ? smb : 0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mb += __shfl_xor_sync(FULL, mb, o);
      if (lane == 0) {
        wcnt[WC_TOT] += __popc(val);
        wcnt[WC_PRES] += __popc(pres);
        wcnt[WC_DISC] += __popc(disc);
        wcnt[WC_OVF] += __popc(ovf);
        wcnt[WC_COR] += __popc(cor);
        wcnt[WC_UNS] += __popc(uns);
        wcnt[WC_ERR] += __popc(errb);
        wcnt[WC_MB] += mb;
      }
    }
    if (fin) {
      if (sst == ST_PRESERVED && sobs) {
#pragma unroll 1
        for (u64 o = sobs; o; o &= o - 1)
          atomicAdd((unsigned long long *)&O.counters[GS_C_PER_OBS + (__ffsll((long long)o) - 1)], 1ull);
        if (O.witness) {
          const u32 wi = atomicAdd(O.witness_count, 1u);
          if (wi < O.witness_cap) O.witness[wi] = shot;
        }
      }
      if (O.mode != MODE_COUNTERS) {
        O.status[sl] = (u8)sst;
        O.aux[sl] = saux;
        O.obs[sl] = sobs;
        const u32 rw64 = (P.nmeas + 63) / 64;
#pragma unroll 1
        for (u32 w = 0; w < rw64; ++w) {
          const u32 lo = recb[(2 * w) * 32u + lane];
          const u32 hi = (2 * w + 1 < P.rec_words32) ? recb[(2 * w + 1) * 32u + lane] : 0u;
          O.rec[sl * rw64 + w] = ((u64)hi << 32) | lo;
        }
        if (O.mode == MODE_DUMP) {
          O.sig[2 * sl] = s_lo;
          O.sig[2 * sl + 1] = s_hi;
          O.cvec[sl] = sc;
          O.dim[sl] = sk;
          const u64 stride = 1ull << P.max_dim;
#pragma unroll 1
          for (u32 j = 0; j < (1u << sk); ++j) O.amps[sl * stride + j] = AN(j);
        }
      }
    }
    __syncwarp();
  }
#undef AN
  flush_counters(O, wcnt, lane);
}

// ---------------------------------------------------------------- wide

template <bool kSmemChi, bool kPhilox>
__global__ void __launch_bounds__(128, GS_WIDE_BLOCKS)
wide_kernel(DevProg P, DevRun R, DevOut O, DevSec S) {
  extern __shared__ __align__(16) u8 smem[];
  const u32 lane = threadIdx.x & 31u;
  const u32 wib = threadIdx.x >> 5;
  const u32 wpb = blockDim.x >> 5;
  const u64 gw = (u64)blockIdx.x * wpb + wib;
  u8 *mine = smem + (size_t)wib * O.warp_bytes;
  unsigned long long *wcnt = reinterpret_cast<unsigned long long *>(mine);
  u32 *win = reinterpret_cast<u32 *>(mine + kCntBytes);
  u32 *recw = O.rec_in_smem ? reinterpret_cast<u32 *>(mine + kCntBytes + kWinBytes)
                            : O.grec + gw * (u64)P.rec_words32;
  double2 *A = kSmemChi ? chi_ptr<true>(reinterpret_cast<double2 *>(mine + O.chi_off))
                        : O.gchi + gw * ((u64)1 << P.max_dim);
  const u32 n = P.n;
  const u64 *__restrict__ ops = P.ops;
  const u64 *__restrict__ tables = P.tables;
  const u64 *__restrict__ locs = P.locs;
  const double2 Z = make_double2(0.0, 0.0);
  constexpr bool philox = kPhilox;
  const bool wide_only = (R.flags & GS_WIDE_ONLY) != 0;
  const u32 sign_bytes = 2u * ((2u * n + 7u) / 8u);
  const u32 SU = slot_u64(P);
  (void)n;

  if (lane < WC_N) wcnt[lane] = 0;
  __syncwarp();
  const u64 total = S.q_in ? (u64)*S.n_in : S.count;

#pragma unroll 1
  for (;;) {
    // @region wide: shot setup
    u64 idx = 0;
    if (lane == 0) idx = atomicAdd(S.work, 1ull);
    idx = __shfl_sync(FULL, idx, 0);
    if (idx >= total) break;
    Rng rng;
    rng.philox = philox;
    rng.master = R.master;
    u64 sl, sig_lo = 0, sig_hi = 0, c = 0, obs = 0, mbytes = 0, gpick = 0;
    u32 cnt = 1, gj = 0, gpos = 0xFFFFFFFFu, fire_pc = 0xFFFFFFFFu;
    const u32 k = S.k0;
    // chi norm, kept as per-lane partial sums and reduced only when a
    // deterministic measurement needs it
    double nrm_l = 0.0;
    if (!S.q_in) {
      sl = S.first + idx;
      rng.shot = R.shot_begin + sl;
      rng.seed = 0;
      if (!philox) rng.seed = R.seeds ? R.seeds[sl] : sha1_seed(R.master, rng.shot);
#pragma unroll 1
      for (u32 w = lane; w < P.rec_words32; w += 32) recw[w] = 0;
      if (lane == 0) A[0] = make_double2(1.0, 0.0);
      nrm_l = lane == 0 ? 1.0 : 0.0;
      if (philox && P.geo_len > 1 && P.nlocs) {
        const GeoCand gc = geo_candidate(tables + P.geo_off, P.geo_len, P.geo_ilq, R.master, rng.shot, 0u, 0u);
        gpos = gc.pos;
        gpick = gc.pick;
        gj = 1;
        fire_pc = gpos < P.nlocs ? 0u : 0xFFFFFFFFu;
      }
    } else {
      const u64 *q = S.q_in + idx * SU;
      sl = q[Q_SL];
      rng.shot = R.shot_begin + sl;
      rng.seed = q[Q_SEED];
      sig_lo = q[Q_LO]; sig_hi = q[Q_HI]; c = q[Q_C]; obs = q[Q_OBS]; mbytes = q[Q_MB];
      gpick = q[Q_PICK];
      cnt = (u32)q[Q_CNTK];
      gj = (u32)q[Q_GEO]; gpos = (u32)(q[Q_GEO] >> 32);
      fire_pc = (u32)q[Q_FIRE];
      const u32 *qr = reinterpret_cast<const u32 *>(q + Q_HDR);
#pragma unroll 1
      for (u32 w = lane; w < P.rec_words32; w += 32) recw[w] = qr[w];
      // chi in, and its norm (same per-lane order + tree as a sum pass)
      const double2 *qc = reinterpret_cast<const double2 *>(q + Q_HDR + rec_u64(P.rec_words32));
#pragma unroll 1
      for (u32 j = lane; j < (1u << k); j += 32) {
        const double2 v = qc[j];
        A[j] = v;
        nrm_l = __dadd_rn(nrm_l, abs2(v));
      }
    }
    if (!philox) fire_pc = 0xFFFFFFFFu;
    u32 kcur = k;
    int status = ST_RUNNING, aux = -1;
    double ps = 1.0;        // renormalisation pending on A (see ldps)
    // SplitMix noise scan state: everything inserted before pc0 is applied
    u32 cursor = P.nlocs;
    if (S.nm0 < P.nnoise) cursor = (u32)__ldg(tables + P.noise_off + 4ull * S.nm0 + 1);
    u32 scanned = cursor >> 5, search_w = scanned;
    u32 next_word_pc = 0xFFFFFFFFu;
    if (!philox && scanned < P.nwords) next_word_pc = (u32)__ldg(tables + P.wordpc_off + scanned);
    __syncwarp();
    u32 wpc = S.pc0;
    u64 hnext = __ldg(ops + wpc);
    u32 exit_pc = 0xFFFFFFFFu;
#pragma unroll 1
    while (status == ST_RUNNING) {
      if (!wide_only) {
        const u32 kind_ = (u32)(hnext & 0xff), k_ = (u32)((hnext >> 16) & 0xff),
                  fl_ = (u32)((hnext >> 24) & 0xff);
        if (!op_is_wide(kind_, k_, fl_)) { exit_pc = wpc; break; }
      }
      // @region wide: noise
      if (wpc >= next_word_pc || wpc >= fire_pc) {
        // apply E = OR of fired letters of one noise instruction
        // (ref noise.py:68-100, state.py:88-102)
        auto apply_error = [&](u64 ex, u64 ez, const u64 *nrec) {
          if (!(ex | ez)) return;
          const ErrAct e = compose_error(tables, ex, ez, __ldg(nrec + 2), __ldg(nrec + 3),
                                         sig_lo, sig_hi);
          const double2 php = ipow(e.xi);
          sweep_phase<kSmemChi>(A, 1u << kcur, par64(e.delt & c), e.dm, php, cneg(php), ps);
          ps = 1.0;
          __syncwarp();
          c ^= e.beta;
          mbytes += 2ull * kEntryBytes * cnt + sign_bytes;
        };
        if (philox) {
          // walk the candidate schedule (lane-uniform, rare)
          fire_pc = 0xFFFFFFFFu;
          while (gpos < P.nlocs) {
            const u64 *nrec = noise_owner(P, gpos);
            const u64 nw0 = __ldg(nrec);
            const u32 ipc = (u32)nw0, nloc = (u32)(nw0 >> 32);
            if (ipc > wpc) { fire_pc = ipc; break; }
            const u32 loc0 = (u32)__ldg(nrec + 1);
            u64 ex = 0, ez = 0;
            while (gpos < loc0 + nloc) {
              const u32 l = gpos;
              bool ok = true;
              if (!P.noise_uniform) ok = geo_accept(R.master, rng.shot, gj - 1, __ldg(tables + P.acc_off + l));
              if (ok) {
                const u64 lw = __ldg(locs + 2ull * l);
                noise_letter((u32)(lw >> 48) & 3, (u32)(lw >> 32) & 0xff, (u32)(lw >> 40) & 0xff,
                             (double)gpick * 0x1.0p-53, ex, ez);
              }
              const GeoCand gc = geo_candidate(tables + P.geo_off, P.geo_len, P.geo_ilq, R.master, rng.shot, gj, l + 1);
              gpos = gc.pos;
              gpick = gc.pick;
              ++gj;
            }
            apply_error(ex, ez, nrec);
          }
        } else {
          // SplitMix: one fire draw per location, 32 locations per ballot
          while (scanned < P.nwords && __ldg(tables + P.wordpc_off + scanned) <= wpc) {
            const u32 l = scanned * 32u + lane;
            bool fire = false;
            if (l < P.nlocs) {
              const u64 lw = __ldg(locs + 2ull * l), thr = __ldg(locs + 2ull * l + 1);
              fire = rng.m53((u32)lw) < thr;
            }
            const u32 bits = __ballot_sync(FULL, fire);
            if (lane == 0) win[scanned & (kWinWords - 1)] = bits;
            ++scanned;
          }
          __syncwarp();
          next_word_pc = scanned < P.nwords ? (u32)__ldg(tables + P.wordpc_off + scanned) : 0xFFFFFFFFu;
          fire_pc = 0xFFFFFFFFu;
#pragma unroll 1
          for (;;) {
            // next fired location >= cursor among the scanned words
            u32 fl_loc = 0xFFFFFFFFu;
            u32 w = max(search_w, cursor >> 5);
#pragma unroll 1
            for (; w < scanned; ++w) {
              u32 bits = win[w & (kWinWords - 1)];
              if (w == (cursor >> 5)) bits &= ~0u << (cursor & 31);
              if (bits) { fl_loc = w * 32u + (__ffs(bits) - 1); break; }
            }
            search_w = w;
            if (fl_loc == 0xFFFFFFFFu) break;
            const u64 *nrec = noise_owner(P, fl_loc);
            const u64 nw0 = __ldg(nrec);
            const u32 ipc = (u32)nw0, nloc = (u32)(nw0 >> 32);
            if (ipc > wpc) { fire_pc = ipc; break; }
            const u32 loc0 = (u32)__ldg(nrec + 1);
            cursor = loc0 + nloc;
            u64 ex = 0, ez = 0;
#pragma unroll 1
            for (u32 i = lane; i < nloc; i += 32) {
              const u32 l = loc0 + i;
              if (!((win[(l >> 5) & (kWinWords - 1)] >> (l & 31)) & 1u)) continue;
              const u64 lw = __ldg(locs + 2ull * l);
              const u32 nk = (u32)(lw >> 48) & 3;
              const double u = nk <= NK_DEP2 ? rng.uniform((u32)lw + 1) : 0.0;
              noise_letter(nk, (u32)(lw >> 32) & 0xff, (u32)(lw >> 40) & 0xff, u, ex, ez);
            }
            apply_error(warp_or64(ex), warp_or64(ez), nrec);
          }
        }
      }

      // @region wide: dispatch
      const u64 *op = ops + wpc;
      const u64 hw = hnext;
      const u32 wkind = (u32)(hw & 0xff), wlen = (u32)((hw >> 8) & 0xff);
      const u32 wk = (u32)((hw >> 16) & 0xff), wfl = (u32)((hw >> 24) & 0xff);
      const u32 winstr = (u32)(hw >> 32);
      wpc += wlen;
      hnext = __ldg(ops + wpc);       // prefetch the next header
      kcur = wk;
      const u32 size = 1u << wk;

      // @region wide: T
      if (wkind == OP_T || wkind == OP_GROW_LIMIT) {
        sig_lo ^= __ldg(op + 1);
        sig_hi ^= __ldg(op + 2);
        // xi0 = xi_s + 2 par(sigma & M); b * i^{xi0} is the host constant
        // b * i^{xi_s} (an exact swap/negation of b), negated when par = 1
        const u32 flip = par64(sig_lo & __ldg(op + 3)) ^ par64(sig_hi & __ldg(op + 4));
        const u64 delta = __ldg(op + 5);
        const u64 w6 = __ldg(op + 6);
        const u32 cb = (u32)w6, dmask = (u32)(w6 >> 32);
        const double2 a = make_double2(dbits(__ldg(op + 7)), dbits(__ldg(op + 8)));
        const double2 bxs = make_double2(dbits(__ldg(op + 9)), dbits(__ldg(op + 10)));
        mbytes += __ldg(op + 11);
        const double2 bx0 = flip ? cneg(bxs) : bxs;
        const u32 dc = par64(delta & c);
        const u32 tcase = wfl & 3u;
        if (tcase == T_DIAG) {
          // beta == 0: pure phase per entry (ref state.py:120-126); the
          // factors have modulus 1, the norm is kept
          sweep_phase<kSmemChi>(A, size, dc, dmask, cadd(a, bx0), cadd(a, cneg(bx0)), ps);
          ps = 1.0;
          __syncwarp();
          mbytes += 32ull * cnt;
          continue;
        }
        const u32 cin = cnt;
        if (wkind == OP_GROW_LIMIT) {
          u32 nz = 0;
          const double2 bx1 = cneg(bx0);
#pragma unroll 1
          for (u32 j = lane; j < size; j += 32) {
            const double2 v = ldps(A, j, ps);
            const u32 s_ = dc ^ par32(j & dmask);
            nz += abs2(cadd(Z, cmul(a, v))) > kPrune2;
            nz += abs2(cadd(Z, cmul(s_ ? bx1 : bx0, v))) > kPrune2;
          }
          nz = warp_sum_u32(nz);
          status = (u64)nz > R.cap ? ST_OVERFLOW : ST_UNSUPPORTED;
          aux = (int)winstr;
          break;
        }
        // beta != 0: pair merge + prune (ref state.py:127-129, 294-306)
        if (ps != 1.0) sweep_scale<kSmemChi>(A, size, ps);   // rare: right after a deferral
        ps = 1.0;
        if (tcase == T_BUTTERFLY && (wfl & TF_FUSE)) {
          // this gate and the next one (also a BUTTERFLY at the same k, no
          // noise between) in one pass
          const u64 *op2 = ops + wpc;
          const u64 h2 = hnext;
          const u32 instr2 = (u32)(h2 >> 32);
          sig_lo ^= __ldg(op2 + 1);
          sig_hi ^= __ldg(op2 + 2);
          const u32 flip2 = par64(sig_lo & __ldg(op2 + 3)) ^ par64(sig_hi & __ldg(op2 + 4));
          const u64 w62 = __ldg(op2 + 6);
          Gate g1, g2;
          g1.a = a; g1.bx0 = bx0; g1.cb = cb; g1.dc = dc; g1.dmask = dmask;
          g2.a = make_double2(dbits(__ldg(op2 + 7)), dbits(__ldg(op2 + 8)));
          const double2 bxs2 = make_double2(dbits(__ldg(op2 + 9)), dbits(__ldg(op2 + 10)));
          g2.bx0 = flip2 ? cneg(bxs2) : bxs2;
          g2.cb = (u32)w62;
          g2.dmask = (u32)(w62 >> 32);
          g2.dc = par64(__ldg(op2 + 5) & c);
          mbytes += __ldg(op2 + 11);
          wpc += (u32)((h2 >> 8) & 0xff);
          hnext = __ldg(ops + wpc);
          const SumNz2 r2 = sweep_butterfly2<kSmemChi>(A, size >> 2, g1, g2);
          __syncwarp();
          const u32 cnt1 = warp_sum_u32(r2.nz1);
          mbytes += (u64)kEntryBytes * (cin + cnt1);
          if ((u64)cnt1 > R.cap) { status = ST_OVERFLOW; aux = (int)winstr; break; }
          if (cnt1 == 0) { status = ST_CORRUPT; aux = (int)winstr; break; }
          cnt = warp_sum_u32(r2.nz);
          nrm_l = r2.sum;
          mbytes += (u64)kEntryBytes * (cnt1 + cnt);
          if ((u64)cnt > R.cap) { status = ST_OVERFLOW; aux = (int)instr2; break; }
          if (cnt == 0) { status = ST_CORRUPT; aux = (int)instr2; break; }
          continue;
        }
        SumNz r;
        if (tcase == T_BUTTERFLY) {
          r = sweep_butterfly<kSmemChi>(A, size >> 1, cb, dc, dmask, a, bx0);
        } else {
          r = sweep_grow<kSmemChi>(A, size, dc, dmask, a, bx0);
          kcur = wk + 1;
        }
        __syncwarp();
        cnt = warp_sum_u32(r.nz);
        nrm_l = r.sum;
        mbytes += (u64)kEntryBytes * (cin + cnt);
        if ((u64)cnt > R.cap) { status = ST_OVERFLOW; aux = (int)winstr; break; }
        if (cnt == 0) { status = ST_CORRUPT; aux = (int)winstr; break; }
        continue;
      }

      // @region wide: meas
      if (wkind == OP_MEAS) {
        sig_lo ^= __ldg(op + 1);
        sig_hi ^= __ldg(op + 2);
        const u32 mcase = wfl & 3u;
        const u32 xi0 = (((wfl >> 2) & 3u) + 2u * (par64(sig_lo & __ldg(op + 3)) ^ par64(sig_hi & __ldg(op + 4)))) & 3u;
        const u64 delta = __ldg(op + 5);
        const u64 w6 = __ldg(op + 6), w7 = __ldg(op + 7);
        const u32 dmask = (u32)w6, tmask = (u32)(w6 >> 32);
        const u32 cb = (u32)w7, t = (u32)(w7 >> 32) & 0xff, isq = (u32)(w7 >> 40) & 0xff;
        const u64 vec = __ldg(op + 8);
        const u64 w13 = __ldg(op + 13);
        const u32 slot = (u32)w13, udraw = (u32)(w13 >> 32);
        mbytes += __ldg(op + 17);
        const u32 dc = par64(delta & c);
        // u < P+ with u in [0, 1-2^-53]: P+ >= 1 or P+ <= 0 decide without
        // drawing (exact); otherwise draw u (ref sampler.py:262, state.py:168)
        auto pick_plus = [&](double pplus) -> bool {
          if (pplus >= 1.0) return true;
          if (pplus <= 0.0) return false;
          return rng.uniform(udraw) < pplus;
        };
        // a renormalisation by rs that needs no data movement: deferred to
        // the next pass over chi (ldps); nonzero count unchanged
        auto defer_scale = [&](double rs, double kept) {
          if (ps != 1.0) sweep_scale<kSmemChi>(A, size, ps);
          ps = rs;
          nrm_l = lane == 0 ? __dmul_rn(__dmul_rn(kept, rs), rs) : 0.0;
        };
        const u32 cin = cnt;
        bool plus;
        if (mcase == M_DET) {
          // beta == 0: filter by eigenvalue (ref state.py:162-176)
          const u32 neg0 = (xi0 >> 1) ^ dc;
          double sp, sm;
          if (dmask == 0) {
            // every coordinate has eigenvalue (-1)^neg0: P+ is the norm
            const double nrm = warp_sum(nrm_l);
            sp = neg0 ? 0.0 : nrm;
            sm = neg0 ? nrm : 0.0;
          } else {
            const double2 part = sweep_det_sums<kSmemChi>(A, size, dmask, neg0, ps);
            sp = warp_sum(part.x);
            sm = warp_sum(part.y);
          }
          plus = pick_plus(sp);
          const double chosen = plus ? sp : __dsub_rn(1.0, sp);
          if (chosen < 1e-12) { status = ST_CORRUPT; aux = (int)winstr; break; }
          const u32 want_neg = plus ? 0u : 1u;
          const double rs = inv_sqrt_norm(plus ? sp : sm);
          if (wfl & MF_COMPACT) {
            const u32 tau = want_neg ^ neg0;
            const SumNz r = sweep_compact<kSmemChi>(A, size >> 1, isq, dmask, tau, rs, ps);
            ps = 1.0;
            __syncwarp();
            cnt = warp_sum_u32(r.nz);
            nrm_l = r.sum;
            if (tau) c ^= vec;
            kcur = wk - 1;
          } else if ((plus ? sm : sp) == 0.0) {
            // the other eigenspace is empty: the filter is a pure
            // renormalisation
            defer_scale(rs, plus ? sp : sm);
          } else {
            const SumNz r = sweep_filter<kSmemChi>(A, size, dmask, neg0, want_neg, rs, ps);
            ps = 1.0;
            __syncwarp();
            cnt = warp_sum_u32(r.nz);
            nrm_l = r.sum;
          }
        } else {
          // beta != 0: pair-merge + tableau pivot (ref state.py:178-208)
          PivotGeo g;
          g.span = mcase == M_PIVOT_SPAN;
          g.npairs = g.span ? (size >> 1) : size;
          g.isq = isq; g.tmask = tmask; g.ct = (u32)(c >> t) & 1u; g.cb = cb;
          g.dc = dc; g.dmask = dmask;
          const double2 xpp = ipow(xi0);   // i^xi0, exact
          const double pp = __dmul_rn(0.5, warp_sum(sweep_pivot_p<kSmemChi>(A, g, xpp, ps)));
          plus = pick_plus(pp);
          const double chosen = plus ? pp : __dsub_rn(1.0, pp);
          if (chosen < 1e-12) { status = ST_CORRUPT; aux = (int)winstr; break; }
          const SumNz w = sweep_pivot_w<kSmemChi>(A, g, xpp, plus, ps);
          ps = 1.0;
          __syncwarp();
          const double sk = warp_sum(w.sum);
          cnt = warp_sum_u32(w.nz);
          if (cnt == 0) { status = ST_CORRUPT; aux = (int)winstr; break; }
          const double rs = inv_sqrt_norm(sk);
          if (g.span) {
            const SumNz r = sweep_compact<kSmemChi>(A, size >> 1, isq, tmask, g.ct, rs, 1.0);
            __syncwarp();
            cnt = warp_sum_u32(r.nz);
            nrm_l = r.sum;
            kcur = wk - 1;
          } else {
            defer_scale(rs, sk);
          }
          if (g.ct) c ^= vec;
          // tableau sign update of the pivot (ref tableau.py:176-200)
          const u32 v = (u32)(sig_hi >> t) & 1u;
          if (v) { sig_lo ^= __ldg(op + 9); sig_hi ^= __ldg(op + 10); }
          sig_lo ^= __ldg(op + 11);
          sig_hi ^= __ldg(op + 12);
          sig_lo = (sig_lo & ~(1ull << t)) | ((u64)v << t);
          sig_hi = (sig_hi & ~(1ull << t)) | ((u64)(plus ? 0u : 1u) << t);
        }
        mbytes += (u64)kEntryBytes * (cin + cnt);
        const u32 bout = plus ? 0u : 1u;
        u32 rb = bout;
        if ((wfl & MF_FLIP) && rng.m53(udraw + 1) < __ldg(op + 14)) rb ^= 1u;
        if (wfl & MF_RECORD) {
          if (lane == 0 && rb) recw[slot >> 5] |= 1u << (slot & 31);
          __syncwarp();
        }
        if ((wfl & MF_RESET) && bout) { sig_lo ^= __ldg(op + 15); sig_hi ^= __ldg(op + 16); }
        continue;
      }

      // @region wide: feedback/detector/end
      if (wkind == OP_FEEDBACK) {
        const u32 idx = (u32)__ldg(op + 1);
        if ((recw[idx >> 5] >> (idx & 31)) & 1u) {
          sig_lo ^= __ldg(op + 2);
          sig_hi ^= __ldg(op + 3);
          mbytes += __ldg(op + 4);
        }
        continue;
      }
      if (wkind == OP_DETECTOR || wkind == OP_OBSERVABLE) {
        const u64 w1 = __ldg(op + 1);
        const u32 id = (u32)w1, nidx = (u32)(w1 >> 32);
        const u64 off = __ldg(op + 2);
        u32 bb = 0;
#pragma unroll 1
        for (u32 i = lane; i < nidx; i += 32) {
          const u32 idx = (u32)__ldg(tables + off + i);
          bb ^= (recw[idx >> 5] >> (idx & 31)) & 1u;
        }
        const u32 parity = __popc(__ballot_sync(FULL, bb)) & 1u;
        if (wkind == OP_DETECTOR) {
          if ((R.flags & GS_POSTSELECT) && parity) { status = ST_DISCARDED; aux = (int)id; }
        } else {
          obs ^= (u64)parity << id;
        }
        continue;
      }
      if (wkind == OP_END) {
        sig_lo ^= __ldg(op + 1);
        sig_hi ^= __ldg(op + 2);
        mbytes += __ldg(op + 3);
        status = ST_PRESERVED;
        break;
      }
      status = ST_UNSUPPORTED;  // unknown opcode: fail loudly
      aux = -2;
    }
    // @region wide: outputs
    __syncwarp();
    if (status == ST_RUNNING) {
      // survivor: hand it to the next (narrow) section's queue
      u32 o = 0;
      if (lane == 0) o = atomicAdd(S.n_out, 1u);
      o = __shfl_sync(FULL, o, 0);
      u64 *q = S.q_out + (u64)o * SU;
      if (lane == 0) {
        q[Q_SL] = sl; q[Q_LO] = sig_lo; q[Q_HI] = sig_hi; q[Q_C] = c; q[Q_OBS] = obs;
        q[Q_MB] = mbytes; q[Q_PICK] = gpick; q[Q_SEED] = rng.seed;
        q[Q_CNTK] = (u64)cnt;
        q[Q_GEO] = (u64)gj | ((u64)gpos << 32);
        q[Q_FIRE] = fire_pc;
      }
      u32 *qr = reinterpret_cast<u32 *>(q + Q_HDR);
#pragma unroll 1
      for (u32 w = lane; w < P.rec_words32; w += 32) qr[w] = recw[w];
      double2 *qc = reinterpret_cast<double2 *>(q + Q_HDR + rec_u64(P.rec_words32));
#pragma unroll 1
      for (u32 j = lane; j < (1u << kcur); j += 32) qc[j] = ldps(A, j, ps);
      (void)exit_pc;
    } else {
      if (lane == 0) {
        wcnt[WC_TOT] += 1;
        wcnt[WC_MB] += mbytes;
        if (status == ST_PRESERVED) {
          wcnt[WC_PRES] += 1;
          if (obs) {
            wcnt[WC_ERR] += 1;
#pragma unroll 1
            for (u64 o = obs; o; o &= o - 1)
              atomicAdd((unsigned long long *)&O.counters[GS_C_PER_OBS + (__ffsll((long long)o) - 1)], 1ull);
            if (O.witness) {
              const u32 wi = atomicAdd(O.witness_count, 1u);
              if (wi < O.witness_cap) O.witness[wi] = rng.shot;
            }
          }
        } else if (status == ST_DISCARDED) wcnt[WC_DISC] += 1;
        else if (status == ST_OVERFLOW) wcnt[WC_OVF] += 1;
        else if (status == ST_CORRUPT) wcnt[WC_COR] += 1;
        else wcnt[WC_UNS] += 1;
      }
      if (O.mode != MODE_COUNTERS) {
        if (lane == 0) {
          O.status[sl] = (u8)status;
          O.aux[sl] = aux;
          O.obs[sl] = obs;
        }
        const u32 rw64 = (P.nmeas + 63) / 64;
#pragma unroll 1
        for (u32 w = lane; w < rw64; w += 32) {
          const u32 lo = recw[2 * w];
          const u32 hi = (2 * w + 1 < P.rec_words32) ? recw[2 * w + 1] : 0u;
          O.rec[sl * rw64 + w] = ((u64)hi << 32) | lo;
        }
        if (O.mode == MODE_DUMP) {
          if (lane == 0) {
            O.sig[2 * sl] = sig_lo;
            O.sig[2 * sl + 1] = sig_hi;
            O.cvec[sl] = c;
            O.dim[sl] = kcur;
          }
          const u64 stride = 1ull << P.max_dim;
#pragma unroll 1
          for (u32 j = lane; j < (1u << kcur); j += 32) O.amps[sl * stride + j] = ldps(A, j, ps);
        }
      }
    }
    __syncwarp();
  }
  flush_counters(O, wcnt, lane);
}

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

}  // namespace gs

// =================================================================== host

struct gs_program {
  gs_program_info info;
  std::vector<u64> ops, tables, locs;
  int dev = -1;
  u64 *d_ops = nullptr, *d_tables = nullptr, *d_locs = nullptr;
};

struct gs_engine {
  int device = 0;
  int num_sms = 0;
  size_t smem_optin = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  long long *d_counters = nullptr;
  size_t counters_cap = 0;
  double2 *d_chi = nullptr;
  size_t chi_bytes = 0;
  u32 *d_rec = nullptr;
  size_t rec_bytes = 0;
  u64 *d_queue[2] = {nullptr, nullptr};
  size_t queue_bytes[2] = {0, 0};
  unsigned long long *d_work = nullptr;
  size_t work_bytes = 0;
  u64 launches = 0;
  double last_ms = 0.0;
};

static thread_local std::string g_err;

static int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(x)                                                            \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess)                                                     \
      return fail(GS_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

extern "C" {

const char *gs_last_error(void) { return g_err.c_str(); }
int gs_abi_version(void) { return GS_ABI_VERSION; }

int gs_program_create(const gs_program_info *info, const uint64_t *ops, size_t n_ops,
                      const uint64_t *tables, size_t n_tables, const uint64_t *locs,
                      size_t n_locs, gs_program **out) {
  if (!info || !ops || !out || n_ops == 0) return fail(GS_ERR_ARG, "null argument");
  if (info->num_qubits < 1 || info->num_qubits > 64)
    return fail(GS_ERR_ARG, "num_qubits must be in 1..64");
  if (info->max_dim > 30) return fail(GS_ERR_ARG, "max_dim must be <= 30");
  if (info->num_obs > 64) return fail(GS_ERR_ARG, "at most 64 observables");
  if (info->num_noise && (!tables || info->noise_off + 4ull * info->num_noise > n_tables))
    return fail(GS_ERR_ARG, "noise table out of range");
  if (info->num_words && (!tables || info->wordpc_off + info->num_words > n_tables))
    return fail(GS_ERR_ARG, "word table out of range");
  if (info->geo_len < 1 || !tables || info->geo_off + info->geo_len > n_tables)
    return fail(GS_ERR_ARG, "geometric gap table out of range");
  if (!info->noise_uniform && info->num_locations &&
      info->acc_off + info->num_locations > n_tables)
    return fail(GS_ERR_ARG, "thinning table out of range");
  if (info->num_words != (info->num_locations + 31) / 32)
    return fail(GS_ERR_ARG, "num_words must be ceil(num_locations/32)");
  if (n_locs < 2ull * info->num_locations) return fail(GS_ERR_ARG, "locs too short");
  gs_program *p = new (std::nothrow) gs_program();
  if (!p) return fail(GS_ERR_NOMEM, "out of host memory");
  p->info = *info;
  p->ops.assign(ops, ops + n_ops);
  if (tables && n_tables) p->tables.assign(tables, tables + n_tables);
  else p->tables.assign(1, 0);
  if (locs && n_locs) p->locs.assign(locs, locs + n_locs);
  else p->locs.assign(2, 0);
  *out = p;
  return GS_OK;
}

int gs_program_destroy(gs_program *p) {
  if (!p) return GS_OK;
  if (p->dev >= 0) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(p->dev);
    cudaFree(p->d_ops);
    cudaFree(p->d_tables);
    cudaFree(p->d_locs);
    cudaSetDevice(cur);
  }
  delete p;
  return GS_OK;
}

int gs_engine_create(int device, gs_engine **out) {
  if (!out) return fail(GS_ERR_ARG, "null argument");
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(GS_ERR_ARG, "bad device index");
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(GS_ERR_UNSUPPORTED, "libgstab_sm100a requires an sm_100 (B200) device");
  gs_engine *e = new (std::nothrow) gs_engine();
  if (!e) return fail(GS_ERR_NOMEM, "out of host memory");
  e->device = device;
  e->num_sms = prop.multiProcessorCount;
  e->smem_optin = prop.sharedMemPerBlockOptin;
  CUDA_TRY(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreate(&e->ev0));
  CUDA_TRY(cudaEventCreate(&e->ev1));
  *out = e;
  return GS_OK;
}

int gs_engine_destroy(gs_engine *e) {
  if (!e) return GS_OK;
  cudaSetDevice(e->device);
  cudaFree(e->d_counters);
  cudaFree(e->d_chi);
  cudaFree(e->d_rec);
  cudaFree(e->d_queue[0]);
  cudaFree(e->d_queue[1]);
  cudaFree(e->d_work);
  if (e->ev0) cudaEventDestroy(e->ev0);
  if (e->ev1) cudaEventDestroy(e->ev1);
  if (e->stream) cudaStreamDestroy(e->stream);
  delete e;
  return GS_OK;
}

uint64_t gs_engine_launches(gs_engine *e) { return e ? e->launches : 0; }
double gs_engine_last_kernel_ms(gs_engine *e) { return e ? e->last_ms : 0.0; }

static int upload(gs_engine *e, gs_program *p) {
  if (p->dev == e->device) return GS_OK;
  if (p->dev >= 0) return fail(GS_ERR_ARG, "program already bound to another device");
  // one zero word past END: the interpreters prefetch the next header
  CUDA_TRY(cudaMalloc(&p->d_ops, (p->ops.size() + 1) * 8));
  CUDA_TRY(cudaMemset(p->d_ops + p->ops.size(), 0, 8));
  CUDA_TRY(cudaMalloc(&p->d_tables, p->tables.size() * 8));
  CUDA_TRY(cudaMalloc(&p->d_locs, p->locs.size() * 8));
  CUDA_TRY(cudaMemcpy(p->d_ops, p->ops.data(), p->ops.size() * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(p->d_tables, p->tables.data(), p->tables.size() * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(p->d_locs, p->locs.data(), p->locs.size() * 8, cudaMemcpyHostToDevice));
  p->dev = e->device;
  return GS_OK;
}

// static section split of the op stream (see the kernels' header comment)
struct Section {
  u32 pc0, k0, nm0;
  bool wide;
};

#ifndef GS_NARROW_SPLIT
#define GS_NARROW_SPLIT 75  // split narrow sections every N ops (0: never) so the survivors of
                            // early discards re-pack into full warps (A/B: 51.2M at 75, 49.4M unsplit,
                            // 50.6M at 150, 50.3M at 40)
#endif

static void sections_of(const gs_program *p, bool wide_only, std::vector<Section> &out) {
  out.clear();
  const std::vector<u64> &ops = p->ops;
  size_t pc = 0, nm = 0;
  u32 nops = 0;
  const u32 nn = p->info.num_noise;
  while (pc < ops.size()) {
    const u64 h = ops[pc];
    const u32 kind = (u32)(h & 0xff), len = (u32)((h >> 8) & 0xff);
    const u32 k = (u32)((h >> 16) & 0xff), fl = (u32)((h >> 24) & 0xff);
    const bool wide = wide_only || gs::op_is_wide(kind, k, fl);
    const bool split = !wide && (GS_NARROW_SPLIT > 0) && nops >= (u32)GS_NARROW_SPLIT;
    if (out.empty() || out.back().wide != wide || split) {
      while (nm < nn && (u32)p->tables[p->info.noise_off + 4 * nm] < (u32)pc) ++nm;
      out.push_back(Section{(u32)pc, k, (u32)nm, wide});
      nops = 0;
    }
    ++nops;
    if (kind == gs::OP_END || len == 0) break;
    pc += len;
  }
}

int gs_program_sections(const gs_program *p, uint32_t flags) {
  if (!p) return fail(GS_ERR_ARG, "null argument");
  std::vector<Section> secs;
  sections_of(p, (flags & GS_WIDE_ONLY) != 0, secs);
  return (int)secs.size();
}


extern "C++" {
// the sampling kernels: RNG mode (x chi placement for the wide kernel)
template <typename F>
static cudaError_t with_narrow_kernel(bool philox, F f) {
  return philox ? f(gs::narrow_kernel<true>) : f(gs::narrow_kernel<false>);
}
template <typename F>
static cudaError_t with_wide_kernel(bool smem_chi, bool philox, F f) {
  if (smem_chi) return philox ? f(gs::wide_kernel<true, true>) : f(gs::wide_kernel<true, false>);
  return philox ? f(gs::wide_kernel<false, true>) : f(gs::wide_kernel<false, false>);
}

struct KernelCfg {
  u32 wpb = 1, blocks = 1, warp_bytes = 0, chi_off = 0, rec_in_smem = 0;
  size_t smem = 0;
};

// warps per block = the most resident warps per SM; grid = SMs x blocks/SM
template <typename W>
static int occupancy(gs_engine *e, u32 warp_bytes, u32 want_wpb, W with, KernelCfg &K) {
  u32 wpb = 1;
  int best = -1;
  for (u32 w = 4; w >= 1; --w) {
    if (want_wpb && w != want_wpb) continue;
    if ((size_t)w * warp_bytes > e->smem_optin) continue;
    int per = 0;
    const size_t sm = (size_t)w * warp_bytes;
    CUDA_TRY(with([&](auto kern) {
      cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      return err != cudaSuccess ? err : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, w * 32, sm);
    }));
    if (per * (int)w > best) { best = per * (int)w; wpb = w; }
  }
  if (best < 1) return fail(GS_ERR_UNSUPPORTED, "per-warp state exceeds shared memory");
  K.wpb = wpb;
  K.warp_bytes = warp_bytes;
  K.smem = (size_t)wpb * warp_bytes;
  CUDA_TRY(with([&](auto kern) {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K.smem);
  }));
  K.blocks = (u32)(e->num_sms * (best / (int)wpb));
  return GS_OK;
}

template <typename T>
static int ensure_buf(T **d, size_t *cap, size_t want) {
  if (want <= *cap) return GS_OK;
  cudaFree(*d);
  *d = nullptr;
  *cap = 0;
  CUDA_TRY(cudaMalloc(d, want));
  *cap = want;
  return GS_OK;
}

}  // extern "C++"

static int launch(gs_engine *e, gs_program *p, const gs_run_params *r, gs::DevOut O,
                  cudaStream_t st, bool timed) {
  if (!e || !p || !r) return fail(GS_ERR_ARG, "null argument");
  if (r->capacity < 1) return fail(GS_ERR_ARG, "capacity must be >= 1");
  if ((r->flags & GS_RNG_PHILOX) && r->seeds)
    return fail(GS_ERR_ARG, "explicit seeds require the SplitMix RNG");
  CUDA_TRY(cudaSetDevice(e->device));
  int rc = upload(e, p);
  if (rc) return rc;
  const bool philox = (r->flags & GS_RNG_PHILOX) != 0;
  const bool wide_only = (r->flags & GS_WIDE_ONLY) != 0;
  gs::DevProg P;
  P.ops = p->d_ops;
  P.tables = p->d_tables;
  P.locs = p->d_locs;
  P.n = p->info.num_qubits;
  P.nmeas = p->info.num_measurements;
  P.max_dim = p->info.max_dim;
  P.nobs = p->info.num_obs;
  P.rec_words32 = ((p->info.num_measurements + 63) / 64) * 2;
  if (P.rec_words32 == 0) P.rec_words32 = 2;
  P.nlocs = p->info.num_locations;
  P.nnoise = p->info.num_noise;
  P.nwords = p->info.num_words;
  P.noise_off = p->info.noise_off;
  P.wordpc_off = p->info.wordpc_off;
  P.geo_off = p->info.geo_off;
  P.geo_len = p->info.geo_len;
  P.acc_off = p->info.acc_off;
  P.noise_uniform = p->info.noise_uniform;
  P.geo_ilq = 0.f;
  if (p->info.geo_len >= 2) {
    const double q = (double)p->tables[p->info.geo_off + 1] * 0x1.0p-53;
    if (q < 1.0) P.geo_ilq = (float)(1.0 / log(q));
  }
  gs::DevRun R;
  R.master = r->master_seed;
  R.shot_begin = r->shot_begin;
  R.shot_count = r->shot_count;
  R.cap = r->capacity;
  R.flags = r->flags;
  R.seeds = nullptr;

  std::vector<Section> secs;
  sections_of(p, wide_only, secs);
  bool any_narrow = false, any_wide = false;
  for (const Section &s : secs) (s.wide ? any_wide : any_narrow) = true;

  // launch shapes: narrow warps hold 32 shots' chi rows and record columns,
  // wide warps one shot's chi (shared memory when 2^max_dim entries fit)
  const size_t chi = (size_t)16 << P.max_dim;
  bool smem_chi;
  if (r->flags & GS_CHI_GLOBAL) smem_chi = false;
  else if (r->flags & GS_CHI_SMEM) smem_chi = chi <= 64 * 1024;
  else smem_chi = chi <= 32 * 1024;
  const size_t nrec_b = (size_t)P.rec_words32 * 4 * 32, wrec_b = (size_t)P.rec_words32 * 4;
  KernelCfg KN, KW;
  KN.rec_in_smem = nrec_b <= 4096;
  KW.rec_in_smem = wrec_b <= 4096;
  if (any_narrow) {
    const u32 wb = (u32)((gs::kCntBytes + gs::kNarrowBytes + (KN.rec_in_smem ? nrec_b : 0) + 15) & ~(size_t)15);
    rc = occupancy(e, wb, r->warps_per_block,
                   [&](auto f) { return with_narrow_kernel(philox, f); }, KN);
    if (rc) return rc;
  }
  if (any_wide) {
    size_t base = gs::kCntBytes + gs::kWinBytes + (KW.rec_in_smem ? ((wrec_b + 15) & ~(size_t)15) : 0);
    KW.chi_off = (u32)base;
    const u32 wb = (u32)(base + (smem_chi ? chi : 0));
    rc = occupancy(e, wb, r->warps_per_block,
                   [&](auto f) { return with_wide_kernel(smem_chi, philox, f); }, KW);
    if (rc) return rc;
    if (!smem_chi) {   // bound the global chi scratch
      const u64 max_warps = ((u64)8 << 30) / chi;
      if ((u64)KW.blocks * KW.wpb > max_warps) KW.blocks = (u32)std::max<u64>(1, max_warps / KW.wpb);
    }
  }
  if (r->blocks) { KN.blocks = r->blocks; KW.blocks = r->blocks; }
  const u64 nwarps = std::max((u64)KN.blocks * KN.wpb, (u64)KW.blocks * KW.wpb);
  if (!smem_chi && any_wide) {
    rc = ensure_buf(&e->d_chi, &e->chi_bytes, (size_t)KW.blocks * KW.wpb * chi);
    if (rc) return rc;
  }
  if (!KN.rec_in_smem || !KW.rec_in_smem) {
    rc = ensure_buf(&e->d_rec, &e->rec_bytes, (size_t)nwarps * nrec_b);
    if (rc) return rc;
  }
  // queues between sections: fixed slots, chunks of at most `chunk` shots
  const u64 slot_b = 8ull * (gs::Q_HDR + gs::rec_u64(P.rec_words32) + 2 * (1u << GS_KN));
  u64 chunk = r->shot_count ? r->shot_count : 1;
  const u64 qbudget = (u64)2 << 30;   // bytes per queue
  if (secs.size() > 1 && chunk * slot_b > qbudget) chunk = std::max<u64>(32, qbudget / slot_b);
  if (r->chunk_shots && r->chunk_shots < chunk) chunk = r->chunk_shots;   // tests
  if (secs.size() > 1) {
    rc = ensure_buf(&e->d_queue[0], &e->queue_bytes[0], (size_t)(chunk * slot_b));
    if (rc) return rc;
    rc = ensure_buf(&e->d_queue[1], &e->queue_bytes[1], (size_t)(chunk * slot_b));
    if (rc) return rc;
  }
  rc = ensure_buf(&e->d_work, &e->work_bytes, sizeof(unsigned long long) * (secs.size() + 2));
  if (rc) return rc;
  u32 *d_qn = reinterpret_cast<u32 *>(e->d_work + secs.size());   // two u32 queue lengths

  u64 *d_seeds = nullptr;
  if (r->seeds && r->shot_count) {
    CUDA_TRY(cudaMallocAsync(&d_seeds, r->shot_count * 8, st));
    CUDA_TRY(cudaMemcpyAsync(d_seeds, r->seeds, r->shot_count * 8, cudaMemcpyHostToDevice, st));
    R.seeds = d_seeds;
  }
  O.gchi = e->d_chi;
  O.grec = e->d_rec;
  if (r->shot_count) {
    if (timed) CUDA_TRY(cudaEventRecord(e->ev0, st));
    for (u64 first = 0; first < r->shot_count; first += chunk) {
      const u64 count = std::min(chunk, r->shot_count - first);
      CUDA_TRY(cudaMemsetAsync(e->d_work, 0, sizeof(unsigned long long) * (secs.size() + 2), st));
      for (size_t i = 0; i < secs.size(); ++i) {
        gs::DevSec S;
        S.pc0 = secs[i].pc0;
        S.k0 = secs[i].k0;
        S.nm0 = secs[i].nm0;
        S.pc_end = (i + 1 < secs.size() && !secs[i + 1].wide) ? secs[i + 1].pc0 : 0xFFFFFFFFu;
        S.first = first;
        S.count = count;
        S.q_in = i ? e->d_queue[(i - 1) & 1] : nullptr;
        S.n_in = i ? d_qn + ((i - 1) & 1) : nullptr;
        S.q_out = i + 1 < secs.size() ? e->d_queue[i & 1] : nullptr;
        S.n_out = d_qn + (i & 1);
        S.work = e->d_work + i;
        if (i >= 1 && i + 1 < secs.size())   // the queue written here was read by section i-1
          CUDA_TRY(cudaMemsetAsync(d_qn + (i & 1), 0, sizeof(u32), st));
        if (secs[i].wide) {
          gs::DevOut Ow = O;
          Ow.warp_bytes = KW.warp_bytes;
          Ow.rec_in_smem = KW.rec_in_smem;
          Ow.chi_off = KW.chi_off;
          CUDA_TRY(with_wide_kernel(smem_chi, philox, [&](auto kern) {
            kern<<<KW.blocks, KW.wpb * 32, KW.smem, st>>>(P, R, Ow, S);
            return cudaGetLastError();
          }));
        } else {
          gs::DevOut On = O;
          On.warp_bytes = KN.warp_bytes;
          On.rec_in_smem = KN.rec_in_smem;
          On.chi_off = 0;
          CUDA_TRY(with_narrow_kernel(philox, [&](auto kern) {
            kern<<<KN.blocks, KN.wpb * 32, KN.smem, st>>>(P, R, On, S);
            return cudaGetLastError();
          }));
        }
        e->launches += 1;
      }
    }
    if (timed) CUDA_TRY(cudaEventRecord(e->ev1, st));
  }
  if (d_seeds) CUDA_TRY(cudaFreeAsync(d_seeds, st));
  return GS_OK;
}

static int ensure_counters(gs_engine *e, size_t n) {
  if (n <= e->counters_cap) return GS_OK;
  cudaFree(e->d_counters);
  e->d_counters = nullptr;
  e->counters_cap = 0;
  CUDA_TRY(cudaMalloc(&e->d_counters, n * 8));
  e->counters_cap = n;
  return GS_OK;
}

static int run_counters_impl(gs_engine *e, gs_program *p, const gs_run_params *r,
                             int64_t *counters, uint64_t *witness, uint32_t witness_cap,
                             uint32_t *witness_count);

int gs_run_counters(gs_engine *e, gs_program *p, const gs_run_params *r, int64_t *counters) {
  return run_counters_impl(e, p, r, counters, nullptr, 0, nullptr);
}

int gs_run_counters_witness(gs_engine *e, gs_program *p, const gs_run_params *r,
                            int64_t *counters, uint64_t *witness, uint32_t witness_cap,
                            uint32_t *witness_count) {
  if (!witness || !witness_count) return fail(GS_ERR_ARG, "null argument");
  return run_counters_impl(e, p, r, counters, witness, witness_cap, witness_count);
}

static int run_counters_impl(gs_engine *e, gs_program *p, const gs_run_params *r,
                             int64_t *counters, uint64_t *witness, uint32_t witness_cap,
                             uint32_t *witness_count) {
  if (!e || !p || !r || !counters) return fail(GS_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(e->device));
  const size_t nc = GS_C_PER_OBS + p->info.num_obs;
  int rc = ensure_counters(e, nc);
  if (rc) return rc;
  CUDA_TRY(cudaMemsetAsync(e->d_counters, 0, nc * 8, e->stream));
  gs::DevOut O;
  memset(&O, 0, sizeof(O));
  O.counters = e->d_counters;
  O.mode = gs::MODE_COUNTERS;
  u64 *d_w = nullptr;
  u32 *d_wc = nullptr;
  if (witness) {
    CUDA_TRY(cudaMallocAsync(&d_w, (witness_cap ? witness_cap : 1) * 8ull, e->stream));
    CUDA_TRY(cudaMallocAsync(&d_wc, 4, e->stream));
    CUDA_TRY(cudaMemsetAsync(d_wc, 0, 4, e->stream));
    O.witness = d_w;
    O.witness_count = d_wc;
    O.witness_cap = witness_cap;
  }
  rc = launch(e, p, r, O, e->stream, true);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(counters, e->d_counters, nc * 8, cudaMemcpyDeviceToHost, e->stream));
  if (witness) {
    CUDA_TRY(cudaMemcpyAsync(witness_count, d_wc, 4, cudaMemcpyDeviceToHost, e->stream));
    if (witness_cap)
      CUDA_TRY(cudaMemcpyAsync(witness, d_w, witness_cap * 8ull, cudaMemcpyDeviceToHost, e->stream));
    cudaFreeAsync(d_w, e->stream);
    cudaFreeAsync(d_wc, e->stream);
  }
  CUDA_TRY(cudaStreamSynchronize(e->stream));
  float ms = 0.f;
  if (r->shot_count) CUDA_TRY(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
  e->last_ms = ms;
  return GS_OK;
}

int gs_run_counters_async(gs_engine *e, gs_program *p, const gs_run_params *r,
                          int64_t *counters_dev, void *stream) {
  if (!e || !p || !r || !counters_dev) return fail(GS_ERR_ARG, "null argument");
  gs::DevOut O;
  memset(&O, 0, sizeof(O));
  O.counters = (long long *)counters_dev;
  O.mode = gs::MODE_COUNTERS;
  return launch(e, p, r, O, (cudaStream_t)stream, false);
}

static int run_out(gs_engine *e, gs_program *p, const gs_run_params *r, uint8_t *status,
                   int32_t *aux, uint64_t *record_bits, uint64_t *obs_bits, uint64_t *sig,
                   uint64_t *cv, double *amps, uint32_t *dim, u32 mode) {
  if (!e || !p || !r || !status || !aux || !record_bits || !obs_bits)
    return fail(GS_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(e->device));
  const size_t nc = GS_C_PER_OBS + p->info.num_obs;
  int rc = ensure_counters(e, nc);
  if (rc) return rc;
  const u64 S = r->shot_count;
  const u64 rw = (p->info.num_measurements + 63) / 64;
  const u64 stride = 1ull << p->info.max_dim;
  gs::DevOut O;
  memset(&O, 0, sizeof(O));
  O.counters = e->d_counters;
  O.mode = mode;
  cudaStream_t st = e->stream;
  CUDA_TRY(cudaMemsetAsync(e->d_counters, 0, nc * 8, st));
  const size_t bytes_rec = (size_t)S * (rw ? rw : 1) * 8;
  CUDA_TRY(cudaMallocAsync(&O.status, S ? S : 1, st));
  CUDA_TRY(cudaMallocAsync(&O.aux, (S ? S : 1) * 4, st));
  CUDA_TRY(cudaMallocAsync(&O.rec, bytes_rec ? bytes_rec : 8, st));
  CUDA_TRY(cudaMallocAsync(&O.obs, (S ? S : 1) * 8, st));
  if (bytes_rec) CUDA_TRY(cudaMemsetAsync(O.rec, 0, bytes_rec, st));
  if (mode == gs::MODE_DUMP) {
    CUDA_TRY(cudaMallocAsync(&O.sig, (S ? S : 1) * 16, st));
    CUDA_TRY(cudaMallocAsync(&O.cvec, (S ? S : 1) * 8, st));
    CUDA_TRY(cudaMallocAsync(&O.dim, (S ? S : 1) * 4, st));
    CUDA_TRY(cudaMallocAsync(&O.amps, (S ? S : 1) * stride * 16, st));
    CUDA_TRY(cudaMemsetAsync(O.amps, 0, (S ? S : 1) * stride * 16, st));
  }
  rc = launch(e, p, r, O, st, true);
  if (rc) return rc;
  if (S) {
    CUDA_TRY(cudaMemcpyAsync(status, O.status, S, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(aux, O.aux, S * 4, cudaMemcpyDeviceToHost, st));
    if (rw) CUDA_TRY(cudaMemcpyAsync(record_bits, O.rec, bytes_rec, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(obs_bits, O.obs, S * 8, cudaMemcpyDeviceToHost, st));
    if (mode == gs::MODE_DUMP) {
      CUDA_TRY(cudaMemcpyAsync(sig, O.sig, S * 16, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaMemcpyAsync(cv, O.cvec, S * 8, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaMemcpyAsync(dim, O.dim, S * 4, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaMemcpyAsync(amps, O.amps, S * stride * 16, cudaMemcpyDeviceToHost, st));
    }
  }
  cudaFreeAsync(O.status, st);
  cudaFreeAsync(O.aux, st);
  cudaFreeAsync(O.rec, st);
  cudaFreeAsync(O.obs, st);
  if (mode == gs::MODE_DUMP) {
    cudaFreeAsync(O.sig, st);
    cudaFreeAsync(O.cvec, st);
    cudaFreeAsync(O.dim, st);
    cudaFreeAsync(O.amps, st);
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  float ms = 0.f;
  if (S) CUDA_TRY(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
  e->last_ms = ms;
  return GS_OK;
}

int gs_run_records(gs_engine *e, gs_program *p, const gs_run_params *r, uint8_t *status,
                   int32_t *aux, uint64_t *record_bits, uint64_t *obs_bits) {
  return run_out(e, p, r, status, aux, record_bits, obs_bits, nullptr, nullptr, nullptr,
                 nullptr, gs::MODE_RECORDS);
}

int gs_dump_shots(gs_engine *e, gs_program *p, const gs_run_params *r, uint8_t *status,
                  int32_t *aux, uint64_t *record_bits, uint64_t *obs_bits, uint64_t *sig,
                  uint64_t *c, double *amps, uint32_t *dim) {
  if (!sig || !c || !amps || !dim) return fail(GS_ERR_ARG, "null argument");
  return run_out(e, p, r, status, aux, record_bits, obs_bits, sig, c, amps, dim,
                 gs::MODE_DUMP);
}

}  // extern "C"

// ------------------------------------------------ kernel plugin API (host)

template <typename T>
static int to_dev(T **d, const void *h, size_t n, cudaStream_t st) {
  CUDA_TRY(cudaMallocAsync((void **)d, (n ? n : 1) * sizeof(T), st));
  if (n && h) CUDA_TRY(cudaMemcpyAsync(*d, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
  return GS_OK;
}

extern "C" {

int gs_anticommute_mask(gs_engine *e, const uint64_t *xs, const uint64_t *zs, uint32_t rows,
                        uint32_t batch, const uint64_t *qx, const uint64_t *qz,
                        uint64_t *out_mask) {
  if (!e || !xs || !zs || !qx || !qz || !out_mask) return fail(GS_ERR_ARG, "null argument");
  if (rows > 128) return fail(GS_ERR_ARG, "rows must be <= 128");
  CUDA_TRY(cudaSetDevice(e->device));
  cudaStream_t st = e->stream;
  u64 *dx, *dz, *dqx, *dqz, *dout;
  const size_t nr = (size_t)rows * batch;
  if (to_dev(&dx, xs, nr, st) || to_dev(&dz, zs, nr, st) || to_dev(&dqx, qx, batch, st) ||
      to_dev(&dqz, qz, batch, st) || to_dev(&dout, nullptr, 2 * (size_t)batch, st))
    return GS_ERR_CUDA;
  if (batch) {
    gs::anticommute_kernel<<<(batch + 3) / 4, 128, 0, st>>>(dx, dz, rows, batch, dqx, dqz, dout);
    CUDA_TRY(cudaGetLastError());
    e->launches += 1;
    CUDA_TRY(cudaMemcpyAsync((void *)out_mask, dout, 16 * (size_t)batch, cudaMemcpyDeviceToHost, st));
  }
  cudaFreeAsync(dx, st); cudaFreeAsync(dz, st); cudaFreeAsync(dqx, st);
  cudaFreeAsync(dqz, st); cudaFreeAsync(dout, st);
  CUDA_TRY(cudaStreamSynchronize(st));
  return GS_OK;
}

int gs_conj_gate_rows(gs_engine *e, uint64_t *xs, uint64_t *zs, uint8_t *ph, uint32_t rows,
                      uint32_t batch, const uint32_t *code, const uint64_t *m1,
                      const uint64_t *m2) {
  if (!e || !xs || !zs || !ph || !code || !m1 || !m2) return fail(GS_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(e->device));
  cudaStream_t st = e->stream;
  const size_t nr = (size_t)rows * batch;
  u64 *dx, *dz, *dm1, *dm2;
  u8 *dph;
  u32 *dcode;
  if (to_dev(&dx, xs, nr, st) || to_dev(&dz, zs, nr, st) ||
      to_dev(&dph, ph, nr, st) || to_dev(&dcode, code, batch, st) ||
      to_dev(&dm1, m1, batch, st) || to_dev(&dm2, m2, batch, st))
    return GS_ERR_CUDA;
  if (nr) {
    gs::conj_gate_kernel<<<(u32)((nr + 255) / 256), 256, 0, st>>>(dx, dz, dph, rows, batch, dcode, dm1, dm2);
    CUDA_TRY(cudaGetLastError());
    e->launches += 1;
    CUDA_TRY(cudaMemcpyAsync(xs, dx, nr * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(zs, dz, nr * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(ph, dph, nr, cudaMemcpyDeviceToHost, st));
  }
  cudaFreeAsync(dx, st); cudaFreeAsync(dz, st); cudaFreeAsync(dph, st);
  cudaFreeAsync(dcode, st); cudaFreeAsync(dm1, st); cudaFreeAsync(dm2, st);
  CUDA_TRY(cudaStreamSynchronize(st));
  return GS_OK;
}

int gs_mul_rows(gs_engine *e, uint64_t *xs, uint64_t *zs, uint8_t *ph, uint32_t rows,
                uint32_t batch, const uint8_t *sel, const uint64_t *px, const uint64_t *pz,
                const uint32_t *pe) {
  if (!e || !xs || !zs || !ph || !sel || !px || !pz || !pe) return fail(GS_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(e->device));
  cudaStream_t st = e->stream;
  const size_t nr = (size_t)rows * batch;
  u64 *dx, *dz, *dpx, *dpz;
  u8 *dph, *dsel;
  u32 *dpe;
  if (to_dev(&dx, xs, nr, st) || to_dev(&dz, zs, nr, st) ||
      to_dev(&dph, ph, nr, st) || to_dev(&dsel, sel, nr, st) ||
      to_dev(&dpx, px, batch, st) || to_dev(&dpz, pz, batch, st) || to_dev(&dpe, pe, batch, st))
    return GS_ERR_CUDA;
  if (nr) {
    gs::mul_rows_kernel<<<(u32)((nr + 255) / 256), 256, 0, st>>>(dx, dz, dph, rows, batch, dsel, dpx, dpz, dpe);
    CUDA_TRY(cudaGetLastError());
    e->launches += 1;
    CUDA_TRY(cudaMemcpyAsync(xs, dx, nr * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(zs, dz, nr * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(ph, dph, nr, cudaMemcpyDeviceToHost, st));
  }
  cudaFreeAsync(dx, st); cudaFreeAsync(dz, st); cudaFreeAsync(dph, st); cudaFreeAsync(dsel, st);
  cudaFreeAsync(dpx, st); cudaFreeAsync(dpz, st); cudaFreeAsync(dpe, st);
  CUDA_TRY(cudaStreamSynchronize(st));
  return GS_OK;
}

int gs_parity_pm(gs_engine *e, const uint64_t *idx, size_t count, uint64_t mask, double *out) {
  if (!e || (count && (!idx || !out))) return fail(GS_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(e->device));
  cudaStream_t st = e->stream;
  u64 *di;
  double *dout;
  if (to_dev(&di, idx, count, st) || to_dev(&dout, nullptr, count, st))
    return GS_ERR_CUDA;
  if (count) {
    gs::parity_pm_kernel<<<(u32)((count + 255) / 256), 256, 0, st>>>(di, count, mask, dout);
    CUDA_TRY(cudaGetLastError());
    e->launches += 1;
    CUDA_TRY(cudaMemcpyAsync(out, dout, count * 8, cudaMemcpyDeviceToHost, st));
  }
  cudaFreeAsync(di, st);
  cudaFreeAsync(dout, st);
  CUDA_TRY(cudaStreamSynchronize(st));
  return GS_OK;
}

}  // extern "C"
