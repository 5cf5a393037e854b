// gs_common.cuh -- op/record layouts, device structs, complex helpers, RNG (SHA-1, SplitMix, Philox, geometric schedule).
// Part of gs_kernels.cu (one translation unit; included inside namespace gs).
#pragma once

enum { OP_END = 0, OP_T = 1, OP_MEAS = 2, OP_NOISE = 3, OP_FEEDBACK = 4,
       OP_DETECTOR = 5, OP_OBSERVABLE = 6, OP_GROW_LIMIT = 7 };
enum { T_DIAG = 0, T_BUTTERFLY = 1, T_GROW = 2 };
enum { TF_FUSE = 16 };   // T flag: apply together with the next BUTTERFLY op
enum { TF_RED = 32 };    // T flag: BUTTERFLY / GROW in the reduced form (t_mix)
enum { TF_FUSEQ = 64 };  // T flag: TF_FUSE if no noise fires before the partner (Philox)
enum { M_DET = 0, M_PIVOT_SPAN = 1, M_PIVOT_NOSPAN = 2 };
enum { MF_RECORD = 16, MF_FLIP = 32, MF_RESET = 64, MF_COMPACT = 128 };
enum { NK_DEP1 = 0, NK_DEP2 = 1, NK_XERR = 2, NK_ZERR = 3 };
enum { ST_RUNNING = 0, ST_PRESERVED = 1, ST_DISCARDED = 2, ST_OVERFLOW = 3,
       ST_CORRUPT = 4, ST_UNSUPPORTED = 5 };
enum { MODE_COUNTERS = 0, MODE_RECORDS = 1, MODE_DUMP = 2 };

constexpr int kWinWords = 48;          // SplitMix fire-bit ring: 1536 locations (>= one
                                       // instruction's 33 words + lookahead; 48 so 14
                                       // warp-form slices of 16 KB chi + ring fit an SM)
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
  u32 kn;                 // narrow chi dimension limit (narrow_kn)
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
  u32 rec_local;        // record words kept warp-locally: in the slice's shared memory
                        // (narrow kn=4, block form) or in registers (warp form, narrow
                        // kn=5); else in the global O.grec buffer
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
// e^{i pi n / 8} * v: the global phase the reduced T ops leave out of chi,
// restored where amplitudes leave the device (dumps)
#define GS_C8 0x1.d906bcf328d46p-1   /* cos(pi/8) */
#define GS_S8 0x1.87de2a6aea963p-2   /* sin(pi/8) */
#define GS_R2 0x1.6a09e667f3bcdp-1   /* sqrt(1/2) */
__constant__ double2 kPhase16[16] = {
    {1.0, 0.0},     {GS_C8, GS_S8},   {GS_R2, GS_R2},   {GS_S8, GS_C8},
    {0.0, 1.0},     {-GS_S8, GS_C8},  {-GS_R2, GS_R2},  {-GS_C8, GS_S8},
    {-1.0, 0.0},    {-GS_C8, -GS_S8}, {-GS_R2, -GS_R2}, {-GS_S8, -GS_C8},
    {0.0, -1.0},    {GS_S8, -GS_C8},  {GS_R2, -GS_R2},  {GS_C8, -GS_S8}};
__device__ __forceinline__ double2 with_phase(u32 n, double2 v) {
  return (n & 15u) ? cmul(kPhase16[n & 15u], v) : v;
}
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

// Threads that share one shot's chi in the wide kernel: one warp (kG = 1,
// every lane its own coordinates) or, for large chi, the whole block of kG
// warps (blockDim = 32 kG).  In the block form every warp runs the shot's
// scalar logic redundantly (same inputs, same results) and only the chi
// passes are split; group reductions sum the warps' totals in warp order
// through a two-slot shared scratch, so every warp sees the same bits.
template <int kG>
__device__ __forceinline__ u32 glane() { return kG == 1 ? (threadIdx.x & 31u) : threadIdx.x; }
template <int kG>
__device__ __forceinline__ void gsync() {
  if (kG == 1) __syncwarp(); else __syncthreads();
}
// barrier on entry to a chi pass (block form): orders it after the previous
// pass's writes by other warps
template <int kG>
__device__ __forceinline__ void gbar_in() {
  if (kG > 1) __syncthreads();
}
struct GroupScratch {
  u64 *slots;   // 2 x 32 words of shared memory (block form only)
  u32 tog;      // alternating half: a slot half is rewritten only after the
                // barrier of the next reduction, which every reader passed
};
template <int kG>
__device__ __forceinline__ double group_sum(double v, GroupScratch &g) {
  v = warp_sum(v);
  if (kG == 1) return v;
  u64 *s = g.slots + 32u * g.tog;
  g.tog ^= 1u;
  if ((threadIdx.x & 31u) == 0) s[threadIdx.x >> 5] = (u64)__double_as_longlong(v);
  __syncthreads();
  double t = __longlong_as_double((long long)s[0]);
#pragma unroll 1
  for (int w = 1; w < kG; ++w) t = __dadd_rn(t, __longlong_as_double((long long)s[w]));
  return t;
}
template <int kG>
__device__ __forceinline__ u32 group_sum_u32(u32 v, GroupScratch &g) {
  v = warp_sum_u32(v);
  if (kG == 1) return v;
  u64 *s = g.slots + 32u * g.tog;
  g.tog ^= 1u;
  if ((threadIdx.x & 31u) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  u32 t = 0;
#pragma unroll 1
  for (int w = 0; w < kG; ++w) t += (u32)s[w];
  return t;
}
// thread 0's value to the whole group (kG == 1: lane 0's)
template <int kG>
__device__ __forceinline__ u64 group_bcast(u64 v, GroupScratch &g) {
  if (kG == 1) return __shfl_sync(FULL, v, 0);
  u64 *s = g.slots + 32u * g.tog;
  g.tog ^= 1u;
  if (threadIdx.x == 0) s[0] = v;
  __syncthreads();
  return s[0];
}
template <int kG>
__device__ __forceinline__ u32 group_bcast32(u32 v, GroupScratch &g) {
  if (kG == 1) return __shfl_sync(FULL, v, 0);
  return (u32)group_bcast<kG>(v, g);
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

constexpr u64 kSplitGamma = 0x9E3779B97F4A7C15ull;
// SplitMix64 draw k = mix(seed + (k + 1) gamma), split so a run of draws can
// step the pre-mix counter by additions
__device__ __forceinline__ u64 splitmix_pre(u64 seed, u32 k) { return seed + (u64)(k + 1ull) * kSplitGamma; }
__device__ __forceinline__ u64 splitmix_mix(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ u64 splitmix(u64 seed, u32 k) { return splitmix_mix(splitmix_pre(seed, k)); }

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

// narrow (lane-per-shot) chi dimension limit kn, a run-time choice: 4, or
// 5 with GS_NARROW_K5 (A/B r02j: the Table-2 d=5 headline +10.3 % at 5, the
// d=3 workload -23 % and the grown proxy -8.5 %; sampler.Program tunes it
// per program by timing both on a probe run -- results are identical).  At
// 5 only the narrow sections that hold a k = 5 op use 2^5 chi rows per lane
// (12 warps/SM); the others keep the 2^4-row, 20-warp layout (Section::kn)
__host__ __device__ __forceinline__ u32 narrow_kn(u32 flags) { return (flags & GS_NARROW_K5) ? 5u : 4u; }
__host__ __device__ __forceinline__ u32 narrow_bytes(u32 kn) { return (1u << kn) * 32u * 16u; }   // An[2^kn][32] double2
constexpr u32 kCntBytes = 64;                              // per-warp counters

__device__ __forceinline__ bool nonzero(double2 v) { return v.x != 0.0 || v.y != 0.0; }

__device__ __forceinline__ u32 lanemask_lt(u32 lane) { return (1u << lane) - 1u; }
