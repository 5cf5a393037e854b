// gs_sweeps.cuh -- warp-cooperative passes over a dense chi array (wide sections).
// Part of gs_kernels.cu (one translation unit; included inside namespace gs).
#pragma once

// @region sweeps
#ifndef GS_GUNROLL
#define GS_GUNROLL 2   // block form (kG > 1, chi in L2): read-only / out-of-place passes
                       // keep this many iterations' loads in flight per thread (A/B r02g: 2 ~ 4 > 1)
#endif
constexpr int kGUnroll = GS_GUNROLL;   // (pragmas do not expand macros)
#ifndef GS_WUNROLL
#define GS_WUNROLL 1   // warp form (chi in shared memory): det-sum / compaction rounds in flight
#endif
constexpr u32 kWUnroll = GS_WUNROLL;
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
// ldps with the "pending scale?" test hoisted out of a pass: passes are
// instantiated for both and dispatch once (ps is uniform over the pass)
template <bool kPS>
__device__ __forceinline__ double2 ldp(const double2 *__restrict__ A, u32 i, double ps) {
  const double2 v = A[i];
  return kPS ? cscale(v, ps) : v;
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

// One T gate's pair update new = a v + (-1)^s b w.  kR: the reduced form of
// a TF_RED op -- T = phi (c I + b' Z) with b' = i ss purely imaginary, the
// global phase phi = e^{+-i pi/8} left out of chi (the kernel counts it in
// `pn` and applies it only where amplitudes leave the device, dumps): 4
// FP64 operations instead of 10 (c v + (-1)^s i ss w).
constexpr double kTc = GS_C8;   // cos(pi/8), ref state.py:107
constexpr double kTs = GS_S8;   // sin(pi/8)
struct Gate {
  double2 a, bx0;   // full form
  double ss;        // reduced form: b' = i ss (per-shot sign included)
  u32 cb, dc, dmask;
};
__device__ __forceinline__ double neg_if1(double x, u32 s) {
  return __longlong_as_double(__double_as_longlong(x) ^ ((long long)s << 63));
}
// The sign arrives as a mask m (0 or 1u << 31, the high word's sign bit) and
// is XORed into the high words of the products ss*w: (-ss)*w == -(ss*w) bit
// for bit, and callers fold the static part of m into the same LOP3 (the
// fused-pair loop: 171 instead of 177 instructions per group).
__device__ __forceinline__ double flip_hi(double x, u32 m) {
  return __hiloint2double(__double2hiint(x) ^ (int)m, __double2loint(x));
}
template <bool kR>
__device__ __forceinline__ double2 t_mix(const Gate &g, double2 v, double2 w, u32 m) {
  if (kR) {
    const double px = flip_hi(__dmul_rn(g.ss, w.y), m), py = flip_hi(__dmul_rn(g.ss, w.x), m);
    return make_double2(__fma_rn(kTc, v.x, -px), __fma_rn(kTc, v.y, py));
  }
  return cadd(cmul(g.a, v), neg_if(cmul(g.bx0, w), m >> 31));
}

#ifndef GS_SGN_OPERAND
#define GS_SGN_OPERAND 1   // A/B r02sgn: +2.0 % headline, +2.0 % grown proxy
#endif
// t_mix with the sign already in the b operand: (-ss) w == -(ss w) and
// cmul(-b, w) == -cmul(b, w) bit for bit, so flipping the operand once per
// sign class (4 per gate and group) replaces flipping each product, and the
// flip leaves the FP64 dependency chain
// (reduced form only: the full form's two-word operand flip measured more
// instructions than the product flips)
struct SgnOp {
  double ss;
  u32 m;
};
template <bool kR>
__device__ __forceinline__ SgnOp sgn_op(const Gate &g, u32 m) {
  SgnOp o;
  o.ss = kR ? flip_hi(g.ss, m) : 0.0;
  o.m = m;
  return o;
}
template <bool kR>
__device__ __forceinline__ double2 t_mix_s(const Gate &g, double2 v, double2 w, const SgnOp &o) {
  if (kR) {
    const double px = __dmul_rn(o.ss, w.y), py = __dmul_rn(o.ss, w.x);
    return make_double2(__fma_rn(kTc, v.x, -px), __fma_rn(kTc, v.y, py));
  }
  return t_mix<false>(g, v, w, o.m);
}

// T with beta in span: new[j] = a v_j + b_j v_{j^cb} (ref state.py:127-129,
// 294-306: a-term then b-term); no renormalisation pending (caller)
template <bool kS, int kG = 1, bool kR = false>
__device__ __forceinline__ SumNz sweep_butterfly(double2 *A_, u32 half, const Gate &g) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = glane<kG>();
  gbar_in<kG>();
  const u32 cb = g.cb, dmask = g.dmask;
  const u32 hb = 31 - __clz(cb);
  SumNz r;
  r.sum = 0.0;
  r.nz = 0;
  const u32 jl = ins_bit(lane, hb, 0);
  const u32 pl = g.dc ^ par32(jl & dmask), pcb = par32(cb & dmask) << 31;
#pragma unroll 1
  for (u32 m = lane; m < half; m += 32u * kG) {
    const u32 jr = ins_bit(m & ~(32u * kG - 1u), hb, 0);
    const u32 j0 = jr | jl, j1 = j0 ^ cb;
    const double2 v0 = A[j0], v1 = A[j1];
    const u32 m0 = (pl ^ par32(jr & dmask)) << 31, m1 = m0 ^ pcb;
#if GS_SGN_OPERAND
    A[j0] = prune_acc(t_mix_s<kR>(g, v0, v1, sgn_op<kR>(g, m1)), r.sum, r.nz);
    A[j1] = prune_acc(t_mix_s<kR>(g, v1, v0, sgn_op<kR>(g, m0)), r.sum, r.nz);
#else
    A[j0] = prune_acc(t_mix<kR>(g, v0, v1, m1), r.sum, r.nz);
    A[j1] = prune_acc(t_mix<kR>(g, v1, v0, m0), r.sum, r.nz);
#endif
  }
  return r;
}

// Two consecutive T gates with partner vectors cb1 != cb2 (compiler flag
// TF_FUSE): one pass over the 4-element groups {x, x^cb1, x^cb2,
// x^cb1^cb2}; gate 1 on the cb1 pairs, prune, gate 2 on the cb2 pairs,
// prune -- exactly the two single-gate passes' arithmetic, half the memory
// traffic and index work.  Groups are enumerated by inserting zeros at the
// pivot bits h1 = top(cb1) and h2 = top(cb2 reduced by cb1).
struct SumNz2 {
  double sum;
  u32 nz, nz1;
};
template <bool kS, int kG = 1, bool kR = false>
__device__ __forceinline__ SumNz2 sweep_butterfly2(double2 *A_, u32 quarter, const Gate &g1,
                                                const Gate &g2) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = glane<kG>();
  gbar_in<kG>();
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
  // static sign masks (bit 31) of the group members relative to x0
  const u32 a1 = par32(g1.cb & g1.dmask) << 31, b1 = par32(g2.cb & g1.dmask) << 31;
  const u32 a2 = par32(g1.cb & g2.dmask) << 31, b2 = par32(g2.cb & g2.dmask) << 31;
#pragma unroll 1
  for (u32 m = lane; m < quarter; m += 32u * kG) {
    const u32 jr = ins_bit(ins_bit(m & ~(32u * kG - 1u), plo, 0), phi, 0);
    const u32 x0 = jr | jl;
    const u32 x1 = x0 ^ g1.cb, x2 = x0 ^ g2.cb, x3 = x1 ^ g2.cb;
    const double2 v0 = A[x0], v1 = A[x1], v2 = A[x2], v3 = A[x3];
    const u32 p1 = (l1 ^ par32(jr & g1.dmask)) << 31, p2 = (l2 ^ par32(jr & g2.dmask)) << 31;
    // gate 1: pairs (x0, x1), (x2, x3)
    const u32 s0 = p1, s1 = p1 ^ a1, s2 = p1 ^ b1, s3 = p1 ^ a1 ^ b1;
    // gate 2: pairs (x0, x2), (x1, x3)
    const u32 t0 = p2, t1 = p2 ^ a2, t2 = p2 ^ b2, t3 = p2 ^ a2 ^ b2;
#if GS_SGN_OPERAND
    const SgnOp o0 = sgn_op<kR>(g1, s0), o1 = sgn_op<kR>(g1, s1), o2 = sgn_op<kR>(g1, s2),
                o3 = sgn_op<kR>(g1, s3);
    const double2 u0 = prune_acc(t_mix_s<kR>(g1, v0, v1, o1), dummy, r.nz1);
    const double2 u1 = prune_acc(t_mix_s<kR>(g1, v1, v0, o0), dummy, r.nz1);
    const double2 u2 = prune_acc(t_mix_s<kR>(g1, v2, v3, o3), dummy, r.nz1);
    const double2 u3 = prune_acc(t_mix_s<kR>(g1, v3, v2, o2), dummy, r.nz1);
    const SgnOp q0 = sgn_op<kR>(g2, t0), q1 = sgn_op<kR>(g2, t1), q2 = sgn_op<kR>(g2, t2),
                q3 = sgn_op<kR>(g2, t3);
    A[x0] = prune_acc(t_mix_s<kR>(g2, u0, u2, q2), r.sum, r.nz);
    A[x2] = prune_acc(t_mix_s<kR>(g2, u2, u0, q0), r.sum, r.nz);
    A[x1] = prune_acc(t_mix_s<kR>(g2, u1, u3, q3), r.sum, r.nz);
    A[x3] = prune_acc(t_mix_s<kR>(g2, u3, u1, q1), r.sum, r.nz);
#else
    const double2 u0 = prune_acc(t_mix<kR>(g1, v0, v1, s1), dummy, r.nz1);
    const double2 u1 = prune_acc(t_mix<kR>(g1, v1, v0, s0), dummy, r.nz1);
    const double2 u2 = prune_acc(t_mix<kR>(g1, v2, v3, s3), dummy, r.nz1);
    const double2 u3 = prune_acc(t_mix<kR>(g1, v3, v2, s2), dummy, r.nz1);
    A[x0] = prune_acc(t_mix<kR>(g2, u0, u2, t2), r.sum, r.nz);
    A[x2] = prune_acc(t_mix<kR>(g2, u2, u0, t0), r.sum, r.nz);
    A[x1] = prune_acc(t_mix<kR>(g2, u1, u3, t3), r.sum, r.nz);
    A[x3] = prune_acc(t_mix<kR>(g2, u3, u1, t1), r.sum, r.nz);
#endif
  }
  (void)dummy;
  return r;
}

// T with a new basis vector: A[j] = a v_j, A[size+j] = b_j v_j (reduced
// form: c v_j and (-1)^s i ss v_j)
template <bool kS, int kG = 1, bool kR = false>
__device__ __forceinline__ SumNz sweep_grow(double2 *A_, u32 size, const Gate &g) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = glane<kG>();
  gbar_in<kG>();
  SumNz r;
  r.sum = 0.0;
  r.nz = 0;
  auto one = [&](u32 j, double2 v) {
    const u32 s = g.dc ^ par32(j & g.dmask);
    if (kR) {
      const double sx = neg_if1(g.ss, s);
      A[j] = prune_acc(make_double2(__dmul_rn(kTc, v.x), __dmul_rn(kTc, v.y)), r.sum, r.nz);
      A[size + j] = prune_acc(make_double2(-__dmul_rn(sx, v.y), __dmul_rn(sx, v.x)), r.sum, r.nz);
    } else {
      A[j] = prune_acc(cmul(g.a, v), r.sum, r.nz);
      A[size + j] = prune_acc(neg_if(cmul(g.bx0, v), s), r.sum, r.nz);
    }
  };
  if (kG > 1) {
    // block form (chi in L2): the loads of kGUnroll iterations first -- they
    // never alias the stores (A[size + j]) or another iteration's A[j] --
    // then the same per-thread order of updates (and of the norm sum)
    constexpr u32 NT = 32u * kG;
#pragma unroll 1
    for (u32 j0 = lane; j0 < size; j0 += NT * kGUnroll) {
      double2 v[kGUnroll];
#pragma unroll
      for (int u = 0; u < kGUnroll; ++u)
        if (j0 + u * NT < size) v[u] = A[j0 + u * NT];
#pragma unroll
      for (int u = 0; u < kGUnroll; ++u)
        if (j0 + u * NT < size) one(j0 + u * NT, v[u]);
    }
    return r;
  }
#pragma unroll 1
  for (u32 j = lane; j < size; j += 32u * kG) one(j, A[j]);
  return r;
}

// diagonal phase: A[j] *= (dc ^ par(j & mask)) ? f1 : f0  (T with beta = 0,
// fired noise Paulis)
template <bool kS, int kG, bool kPS>
__device__ __forceinline__ void sweep_phase_impl(double2 *A_, u32 size, u32 dc, u32 mask,
                                         double2 f0, double2 f1, double ps) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = glane<kG>();
  gbar_in<kG>();
#pragma unroll 1
  for (u32 j = lane; j < size; j += 32u * kG)
    A[j] = cmul(ldp<kPS>(A, j, ps), (dc ^ par32(j & mask)) ? f1 : f0);
}
template <bool kS, int kG = 1>
__device__ __forceinline__ void sweep_phase(double2 *A_, u32 size, u32 dc, u32 mask,
                                         double2 f0, double2 f1, double ps) {
  if (ps == 1.0) sweep_phase_impl<kS, kG, false>(A_, size, dc, mask, f0, f1, ps);
  else sweep_phase_impl<kS, kG, true>(A_, size, dc, mask, f0, f1, ps);
}

// beta = 0 measurement weights: (sum over +1 eigen-entries, sum over -1)
template <bool kS, int kG, bool kPS>
__device__ __forceinline__ double2 sweep_det_sums_impl(double2 *A_, u32 size, u32 dmask, u32 neg0,
                                               double ps) {
  const double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = glane<kG>();
  gbar_in<kG>();
  double sp = 0.0, sm = 0.0;
#pragma unroll (kG > 1 ? kGUnroll : kWUnroll)
  for (u32 j = lane; j < size; j += 32u * kG) {
    const double a2 = abs2(ldp<kPS>(A, j, ps));
    if (neg0 ^ par32(j & dmask)) sm = __dadd_rn(sm, a2); else sp = __dadd_rn(sp, a2);
  }
  return make_double2(sp, sm);
}
template <bool kS, int kG = 1>
__device__ __forceinline__ double2 sweep_det_sums(double2 *A_, u32 size, u32 dmask, u32 neg0,
                                               double ps) {
  if (ps == 1.0) return sweep_det_sums_impl<kS, kG, false>(A_, size, dmask, neg0, ps);
  return sweep_det_sums_impl<kS, kG, true>(A_, size, dmask, neg0, ps);
}

// keep the chosen eigen-entries, scaled by rs; zero the others
template <bool kS, int kG, bool kPS>
__device__ __forceinline__ SumNz sweep_filter_impl(double2 *A_, u32 size, u32 dmask, u32 neg0,
                                           u32 want_neg, double rs, double ps) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = glane<kG>();
  gbar_in<kG>();
  SumNz r;
  r.sum = 0.0;
  r.nz = 0;
#pragma unroll 1
  for (u32 j = lane; j < size; j += 32u * kG) {
    const double2 v = ldp<kPS>(A, j, ps);
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
template <bool kS, int kG = 1>
__device__ __forceinline__ SumNz sweep_filter(double2 *A_, u32 size, u32 dmask, u32 neg0,
                                           u32 want_neg, double rs, double ps) {
  if (ps == 1.0) return sweep_filter_impl<kS, kG, false>(A_, size, dmask, neg0, want_neg, rs, ps);
  return sweep_filter_impl<kS, kG, true>(A_, size, dmask, neg0, want_neg, rs, ps);
}

// in-place compaction dropping coordinate isq: A[jp] = rs * A[src(jp)],
// src(jp) = j0 | ((tau ^ par(j0 & mask)) << isq), j0 = jp with a 0 inserted
// at isq; src(jp) >= jp, so reads of a round finish before its writes
template <bool kS, int kG, bool kPS>
__device__ __forceinline__ SumNz sweep_compact_impl(double2 *A_, u32 half, u32 isq, u32 mask, u32 tau,
                                            double rs, double ps) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = glane<kG>();
  gbar_in<kG>();
  SumNz r;
  r.sum = 0.0;
  r.nz = 0;
  // kB rounds per barrier pair: a batch reads src(jp) >= jp for its own jp
  // range before any of its writes, and later batches read above it, so
  // batching keeps the in-place order safe with kB loads in flight per lane
  // (and the per-lane order of the norm sum)
  constexpr u32 kB = kG == 1 ? kWUnroll : 1;
  constexpr u32 NT = 32u * kG;
#pragma unroll 1
  for (u32 b0 = 0; b0 < half; b0 += NT * kB) {
    double2 v[kB];
#pragma unroll
    for (u32 u = 0; u < kB; ++u) {
      const u32 jp = b0 + u * NT + lane;
      v[u] = make_double2(0.0, 0.0);
      if (jp < half) {
        const u32 j0 = ins_bit(jp, isq, 0);
        v[u] = ldp<kPS>(A, j0 | ((tau ^ par32(j0 & mask)) << isq), ps);
      }
    }
    gsync<kG>();
#pragma unroll
    for (u32 u = 0; u < kB; ++u) {
      const u32 jp = b0 + u * NT + lane;
      if (jp < half) {
        const double2 w = cscale(v[u], rs);
        A[jp] = w;
        r.sum = __dadd_rn(r.sum, abs2(w));
        r.nz += nonzero(w);
      }
    }
    gsync<kG>();
  }
  return r;
}
// compaction that only moves (the renormalisation is deferred by the
// caller into the next pass's loads, ldps): A[jp] = ps * A[src(jp)], same
// round structure as sweep_compact; returns the nonzero count
template <bool kS, int kG, bool kPS>
__device__ __forceinline__ u32 sweep_compact_move_impl(double2 *A_, u32 half, u32 isq, u32 mask, u32 tau,
                                                    double ps) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = glane<kG>();
  gbar_in<kG>();
  u32 nz = 0;
#pragma unroll 1
  for (u32 b0 = 0; b0 < half; b0 += 32u * kG) {
    const u32 jp = b0 + lane;
    double2 v = make_double2(0.0, 0.0);
    if (jp < half) {
      const u32 j0 = ins_bit(jp, isq, 0);
      v = ldp<kPS>(A, j0 | ((tau ^ par32(j0 & mask)) << isq), ps);
    }
    gsync<kG>();
    if (jp < half) {
      A[jp] = v;
      nz += nonzero(v);
    }
    gsync<kG>();
  }
  return nz;
}
template <bool kS, int kG = 1>
__device__ __forceinline__ u32 sweep_compact_move(double2 *A_, u32 half, u32 isq, u32 mask, u32 tau,
                                               double ps) {
  if (ps == 1.0) return sweep_compact_move_impl<kS, kG, false>(A_, half, isq, mask, tau, ps);
  return sweep_compact_move_impl<kS, kG, true>(A_, half, isq, mask, tau, ps);
}
// out of place (ping-pong buffers, global chi): D[jp] = rs * A[src(jp)] in
// one pass, no per-round barriers
template <int kG>
__device__ __forceinline__ SumNz sweep_compact_to(const double2 *__restrict__ A, double2 *__restrict__ D,
                                               u32 half, u32 isq, u32 mask, u32 tau, double rs,
                                               double ps) {
  const u32 lane = glane<kG>();
  gbar_in<kG>();
  SumNz r;
  r.sum = 0.0;
  r.nz = 0;
#pragma unroll (kG > 1 ? kGUnroll : 1)
  for (u32 jp = lane; jp < half; jp += 32u * kG) {
    const u32 j0 = ins_bit(jp, isq, 0);
    const double2 w = cscale(ldps(A, j0 | ((tau ^ par32(j0 & mask)) << isq), ps), rs);
    D[jp] = w;
    r.sum = __dadd_rn(r.sum, abs2(w));
    r.nz += nonzero(w);
  }
  return r;
}
template <bool kS, int kG = 1>
__device__ __forceinline__ SumNz sweep_compact(double2 *A_, u32 half, u32 isq, u32 mask, u32 tau,
                                            double rs, double ps) {
  if (ps == 1.0) return sweep_compact_impl<kS, kG, false>(A_, half, isq, mask, tau, rs, ps);
  return sweep_compact_impl<kS, kG, true>(A_, half, isq, mask, tau, rs, ps);
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
template <bool kS, int kG = 1>
__device__ __forceinline__ double sweep_pivot_p(double2 *A_, PivotGeo g, double2 xpp, double ps) {
  const double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = glane<kG>();
  gbar_in<kG>();
  double sp = 0.0;
#pragma unroll (kG > 1 ? kGUnroll : 1)
  for (u32 m = lane; m < g.npairs; m += 32u * kG) {
    double2 vr, pr;
    u32 d_;
    pivot_terms(A, g, xpp, m, vr, pr, d_, ps);
    sp = __dadd_rn(sp, abs2(cadd(vr, pr)));
  }
  return sp;
}
template <bool kS, int kG = 1>
__device__ __forceinline__ SumNz sweep_pivot_w(double2 *A_, PivotGeo g, double2 xpp, bool plus,
                                            double ps) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = glane<kG>();
  gbar_in<kG>();
  SumNz r;
  r.sum = 0.0;
  r.nz = 0;
#pragma unroll 1
  for (u32 m = lane; m < g.npairs; m += 32u * kG) {
    double2 vr, pr;
    u32 dst;
    pivot_terms(A, g, xpp, m, vr, pr, dst, ps);
    A[dst] = prune_acc(plus ? cadd(vr, pr) : csub(vr, pr), r.sum, r.nz);
  }
  return r;
}

// span pivot in one pass (ping-pong buffers): sums P+ = sum |w+|^2 in the
// order sweep_pivot_p does, and writes both outcomes' merged, pruned pairs
// to their compacted slots of D -- w+ at m, w- at half + m (the compaction
// of the rep slots, sweep_compact with mask = tmask, tau = ct, reads rep(m)
// for slot m) -- with each outcome's kept sum and count
struct PivotBoth {
  double pp, sump, summ;
  u32 nzp, nzm;
};
template <int kG>
__device__ __forceinline__ PivotBoth sweep_pivot_both(const double2 *__restrict__ A, double2 *__restrict__ D,
                                                   PivotGeo g, double2 xpp, double ps) {
  const u32 lane = glane<kG>();
  gbar_in<kG>();
  PivotBoth r;
  r.pp = 0.0; r.sump = 0.0; r.summ = 0.0;
  r.nzp = 0; r.nzm = 0;
  double2 *__restrict__ Dm = D + g.npairs;
#pragma unroll (kG > 1 ? kGUnroll : 1)
  for (u32 m = lane; m < g.npairs; m += 32u * kG) {
    double2 vr, pr;
    u32 dst;
    pivot_terms(A, g, xpp, m, vr, pr, dst, ps);
    const double2 wp = cadd(vr, pr);
    r.pp = __dadd_rn(r.pp, abs2(wp));
    D[m] = prune_acc(wp, r.sump, r.nzp);
    Dm[m] = prune_acc(csub(vr, pr), r.summ, r.nzm);
  }
  return r;
}

// no-span pivot without a pending scale: rep entries keep v (w = v +- (-0)
// == v), so only the part entries -- those with ct ^ par(m & tmask) = 1, an
// affine half enumerated by inserting the parity bit at the top bit h of
// tmask -- are rewritten, as +-(+-i^xi0) v (exact rotations: no entry's
// modulus changes, the norm and nonzero count carry over)
template <bool kS, int kG = 1>
__device__ __forceinline__ void sweep_pivot_part(double2 *A_, const PivotGeo &g, double2 xpp, bool plus,
                                                 u32 size) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = glane<kG>();
  gbar_in<kG>();
  const double2 xp = plus ? xpp : cneg(xpp), xm = cneg(xp);
  if (g.tmask == 0) {
    if (!g.ct) return;
#pragma unroll 1
    for (u32 m = lane; m < size; m += 32u * kG)
      A[m] = cmul((g.dc ^ par32(m & g.dmask)) ? xm : xp, A[m]);
    return;
  }
  const u32 h = 31 - __clz(g.tmask);
#pragma unroll 1
  for (u32 i = lane; i < (size >> 1); i += 32u * kG) {
    const u32 j0 = ins_bit(i, h, 0);
    const u32 m = j0 | ((g.ct ^ 1u ^ par32(j0 & g.tmask)) << h);
    A[m] = cmul((g.dc ^ par32(m & g.dmask)) ? xm : xp, A[m]);
  }
}

// apply a pending renormalisation in place: A[j] = ps * A[j]
template <bool kS, int kG = 1>
__device__ __forceinline__ void sweep_scale(double2 *A_, u32 size, double ps) {
  double2 *__restrict__ A = chi_ptr<kS>(A_);
  const u32 lane = glane<kG>();
  gbar_in<kG>();
#pragma unroll 1
  for (u32 j = lane; j < size; j += 32u * kG) A[j] = cscale(A[j], ps);
}
