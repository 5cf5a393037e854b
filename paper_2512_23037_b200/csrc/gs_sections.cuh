// gs_sections.cuh -- section pipeline: shared helpers, narrow_kernel (lane per shot), wide_kernel (warp per shot).
// Part of gs_kernels.cu (one translation unit; included inside namespace gs).
#pragma once

// ---------------------------------------------------------------- kernels
//
// Execution model: breadth-first SECTIONS.  k is static per op
// (shot-invariant basis, compiler.py), so the op stream splits on the host
// into alternating sections of narrow ops (chi dimension k <= kn before
// and after the op) and wide ops (k > kn, GROW_LIMIT).  One launch per
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
// slots: state words, record bits, chi of dimension <= kn) read by the
// next section's launch.  Each launch keeps only its own code hot, which is
// what the instruction cache needs (B200: 32 KB L1.5).
// GS_WIDE_ONLY runs the whole program as one wide section (A/B, tests).

#ifndef GS_NARROW_WARPS_K5
#define GS_NARROW_WARPS_K5 14   // kn=5 narrow build: most warps per block (14 x 16 KB of chi rows)
#endif
#ifndef GS_COMPACT_DEFER
#define GS_COMPACT_DEFER 1   // beta = 0 compactions move only, renormalisation deferred (A/B r02gg)
#endif
#ifndef GS_NARROW_RED
#define GS_NARROW_RED 1   // reduced T form in the narrow kernel too (A/B r02ff)
#endif
#ifndef GS_NARROW_BLOCKS
#define GS_NARROW_BLOCKS 5   // <= 102 registers: 20 warps/SM (A/B: 47.4M vs 46.4M at 4)
#endif
#ifndef GS_WIDE_BLOCKS
// launch bound only: blocks of up to GS_WIDE_WARPS warps, 1 resident ->
// <= 146 registers, which 14 warps of the warp form can hold (round 1 held
// the wide kernel to 128 registers for 13 one-warp blocks: r01bl)
#define GS_WIDE_BLOCKS 1
#endif
#ifndef GS_WIDE_WARPS
#define GS_WIDE_WARPS 14   // most warps per wide block (warp form: 14 x 16 KB of chi fit an SM)
#endif
#ifndef GS_BLOCK_WARPS
#define GS_BLOCK_WARPS 16  // warps sharing one shot's chi (block form)
#endif
#ifndef GS_BLOCK_MINB
#define GS_BLOCK_MINB 1   // resident blocks the block form is compiled for (register bound)
#endif
#ifndef GS_BLOCK_MIN_DIM
#define GS_BLOCK_MIN_DIM 13   // chi dimension from which the block form is the default
#endif

__host__ __device__ __forceinline__ bool op_is_wide(u32 kind, u32 k, u32 fl, u32 kn) {
  return kind == OP_GROW_LIMIT || k > kn ||
         (kind == OP_T && (fl & 3u) == T_GROW && k + 1 > kn);
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
// the chi rows [0, 2^kn)
enum { Q_SL = 0, Q_LO, Q_HI, Q_C, Q_OBS, Q_MB, Q_PICK, Q_SEED, Q_CNTK, Q_GEO, Q_FIRE, Q_HDR = 12 };

struct DevSec {
  u32 pc0, k0, nm0;        // first op, its chi dimension, first noise instr. with ipc >= pc0
  u32 pc_end;              // stop before this op: the next section's first (0xFFFFFFFF: last section)
  u64 first, count;        // fresh shots (q_in == nullptr): run-local indices [first, first+count)
  const u64 *q_in;         // else: queue slots and their number
  const u32 *n_in;
  u64 *q_out;              // survivors at the section end (nullptr: last section)
  u32 *n_out;
  unsigned long long *work; // atomic work counter
  u32 pn0;                 // reduced-T phase count at pc0 (static; see t_mix)
  u32 kn;                  // narrow sections: chi rows per lane 2^kn (4 or 5)
};

// record words of a slot, rounded to 16 B so the chi rows are double2-aligned
__host__ __device__ __forceinline__ u32 rec_u64(u32 rec_words32) { return ((rec_words32 + 3) / 4) * 2; }

__device__ __forceinline__ u32 slot_u64(const DevProg &P) {
  return Q_HDR + rec_u64(P.rec_words32) + 2 * (1u << P.kn);
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

// the warp form's counters: lane i holds counter i (WC_* order)
__device__ __forceinline__ void flush_counter_regs(const DevOut &O, u64 cntl, u32 lane) {
  if (lane < WC_N && cntl) {
    const int dst[WC_N] = {GS_C_TOTAL, GS_C_PRESERVED, GS_C_DISCARDED, GS_C_OVERFLOW,
                           GS_C_CORRUPT, GS_C_UNSUPPORTED, GS_C_ERROR_SHOTS, GS_C_MODEL_BYTES};
    atomicAdd((unsigned long long *)O.counters + dst[lane], (unsigned long long)cntl);
  }
}

// ---------------------------------------------------------------- narrow

// dumps: restore the global phase of earlier reduced T ops (cold path, out
// of line so the narrow kernel's registers are unaffected)
__device__ __noinline__ void narrow_dump_phase(double2 *amps, u32 n, u32 pn) {
#pragma unroll 1
  for (u32 j = 0; j < n; ++j) amps[j] = with_phase(pn, amps[j]);
}

// @region narrow: prologue
// kK5: the narrow limit kn = 5 build -- 16 KB of chi rows per warp make
// shared memory the occupancy limit (3 blocks = 12 warps/SM), so it is
// compiled for 3 resident blocks (more registers: no spills in the queue
// reads); kn = 4 keeps 5 blocks = 20 warps/SM
//
// The kn = 5 build also keeps the warp's counters (lane i: counter i) and a
// shot's record words (up to kNarrowRecRegs, one register each; indices are
// warp-uniform, so the unrolled selects stay in registers) out of shared
// memory: a warp's slice is its 16 KB of chi rows alone and 14 warps fit
// an SM in 7-warp blocks instead of 12 (host: rec_local = 1 means "record
// words in registers" for this build)
constexpr u32 kNarrowRecRegs = 4;   // 128 measurements
template <bool kPhilox, bool kK5>
__global__ void __launch_bounds__(kK5 ? 32 * GS_NARROW_WARPS_K5 : 128, kK5 ? 1 : GS_NARROW_BLOCKS)
narrow_kernel(DevProg P, DevRun R, DevOut O, DevSec S) {
  extern __shared__ __align__(16) u8 smem[];
  const u32 lane = threadIdx.x & 31u;
  const u32 wib = threadIdx.x >> 5;
  const u32 wpb = blockDim.x >> 5;
  const u64 gw = (u64)blockIdx.x * wpb + wib;
  u8 *mine = smem + (size_t)wib * O.warp_bytes;
  constexpr bool kReg = kK5;
  const bool rec_reg = kReg && O.rec_local;
  u64 cntl = 0;                   // kReg: counter WC_[lane]
  u32 rr[kNarrowRecRegs] = {};    // rec_reg: this lane's record words
  unsigned long long *wcnt = kReg ? nullptr : reinterpret_cast<unsigned long long *>(mine);
  double2 *An = reinterpret_cast<double2 *>(mine + (kReg ? 0u : kCntBytes));
  // record bits, one column per lane: word w of lane l at recb[w * 32 + l]
  u32 *recb = rec_reg ? nullptr
              : (O.rec_local ? reinterpret_cast<u32 *>(mine + kCntBytes + narrow_bytes(S.kn))
                               : O.grec + gw * (u64)P.rec_words32 * 32u);
  // record word w (warp-uniform) of this lane's shot
  auto rec_get = [&](u32 w) -> u32 {
    if (!rec_reg) return recb[w * 32u + lane];
    u32 v = 0;
#pragma unroll
    for (u32 i = 0; i < kNarrowRecRegs; ++i)
      if (i == w) v = rr[i];
    return v;
  };
  auto rec_set = [&](u32 w, u32 v) {
    if (!rec_reg) { recb[w * 32u + lane] = v; return; }
#pragma unroll
    for (u32 i = 0; i < kNarrowRecRegs; ++i)
      if (i == w) rr[i] = v;
  };
  const u32 n = P.n;
  const u64 *__restrict__ ops = P.ops;
  const u64 *__restrict__ tables = P.tables;
  const u64 *__restrict__ locs = P.locs;
  const double2 Z = make_double2(0.0, 0.0);
  constexpr bool philox = kPhilox;   // RNG mode is a template parameter
  const u32 sign_bytes = 2u * ((2u * n + 7u) / 8u);
  const u32 SU = slot_u64(P);
#define AN(j) An[(j) * 32u + lane]

  if (!kReg && lane < WC_N) wcnt[lane] = 0;
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
    // chi unchanged since a sum of all |v|^2 came out exactly 1 (so the next
    // dmask = 0 measurement's sums are known without the loop)
    bool sone = false;
    int sst = valid ? ST_RUNNING : ST_PRESERVED, saux = -1;
    // Philox fire schedule of this shot
    u32 sgj = 0, sgpos = 0xFFFFFFFFu, sfire = 0xFFFFFFFFu;
    // GS_NARROW_RED: chi = e^{i pi spn / 8} * An (reduced T ops, as the wide
    // kernel's pn; static per op, per lane only because lanes stop apart)
    u32 spn = S.pn0;
    u64 sgpick = 0;
    if (!S.q_in) {
      sl = S.first + idx;
      shot = R.shot_begin + sl;
      if (valid && !philox) seed = R.seeds ? R.seeds[sl] : sha1_seed(R.master, shot);
#pragma unroll 1
      for (u32 w = 0; w < P.rec_words32; ++w) rec_set(w, 0u);
      AN(0) = make_double2(1.0, 0.0);
      sone = true;
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
      for (u32 w = 0; w < P.rec_words32; ++w) rec_set(w, __ldg(qr + w));
      // chi rows: every lane reads its own slot (a strided gather across
      // the warp), so keep several loads in flight per lane instead of one
      const double2 *qc = reinterpret_cast<const double2 *>(q + Q_HDR + rec_u64(P.rec_words32));
      const u32 n0 = 1u << S.k0;
#pragma unroll 1
      constexpr u32 kQ = kK5 ? 8u : 1u;
      for (u32 j0 = 0; j0 < n0; j0 += kQ) {
        double2 t[kQ];
#pragma unroll
        for (u32 u = 0; u < kQ; ++u)
          if (j0 + u < n0) t[u] = __ldg(qc + j0 + u);
#pragma unroll
        for (u32 u = 0; u < kQ; ++u)
          if (j0 + u < n0) AN(j0 + u) = t[u];
      }
    }
    __syncwarp();

    u32 pc = S.pc0, nm = S.nm0;
    u32 exit_k = 0;
    u64 hnext = __ldg(ops + pc);
#pragma unroll 1
    for (;;) {
      if (!__any_sync(FULL, sst == ST_RUNNING)) break;
      const u64 h = hnext;
      const u32 kind = (u32)(h & 0xff), len = (u32)((h >> 8) & 0xff);
      const u32 k = (u32)((h >> 16) & 0xff), fl = (u32)((h >> 24) & 0xff);
      const u32 instr = (u32)(h >> 32);
      if (pc == S.pc_end) { exit_k = k; break; }   // the next section starts (host plan)
      // ============================== narrow op, lane per shot
      // @region narrow: noise
      // apply E to this lane's shot (ref state.py:88-102)
      auto lane_error = [&](u64 ex, u64 ez, const u64 *nrec, u32 size) {
        sone = false;
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
          // one instruction's locations share their kind and threshold and
          // draw at d0, d0 + step, ... (compiler.py emit_noise; DEPOLARIZE
          // draws twice per location), so the fire test walks SplitMix's
          // pre-mix counter z = seed + (d + 1) gamma by additions and loads a
          // location word only when it fires (same draws, same bits)
          if (nloc) {
            const u64 lw0 = __ldg(locs + 2ull * loc0), thr = __ldg(locs + 2ull * loc0 + 1);
            const u32 step = (((u32)(lw0 >> 48) & 3) <= NK_DEP2) ? 2u : 1u;
            u64 z = splitmix_pre(seed, (u32)lw0);
            const u64 dz = (u64)step * kSplitGamma;
#pragma unroll 1
            for (u32 l = loc0; l < loc0 + nloc; ++l, z += dz) {
              if ((splitmix_mix(z) >> 11) < thr) {
                const u64 lw = __ldg(locs + 2ull * l);
                const u32 nk = (u32)(lw >> 48) & 3;
                const double u = nk <= NK_DEP2 ? (double)(splitmix_mix(z + kSplitGamma) >> 11) * 0x1.0p-53 : 0.0;
                noise_letter(nk, (u32)(lw >> 32) & 0xff, (u32)(lw >> 40) & 0xff, u, ex, ez);
              }
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
      hnext = __ldg(ops + pc);   // the next header, loaded while this op runs
      if (sst != ST_RUNNING) continue;
      sk = k;

      // @region narrow: T
      if (kind == OP_T) {
        sone = false;
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
        if (GS_NARROW_RED && (fl & TF_RED)) {
          // reduced form (gs_sweeps.cuh t_mix): c v + (-1)^s i ss w, the
          // global phase counted in spn -- 4 FP64 operations per entry
          const u64 w12 = __ldg(op + 12);
          const double ssr = neg_if1(kTs, ((u32)w12 & 1u) ^ flip);
          spn = (spn + ((w12 & 2u) ? 15u : 1u)) & 15u;
          if (tcase == T_BUTTERFLY) {
            const u32 hb = 31 - __clz(cb);
#pragma unroll 1
            for (u32 m = 0; m < (size >> 1); ++m) {
              const u32 j0 = ins_bit(m, hb, 0), j1 = j0 ^ cb;
              const double2 v0 = AN(j0), v1 = AN(j1);
              const double sx0 = neg_if1(ssr, dc ^ par32(j1 & dmask));
              const double sx1 = neg_if1(ssr, dc ^ par32(j0 & dmask));
              const double2 n0 = prune(make_double2(__fma_rn(kTc, v0.x, -__dmul_rn(sx0, v1.y)),
                                                    __fma_rn(kTc, v0.y, __dmul_rn(sx0, v1.x))));
              const double2 n1 = prune(make_double2(__fma_rn(kTc, v1.x, -__dmul_rn(sx1, v0.y)),
                                                    __fma_rn(kTc, v1.y, __dmul_rn(sx1, v0.x))));
              AN(j0) = n0;
              AN(j1) = n1;
              nz += nonzero(n0) + nonzero(n1);
            }
          } else {
#pragma unroll 1
            for (u32 j = 0; j < size; ++j) {
              const double2 v = AN(j);
              const double sx = neg_if1(ssr, dc ^ par32(j & dmask));
              const double2 n0 = prune(make_double2(__dmul_rn(kTc, v.x), __dmul_rn(kTc, v.y)));
              const double2 n1 = prune(make_double2(-__dmul_rn(sx, v.y), __dmul_rn(sx, v.x)));
              AN(j) = n0;
              AN(size + j) = n1;
              nz += nonzero(n0) + nonzero(n1);
            }
            sk = k + 1;
          }
        } else if (tcase == T_BUTTERFLY) {
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
          if (sone && dmask == 0) {
            // same entries, same order: the loop would return exactly these
            sp = neg0 ? 0.0 : 1.0;
            sm = neg0 ? 1.0 : 0.0;
          } else {
#pragma unroll 1
            for (u32 j = 0; j < size; ++j) {
              const double a2 = abs2(AN(j));
              if (neg0 ^ par32(j & dmask)) sm = __dadd_rn(sm, a2); else sp = __dadd_rn(sp, a2);
            }
          }
          sone = false;
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
          } else if (rs == 1.0 && dmask == 0 && neg0 == want_neg) {
            nz = scnt;   // every entry kept and scaled by exactly 1: nothing changes
            sone = true;
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
          sone = false;
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
        if ((fl & MF_RECORD) && rb) rec_set(slot >> 5, rec_get(slot >> 5) | (1u << (slot & 31)));
        if ((fl & MF_RESET) && bout) { s_lo ^= __ldg(op + 15); s_hi ^= __ldg(op + 16); }
        continue;
      }

      // @region narrow: feedback/detector/end
      if (kind == OP_FEEDBACK) {
        const u32 idx = (u32)__ldg(op + 1);
        if ((rec_get(idx >> 5) >> (idx & 31)) & 1u) {
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
          parity ^= (rec_get(idx >> 5) >> (idx & 31)) & 1u;
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
        for (u32 w = 0; w < P.rec_words32; ++w) qr[w] = rec_get(w);
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
      if (kReg) {   // lane i accumulates counter i
        u32 m = 0;
        switch (lane) {
          case WC_TOT: m = val; break;
          case WC_PRES: m = pres; break;
          case WC_DISC: m = disc; break;
          case WC_OVF: m = ovf; break;
          case WC_COR: m = cor; break;
          case WC_UNS: m = uns; break;
          case WC_ERR: m = errb; break;
          default: break;
        }
        cntl += lane == WC_MB ? mb : (u64)__popc(m);
      } else if (lane == 0) {
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
          const u32 lo = rec_get(2 * w);
          const u32 hi = (2 * w + 1 < P.rec_words32) ? rec_get(2 * w + 1) : 0u;
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
          if (spn) narrow_dump_phase(O.amps + sl * stride, 1u << sk, spn);
        }
      }
    }
    __syncwarp();
  }
#undef AN
  if (kReg) flush_counter_regs(O, cntl, lane);
  else flush_counters(O, wcnt, lane);
}

// ---------------------------------------------------------------- wide

#define GS_WIDE_SPARSE 0
#include "gs_wide.cuh"
#undef GS_WIDE_SPARSE
#define GS_WIDE_SPARSE 1
#include "gs_wide.cuh"
#undef GS_WIDE_SPARSE

// ---------------------------------------------------------------- section stats
// GS_SECTION_STATS (measurement only): after a section launch, on its stream,
// attribute the SURVEY §8(d) model bytes it executed: shots that finished in
// it added their totals to the MODEL_BYTES counter (delta since the last
// snapshot), shots it handed on carry their running totals in Q_MB, shots it
// received brought theirs in.  st = [shots_in, shots_out, model_bytes, -].
__global__ void mb_snapshot_kernel(const long long *mb_counter, u64 *mb_prev) {
  *mb_prev = (u64)*mb_counter;
}

__global__ void section_stats_kernel(const u64 *q_in, const u32 *n_in, u64 fresh,
                                     const u64 *q_out, const u32 *n_out, u32 su,
                                     const long long *mb_counter, u64 *mb_prev, u64 *st) {
  const u64 nin = q_in ? (u64)*n_in : fresh;
  const u64 nout = q_out ? (u64)*n_out : 0ull;
  const u64 nq = q_in ? (nin > nout ? nin : nout) : nout;
  u64 acc = 0;   // out - in, two's complement
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += (u64)gridDim.x * blockDim.x) {
    if (q_in && i < nin) acc -= q_in[i * su + Q_MB];
    if (i < nout) acc += q_out[i * su + Q_MB];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
  if ((threadIdx.x & 31u) == 0 && acc) atomicAdd((unsigned long long *)st + 2, acc);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const u64 now = (u64)*mb_counter;
    atomicAdd((unsigned long long *)st + 2, now - *mb_prev);
    *mb_prev = now;
    atomicAdd((unsigned long long *)st + 0, nin);
    atomicAdd((unsigned long long *)st + 1, nout);
  }
}
