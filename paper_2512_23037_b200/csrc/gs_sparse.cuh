// gs_sparse.cuh -- sparse chi for the warp-per-shot kernel (run flag GS_SPARSE).
// Part of gs_kernels.cu (one translation unit; included inside namespace gs).
//
// The dense forms hold chi over all 2^k coordinates of the static span.  A
// circuit whose T gates cancel (or whose support stays far below 2^k) keeps
// k growing while the reference's map holds a handful of entries (ref
// state.py:294-306) -- past the dense dimension limit such shots would end
// UNSUPPORTED.  The sparse form stores the nonzero entries alone, as an
// unordered list of (coordinate, amplitude) pairs in two global buffers
// (ping-pong, 2 x capacity entries each).  The two passes that need a
// partner's value (T butterflies, span pivots; partner = key ^ cb) find it
// by a warp match on the pair's id when the list fits one warp round (<= 32
// entries), else through a per-warp open-addressing hash table (coordinate
// -> list index; generation-tagged, so filling it for a pass never clears
// it).  Every entry's arithmetic is the dense passes' (gs_sweeps.cuh) with
// an absent partner read as the zero the dense array would hold, so
// amplitudes agree bit for bit with the warp form; only the order of the
// norm sums differs (a few ulps, as between the reference and the dense
// forms).  Coordinates are u32 (k <= 30, compiler.py); list indices fit the
// table entries' 16-bit field (capacity <= 2^16, checked on the host).
#pragma once

#ifndef GS_SPARSE_MINB
#define GS_SPARSE_MINB 1   // resident 14-warp blocks per SM the register budget targets
#endif
#ifndef GS_SPARSE_GB
#define GS_SPARSE_GB 8     // workspace budget (GB) bounding the resident warps
#endif

// @region sparse
struct SpChi {
  u32 *key;        // current list: coordinates
  double2 *amp;    //               amplitudes
  u32 n;           // entries (all nonzero)
  u32 cur;         // buffer holding the list
  u32 *kb[2];      // ping-pong buffers of `cap2` entries
  double2 *ab[2];
  u32 cap2;
  u64 *tab;        // hash table, 2^hbits slots: gen << 48 | key << 16 | index
  u32 hbits;
  u32 hcur;        // slots in use by the current fill: the 2^hcur >= 2n prefix
                   // (a compact region for short lists: better L2 locality)
  u32 gen;         // generation of the current fill (0: table not yet cleared)
};

// workspace geometry for a capacity (host and device): per warp [hash
// table: 2^hbits u64][2 x cap2 keys][2 x cap2 amplitudes], cap2 = 2 x
// capacity (a T at most doubles the <= capacity entries it starts from),
// 2^hbits >= 2 x capacity slots (load <= 1/2)
struct SpGeo {
  u32 cap2, hbits;
  u64 stride;   // bytes per warp
};
__host__ __device__ __forceinline__ SpGeo sp_geometry(u64 cap) {
  SpGeo g;
  g.hbits = 6;
  while ((1ull << g.hbits) < 2ull * cap) ++g.hbits;
  g.cap2 = (u32)(2 * cap);
  g.stride = (8ull << g.hbits) + 40ull * g.cap2;
  return g;
}

__device__ __forceinline__ void sp_init(SpChi &s, u8 *ws, u32 cap2, u32 hbits) {
  s.tab = reinterpret_cast<u64 *>(ws);
  s.hbits = hbits;
  s.hcur = hbits;
  u8 *p = ws + (8ull << hbits);
  s.kb[0] = reinterpret_cast<u32 *>(p);
  s.kb[1] = s.kb[0] + cap2;
  s.ab[0] = reinterpret_cast<double2 *>(p + 8ull * cap2);
  s.ab[1] = s.ab[0] + cap2;
  s.cap2 = cap2;
  s.gen = 0;
  s.cur = 0;
  s.key = s.kb[0];
  s.amp = s.ab[0];
  s.n = 0;
}

// a new shot: chi = |0>
__device__ __forceinline__ void sp_reset(SpChi &s, u32 lane) {
  s.cur = 0;
  s.key = s.kb[0];
  s.amp = s.ab[0];
  s.n = 1;
  if (lane == 0) {
    s.key[0] = 0;
    s.amp[0] = make_double2(1.0, 0.0);
  }
  __syncwarp();
}

__device__ __forceinline__ u32 sp_hash(u32 key, u32 hbits) { return (key * 0x9E3779B1u) >> (32 - hbits); }

// index the current list (every key is distinct; n <= capacity <= 2^16):
// slots of older generations count as empty, and one atomicMax per entry
// claims a slot -- a newer generation always wins; within a generation the
// larger entry wins and the displaced one continues along its own probe
// sequence (it only moves forward past occupied slots, so lookups still
// reach it).  No table read before the swap, no clearing after the pass.
__device__ __forceinline__ void sp_build(SpChi &s, u32 lane) {
  if (s.gen == 0 || s.gen == 0xFFFFu) {
    const u32 hm = (1u << s.hbits) - 1u;   // first use in this launch / generations exhausted
#pragma unroll 1
    for (u32 i = lane; i <= hm; i += 32) s.tab[i] = 0;
    __syncwarp();
    s.gen = 0;
  }
  ++s.gen;
  s.hcur = max(6u, min(s.hbits, 32u - __clz(2u * s.n - 1u)));   // 2^hcur >= 2n
  const u32 hm = (1u << s.hcur) - 1u;
  const u64 g = (u64)s.gen << 48;
  // two rounds per iteration: both first swaps in flight before either
  // resolves (the swaps are L2 round trips)
#pragma unroll 1
  for (u32 i0 = 0; i0 < s.n; i0 += 64) {
    u64 ent[2], old[2];
    u32 h[2];
    bool live[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const u32 i = i0 + 32u * u + lane;
      live[u] = i < s.n;
      ent[u] = live[u] ? (g | ((u64)s.key[i] << 16) | i) : 0ull;
      h[u] = sp_hash((u32)(ent[u] >> 16), s.hcur);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
      old[u] = live[u] ? atomicMax(reinterpret_cast<unsigned long long *>(s.tab + h[u]), ent[u]) : 0ull;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (!live[u]) continue;
#pragma unroll 1
      for (;;) {
        if ((old[u] >> 48) != s.gen) break;   // an empty (older) slot: claimed
        if (old[u] < ent[u]) ent[u] = old[u]; // displaced it: re-home the old entry
        h[u] = (h[u] + 1u) & hm;              // (else taken in this fill: probe on)
        old[u] = atomicMax(reinterpret_cast<unsigned long long *>(s.tab + h[u]), ent[u]);
      }
    }
  }
  __syncwarp();
}
// list index of `key`, or -1, from its first probe (slot h, entry e);
// table reads bypass L1 (the swaps ran in L2)
__device__ __forceinline__ int sp_resolve(const SpChi &s, u32 key, u32 h, u64 e) {
  const u32 hm = (1u << s.hcur) - 1u;
#pragma unroll 1
  for (;;) {
    if ((u32)(e >> 48) != s.gen) return -1;
    if ((u32)((e >> 16) & 0xFFFFFFFFull) == key) return (int)(e & 0xFFFFu);
    h = (h + 1u) & hm;
    e = __ldcg(reinterpret_cast<const unsigned long long *>(s.tab + h));
  }
}
__device__ __forceinline__ u64 sp_probe(const SpChi &s, u32 h) {
  return __ldcg(reinterpret_cast<const unsigned long long *>(s.tab + h));
}
__device__ __forceinline__ int sp_find(const SpChi &s, u32 key) {
  const u32 h = sp_hash(key, s.hcur);
  return sp_resolve(s, key, h, sp_probe(s, h));
}

// the list index of entry (lane, key j)'s partner j ^ cb, or -1: a warp
// match on the pair id (the member with cb's top bit clear) for lists of
// <= 32 entries (list index = lane), else the hash table
__device__ __forceinline__ int sp_partner(const SpChi &s, bool small, bool act, u32 j, u32 cb, u32 lane) {
  if (small) {
    const u32 hb = 31 - __clz(cb);
    const u32 pid = act ? (((j >> hb) & 1u) ? j ^ cb : j) : (0x80000000u | lane);   // keys < 2^30
    const u32 pl = __match_any_sync(FULL, pid) & ~(1u << lane);
    return pl ? __ffs(pl) - 1 : -1;
  }
  return act ? sp_find(s, j ^ cb) : -1;
}

// warp-aggregated append of the lanes with `has` at out[base + rank]
__device__ __forceinline__ u32 sp_put(u32 *ok, double2 *oa, u32 base, bool has, u32 key, double2 v,
                                      u32 lane) {
  const u32 m = __ballot_sync(FULL, has);
  if (has) {
    const u32 p = base + __popc(m & ((1u << lane) - 1u));
    ok[p] = key;
    oa[p] = v;
  }
  return base + __popc(m);
}
// prune test with the dense passes' accounting (prune_acc)
__device__ __forceinline__ bool sp_keep(double2 v, double &sum, u32 &nz) {
  const double q = abs2(v);
  if (q > kPrune2) {
    sum = __dadd_rn(sum, q);
    nz += 1;
    return true;
  }
  return false;
}
// the finished output list (in buffer `b` at `off`) becomes the current one
__device__ __forceinline__ void sp_take(SpChi &s, u32 b, u32 off, u32 n) {
  __syncwarp();
  s.cur = b;
  s.key = s.kb[b] + off;
  s.amp = s.ab[b] + off;
  s.n = n;
}

// T with beta in span (sweep_butterfly): new[j] = a v_j + b_j v_{j^cb}; an
// entry whose partner is absent also creates the partner
template <bool kR>
__device__ __forceinline__ SumNz sp_butterfly(SpChi &s, const Gate &g, u32 lane) {
  const bool small = s.n <= 32;
  if (!small) sp_build(s, lane);
  const u32 ob = s.cur ^ 1u;
  u32 *ok = s.kb[ob];
  double2 *oa = s.ab[ob];
  SumNz r;
  r.sum = 0.0;
  r.nz = 0;
  u32 base = 0;
  const double2 Z = make_double2(0.0, 0.0);
  // two rounds per iteration: both rounds' loads and first probes in
  // flight before either resolves
#pragma unroll 1
  for (u32 i0 = 0; i0 < s.n; i0 += 64) {
    u32 j[2], p[2];
    double2 v[2], w[2];
    int ip[2];
    bool act[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const u32 i = i0 + 32u * u + lane;
      act[u] = i < s.n;
      j[u] = act[u] ? s.key[i] : 0u;
      v[u] = act[u] ? s.amp[i] : Z;
      p[u] = j[u] ^ g.cb;
      w[u] = Z;
    }
    if (small) {   // one round (n <= 32)
      ip[0] = sp_partner(s, true, act[0], j[0], g.cb, lane);
      ip[1] = -1;
    } else {
      u32 h[2];
      u64 e[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        h[u] = sp_hash(p[u], s.hcur);
        e[u] = act[u] ? sp_probe(s, h[u]) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) ip[u] = act[u] ? sp_resolve(s, p[u], h[u], e[u]) : -1;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (ip[u] >= 0) w[u] = s.amp[ip[u]];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const u32 mj = (g.dc ^ par32(j[u] & g.dmask)) << 31, mp = (g.dc ^ par32(p[u] & g.dmask)) << 31;
      const double2 nj = t_mix<kR>(g, v[u], w[u], mp);
      const bool k1 = act[u] && sp_keep(nj, r.sum, r.nz);
      base = sp_put(ok, oa, base, k1, j[u], nj, lane);
      const bool add = act[u] && ip[u] < 0;
      const double2 np = t_mix<kR>(g, Z, v[u], mj);
      const bool k2 = add && sp_keep(np, r.sum, r.nz);
      base = sp_put(ok, oa, base, k2, p[u], np, lane);
    }
  }
  sp_take(s, ob, 0, base);
  return r;
}

// T with a new basis vector k (sweep_grow): (j, a v_j), (j | 2^k, b_j v_j)
template <bool kR>
__device__ __forceinline__ SumNz sp_grow(SpChi &s, const Gate &g, u32 k, u32 lane) {
  const u32 ob = s.cur ^ 1u;
  u32 *ok = s.kb[ob];
  double2 *oa = s.ab[ob];
  SumNz r;
  r.sum = 0.0;
  r.nz = 0;
  u32 base = 0;
#pragma unroll 1
  for (u32 i0 = 0; i0 < s.n; i0 += 32) {
    const u32 i = i0 + lane;
    const bool act = i < s.n;
    u32 j = 0;
    double2 v = make_double2(0.0, 0.0);
    if (act) {
      j = s.key[i];
      v = s.amp[i];
    }
    const u32 sg = g.dc ^ par32(j & g.dmask);
    double2 lo, hi;
    if (kR) {
      const double sx = neg_if1(g.ss, sg);
      lo = make_double2(__dmul_rn(kTc, v.x), __dmul_rn(kTc, v.y));
      hi = make_double2(-__dmul_rn(sx, v.y), __dmul_rn(sx, v.x));
    } else {
      lo = cmul(g.a, v);
      hi = neg_if(cmul(g.bx0, v), sg);
    }
    const bool k1 = act && sp_keep(lo, r.sum, r.nz);
    base = sp_put(ok, oa, base, k1, j, lo, lane);
    const bool k2 = act && sp_keep(hi, r.sum, r.nz);
    base = sp_put(ok, oa, base, k2, j | (1u << k), hi, lane);
  }
  sp_take(s, ob, 0, base);
  return r;
}

// nonzeros a T would leave at the dimension limit (OP_GROW_LIMIT)
__device__ __forceinline__ u32 sp_grow_count(const SpChi &s, double2 a, double2 bx0, u32 dc, u32 dmask,
                                             double ps, u32 lane) {
  const double2 Z = make_double2(0.0, 0.0), bx1 = cneg(bx0);
  u32 nz = 0;
#pragma unroll 1
  for (u32 i = lane; i < s.n; i += 32) {
    const double2 v = ps != 1.0 ? cscale(s.amp[i], ps) : s.amp[i];
    const u32 sg = dc ^ par32(s.key[i] & dmask);
    nz += abs2(cadd(Z, cmul(a, v))) > kPrune2;
    nz += abs2(cadd(Z, cmul(sg ? bx1 : bx0, v))) > kPrune2;
  }
  return nz;
}

// diagonal phase (sweep_phase), in place
__device__ __forceinline__ void sp_phase(SpChi &s, u32 dc, u32 mask, double2 f0, double2 f1, double ps,
                                         u32 lane) {
#pragma unroll 1
  for (u32 i = lane; i < s.n; i += 32) {
    const double2 v = ps != 1.0 ? cscale(s.amp[i], ps) : s.amp[i];
    s.amp[i] = cmul(v, (dc ^ par32(s.key[i] & mask)) ? f1 : f0);
  }
  __syncwarp();
}
__device__ __forceinline__ void sp_scale(SpChi &s, double ps, u32 lane) {
#pragma unroll 1
  for (u32 i = lane; i < s.n; i += 32) s.amp[i] = cscale(s.amp[i], ps);
  __syncwarp();
}

// beta = 0 measurement weights (sweep_det_sums)
__device__ __forceinline__ double2 sp_det_sums(const SpChi &s, u32 dmask, u32 neg0, double ps, u32 lane) {
  double sp = 0.0, sm = 0.0;
#pragma unroll 1
  for (u32 i = lane; i < s.n; i += 32) {
    const double2 v = ps != 1.0 ? cscale(s.amp[i], ps) : s.amp[i];
    const double a2 = abs2(v);
    if (neg0 ^ par32(s.key[i] & dmask)) sm = __dadd_rn(sm, a2); else sp = __dadd_rn(sp, a2);
  }
  return make_double2(sp, sm);
}

// keep the chosen eigen-entries scaled by rs (sweep_filter)
__device__ __forceinline__ SumNz sp_filter(SpChi &s, u32 dmask, u32 neg0, u32 want_neg, double rs,
                                           double ps, u32 lane) {
  const u32 ob = s.cur ^ 1u;
  SumNz r;
  r.sum = 0.0;
  r.nz = 0;
  u32 base = 0;
#pragma unroll 1
  for (u32 i0 = 0; i0 < s.n; i0 += 32) {
    const u32 i = i0 + lane;
    bool has = false;
    u32 j = 0;
    double2 w = make_double2(0.0, 0.0);
    if (i < s.n) {
      j = s.key[i];
      if ((neg0 ^ par32(j & dmask)) == want_neg) {
        const double2 v = ps != 1.0 ? cscale(s.amp[i], ps) : s.amp[i];
        w = cscale(v, rs);
        has = nonzero(w);
        if (has) {
          r.sum = __dadd_rn(r.sum, abs2(w));
          r.nz += 1;
        }
      }
    }
    base = sp_put(s.kb[ob], s.ab[ob], base, has, j, w, lane);
  }
  sp_take(s, ob, 0, base);
  return r;
}

// drop coordinate isq keeping the entries j = src(del(j)) (sweep_compact_move):
// moved with the pending scale applied; returns the nonzero count
__device__ __forceinline__ u32 sp_compact_move(SpChi &s, u32 isq, u32 mask, u32 tau, double ps, u32 lane) {
  const u32 ob = s.cur ^ 1u;
  const u32 lo = (1u << isq) - 1u;
  u32 base = 0;
#pragma unroll 1
  for (u32 i0 = 0; i0 < s.n; i0 += 32) {
    const u32 i = i0 + lane;
    bool has = false;
    u32 jp = 0;
    double2 v = make_double2(0.0, 0.0);
    if (i < s.n) {
      const u32 j = s.key[i];
      const u32 j0 = j & ~(1u << isq);
      if (((j >> isq) & 1u) == (tau ^ par32(j0 & mask))) {
        v = ps != 1.0 ? cscale(s.amp[i], ps) : s.amp[i];
        has = nonzero(v);
        jp = (j & lo) | ((j >> 1) & ~lo);
      }
    }
    base = sp_put(s.kb[ob], s.ab[ob], base, has, jp, v, lane);
  }
  sp_take(s, ob, 0, base);
  return base;
}

// span pivot in one pass (sweep_pivot_both): pairs (rep, rep ^ cb), rep =
// j0 | ((ct ^ par(j0 & tmask)) << isq); a pair is handled by its rep entry,
// or by its part entry when the rep is absent; w+ goes to the other buffer
// at 0, w- at cap2 / 2, both keyed by the rep with coordinate isq removed
__device__ __forceinline__ PivotBoth sp_pivot_both(SpChi &s, const PivotGeo &g, double2 xpp, double ps,
                                                   u32 &np, u32 &nm, u32 lane) {
  const bool small = s.n <= 32;
  if (!small) sp_build(s, lane);
  const u32 ob = s.cur ^ 1u;
  const u32 half = s.cap2 >> 1;
  const u32 lo = (1u << g.isq) - 1u;
  const double2 xpm = cneg(xpp), Z = make_double2(0.0, 0.0);
  PivotBoth r;
  r.pp = 0.0; r.sump = 0.0; r.summ = 0.0;
  r.nzp = 0; r.nzm = 0;
  u32 bp = 0, bm = 0;
  // two rounds per iteration, both rounds' partner probes in flight first
  // (as sp_butterfly)
#pragma unroll 1
  for (u32 i0 = 0; i0 < s.n; i0 += 64) {
    u32 j[2];
    int ip[2];
    bool in[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const u32 i = i0 + 32u * u + lane;
      in[u] = i < s.n;
      j[u] = in[u] ? s.key[i] : 0u;
    }
    if (small) {   // one round (n <= 32)
      ip[0] = sp_partner(s, true, in[0], j[0], g.cb, lane);
      ip[1] = -1;
    } else {
      u32 h[2];
      u64 e[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        h[u] = sp_hash(j[u] ^ g.cb, s.hcur);
        e[u] = in[u] ? sp_probe(s, h[u]) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) ip[u] = in[u] ? sp_resolve(s, j[u] ^ g.cb, h[u], e[u]) : -1;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const u32 i = i0 + 32u * u + lane;
      bool act = in[u];
      u32 rep = 0, part = 0;
      double2 vr = Z, vp = Z;
      if (act) {
        const double2 v = ps != 1.0 ? cscale(s.amp[i], ps) : s.amp[i];
        const u32 j0 = j[u] & ~(1u << g.isq);
        if (((j[u] >> g.isq) & 1u) == (g.ct ^ par32(j0 & g.tmask))) {
          rep = j[u];
          part = j[u] ^ g.cb;
          vr = v;
          if (ip[u] >= 0) vp = ps != 1.0 ? cscale(s.amp[ip[u]], ps) : s.amp[ip[u]];
        } else {
          part = j[u];
          rep = j[u] ^ g.cb;
          vp = v;
          act = ip[u] < 0;   // else the rep entry handles the pair
        }
      }
      const double2 pr = cmul((g.dc ^ par32(part & g.dmask)) ? xpm : xpp, vp);
      const double2 wp = cadd(vr, pr), wm = csub(vr, pr);
      if (act) r.pp = __dadd_rn(r.pp, abs2(wp));
      const u32 key = (rep & lo) | ((rep >> 1) & ~lo);
      const bool kp = act && sp_keep(wp, r.sump, r.nzp);
      bp = sp_put(s.kb[ob], s.ab[ob], bp, kp, key, wp, lane);
      const bool km = act && sp_keep(wm, r.summ, r.nzm);
      bm = sp_put(s.kb[ob] + half, s.ab[ob] + half, bm, km, key, wm, lane);
    }
  }
  __syncwarp();
  np = bp;
  nm = bm;
  return r;
}

// no-span pivot (pivot_terms, span = false): rep entries keep v, part
// entries -- ct ^ par(j & tmask) = 1 -- become +-(+-i^xi0) v.  Without a
// pending scale an in-place rotation (sweep_pivot_part); with one, the
// pruned rewrite of sweep_pivot_w
__device__ __forceinline__ void sp_pivot_part(SpChi &s, const PivotGeo &g, double2 xpp, bool plus, u32 lane) {
  const double2 xp = plus ? xpp : cneg(xpp), xm = cneg(xp);
#pragma unroll 1
  for (u32 i = lane; i < s.n; i += 32) {
    const u32 m = s.key[i];
    if (g.ct ^ par32(m & g.tmask)) s.amp[i] = cmul((g.dc ^ par32(m & g.dmask)) ? xm : xp, s.amp[i]);
  }
  __syncwarp();
}
__device__ __forceinline__ SumNz sp_pivot_w(SpChi &s, const PivotGeo &g, double2 xpp, bool plus, double ps,
                                            u32 lane) {
  const u32 ob = s.cur ^ 1u;
  const double2 xpm = cneg(xpp);
  SumNz r;
  r.sum = 0.0;
  r.nz = 0;
  u32 base = 0;
#pragma unroll 1
  for (u32 i0 = 0; i0 < s.n; i0 += 32) {
    const u32 i = i0 + lane;
    const bool act = i < s.n;
    u32 m = 0;
    double2 w = make_double2(0.0, 0.0);
    if (act) {
      m = s.key[i];
      const double2 v = ps != 1.0 ? cscale(s.amp[i], ps) : s.amp[i];
      double2 vr, pr;
      if (g.ct ^ par32(m & g.tmask)) {
        vr = make_double2(0.0, 0.0);
        pr = cmul((g.dc ^ par32(m & g.dmask)) ? xpm : xpp, v);
      } else {
        vr = v;
        pr = make_double2(-0.0, -0.0);
      }
      w = plus ? cadd(vr, pr) : csub(vr, pr);
    }
    const bool k = act && sp_keep(w, r.sum, r.nz);
    base = sp_put(s.kb[ob], s.ab[ob], base, k, m, w, lane);
  }
  sp_take(s, ob, 0, base);
  return r;
}
