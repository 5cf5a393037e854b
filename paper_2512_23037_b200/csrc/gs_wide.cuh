// gs_wide.cuh -- the warp/block-per-shot section kernel body, included twice
// by gs_sections.cuh: GS_WIDE_SPARSE 0 -> wide_kernel<kSmemChi, kPhilox, kG>
// (dense chi), 1 -> sparse_kernel<kPhilox> (the sp_* list passes of
// gs_sparse.cuh).  The dense text is kept free of sparse code so its
// instantiations compile exactly as they would alone.
// (no include guard: included once per GS_WIDE_SPARSE value)

// @region wide: prologue
#if GS_WIDE_SPARSE
// sparse_kernel: warp per shot on the sparse chi of gs_sparse.cuh (one
// section, the whole program); the dense forms' body with the chi passes
// swapped for the sp_* list passes
template <bool kPhilox>
__global__ void __launch_bounds__(32 * GS_WIDE_WARPS, GS_SPARSE_MINB)
sparse_kernel(DevProg P, DevRun R, DevOut O, DevSec S) {
  constexpr bool kSmemChi = false;
  constexpr int kG = 1;
#else
// kG = 1: warp per shot, kG > 1: block of kG warps per shot (large chi,
// see GroupScratch)
template <bool kSmemChi, bool kPhilox, int kG>
#ifdef GS_WIDE_MAXREG
__global__ void __maxnreg__(GS_WIDE_MAXREG)
#else
__global__ void __launch_bounds__(kG == 1 ? 32 * GS_WIDE_WARPS : 32 * kG,
                                  kG == 1 ? GS_WIDE_BLOCKS : (kG == 8 ? 2 : GS_BLOCK_MINB))
#endif
wide_kernel(DevProg P, DevRun R, DevOut O, DevSec S) {
#endif
  extern __shared__ __align__(16) u8 smem[];
  const u32 lane = threadIdx.x & 31u;
  const u32 wib = threadIdx.x >> 5;
  const u32 wpb = blockDim.x >> 5;
  const u64 gw = (u64)blockIdx.x * wpb + wib;
  u8 *mine = smem + (size_t)wib * O.warp_bytes;
  // warp form (kReg): the shot counters and (up to 32) record words live in
  // registers -- lane i holds counter i and record word i -- so a warp's
  // shared-memory slice is chi alone (plus the SplitMix fire-bit ring) and
  // 14 warps fit an SM at 16 KB of chi instead of 13 (host: rec_local = 1
  // means "record words in registers" for this form); the block form keeps
  // both in its per-warp slices
  constexpr bool kReg = kG == 1;
  const bool rec_reg = kReg && O.rec_local;
  u64 cntl = 0;   // kReg: counter WC_[lane]
  u32 rwl = 0;    // rec_reg: record word [lane]
  unsigned long long *wcnt = kReg ? nullptr : reinterpret_cast<unsigned long long *>(mine);
  u32 *win = reinterpret_cast<u32 *>(mine + (kReg ? 0u : kCntBytes));
  u32 *recw = rec_reg ? nullptr
              : (O.rec_local ? reinterpret_cast<u32 *>(mine + kCntBytes + kWinBytes)
                               : O.grec + gw * (u64)P.rec_words32);
  // block form: per-warp slices, then the group scratch, then chi
  const u32 gl = glane<kG>();
  constexpr u32 NT = 32u * kG;
  const bool leader = kG == 1 || wib == 0;   // the warp that writes outputs
  GroupScratch grp;
  grp.slots = reinterpret_cast<u64 *>(smem + (size_t)wpb * O.warp_bytes);
  grp.tog = 0;
  // block form on global memory (kPP): two chi buffers per block of 1.5 x
  // 2^max_dim entries each (ping-pong).  The compacting passes write the
  // other buffer in one pass without per-round barriers; a span pivot writes
  // both outcomes' compacted halves there (w+ at [0, half), w- at [half,
  // 2 half)) while it sums P+, and chi continues at the chosen half -- so a
  // later growth to 2^max_dim from an offset of half still fits
  constexpr bool kPP = kG > 1 && !kSmemChi;
  const u64 pp_stride = ((u64)3 << P.max_dim) >> 1;
  double2 *A = kSmemChi ? chi_ptr<true>(reinterpret_cast<double2 *>(
                              kG == 1 ? mine + O.chi_off : smem + O.chi_off))
                        : O.gchi + (kG == 1 ? gw * ((u64)1 << P.max_dim) : 2ull * blockIdx.x * pp_stride);
  double2 *const b0 = A;
  double2 *const b1 = kPP ? A + pp_stride : nullptr;
  u32 cur = 0;   // kPP: the buffer A lies in
#if GS_WIDE_SPARSE
  SpChi spc;
  {
    const SpGeo sg = sp_geometry(R.cap);
    sp_init(spc, reinterpret_cast<u8 *>(O.gchi) + gw * sg.stride, sg.cap2, sg.hbits);
  }
#endif
  const u32 n = P.n;
  const u64 *__restrict__ ops = P.ops;
  const u64 *__restrict__ tables = P.tables;
  const u64 *__restrict__ locs = P.locs;
  const double2 Z = make_double2(0.0, 0.0);
  constexpr bool philox = kPhilox;
  const u32 sign_bytes = 2u * ((2u * n + 7u) / 8u);
  const u32 SU = slot_u64(P);
  (void)n;

  if (!kReg && lane < WC_N) wcnt[lane] = 0;
  __syncwarp();
  const u64 total = S.q_in ? (u64)*S.n_in : S.count;
  // record-bit access (registers or memory), warp-uniform / per-lane index
  auto rec_bit = [&](u32 idx) -> u32 {
    if (rec_reg) return (__shfl_sync(FULL, rwl, idx >> 5) >> (idx & 31)) & 1u;
    return (recw[idx >> 5] >> (idx & 31)) & 1u;
  };

#pragma unroll 1
  for (;;) {
    // @region wide: shot setup
    u64 idx = 0;
    if (gl == 0) idx = atomicAdd(S.work, 1ull);
    idx = group_bcast<kG>(idx, grp);
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
    // after a deferred renormalisation the norm sits in thread 0's nrm_l
    // alone and every thread knows it (nrm_u): the reduction would return
    // exactly nrm_u (x + 0.0 == x), so consecutive dmask = 0 measurements
    // skip it
    bool nrm_lane0 = false;
    double nrm_u = 0.0;
    if (!S.q_in) {
      sl = S.first + idx;
      rng.shot = R.shot_begin + sl;
      rng.seed = 0;
      if (!philox) rng.seed = R.seeds ? R.seeds[sl] : sha1_seed(R.master, rng.shot);
      if (rec_reg) rwl = 0;
      else {
#pragma unroll 1
        for (u32 w = lane; w < P.rec_words32; w += 32) recw[w] = 0;
      }
#if GS_WIDE_SPARSE
      sp_reset(spc, lane);
#else
      if (gl == 0) A[0] = make_double2(1.0, 0.0);
#endif
      nrm_l = gl == 0 ? 1.0 : 0.0;
      nrm_lane0 = true;
      nrm_u = 1.0;
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
      if (rec_reg) rwl = lane < P.rec_words32 ? qr[lane] : 0u;
      else {
#pragma unroll 1
        for (u32 w = lane; w < P.rec_words32; w += 32) recw[w] = qr[w];
      }
      // chi in, and its norm (same per-lane order + tree as a sum pass)
      const double2 *qc = reinterpret_cast<const double2 *>(q + Q_HDR + rec_u64(P.rec_words32));
#if !GS_WIDE_SPARSE   // (the sparse form runs as one section)
#pragma unroll 1
      for (u32 j = gl; j < (1u << k); j += NT) {
        const double2 v = qc[j];
        A[j] = v;
        nrm_l = __dadd_rn(nrm_l, abs2(v));
      }
#endif
    }
    if (!philox) fire_pc = 0xFFFFFFFFu;
    if (kG > 1) __syncthreads();   // chi init before the first pass
    u32 kcur = k;
    u32 pn = S.pn0;   // chi = e^{i pi pn / 8} * A (reduced T ops, TF_RED)
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
      if (wpc == S.pc_end) { exit_pc = wpc; break; }   // the next (narrow) section starts
      // @region wide: noise
      if (wpc >= next_word_pc || wpc >= fire_pc) {
        // apply E = OR of fired letters of one noise instruction
        // (ref noise.py:68-100, state.py:88-102)
        auto apply_error = [&](u64 ex, u64 ez, const u64 *nrec) {
          if (!(ex | ez)) return;
          const ErrAct e = compose_error(tables, ex, ez, __ldg(nrec + 2), __ldg(nrec + 3),
                                         sig_lo, sig_hi);
          const double2 php = ipow(e.xi);
#if GS_WIDE_SPARSE
          sp_phase(spc, par64(e.delt & c), e.dm, php, cneg(php), ps, lane);
#else
          sweep_phase<kSmemChi, kG>(A, 1u << kcur, par64(e.delt & c), e.dm, php, cneg(php), ps);
#endif
          ps = 1.0;
          gsync<kG>();
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
          // SplitMix: one fire draw per location, 32 locations per ballot,
          // into a ring of kWinWords fire-bit words.  A stretch of more than
          // kWinWords words inserted before one op is scanned in bounded
          // steps: the words still to be read lie at or above `low` (the
          // search resumes at max(search_w, cursor / 32), and the owner of a
          // fire found there starts at most 33 words earlier -- <= 1024
          // locations per instruction, compiler.py), and an instruction is
          // applied only once all its words are scanned (the scan then keeps
          // its first word live: <= 33 words per instruction < kWinWords)
          u32 pend_lo = 0xFFFFFFFFu;   // first word of an instruction waiting for its last words
          for (;;) {
            const u32 low = pend_lo != 0xFFFFFFFFu ? max(cursor >> 5, pend_lo)
                                                   : max(cursor >> 5, search_w > 33u ? search_w - 33u : 0u);
            while (scanned < P.nwords && scanned - low < (u32)kWinWords &&
                   __ldg(tables + P.wordpc_off + scanned) <= wpc) {
              const u32 l = scanned * 32u + lane;
              bool fire = false;
              if (l < P.nlocs) {
                const u64 lw = __ldg(locs + 2ull * l), thr = __ldg(locs + 2ull * l + 1);
                fire = rng.m53((u32)lw) < thr;
              }
              const u32 bits = __ballot_sync(FULL, fire);
              if (lane == 0) win[scanned % (u32)kWinWords] = bits;
              ++scanned;
            }
            __syncwarp();
            fire_pc = 0xFFFFFFFFu;
            bool need_scan = false;
#pragma unroll 1
            for (;;) {
              // next fired location >= cursor among the scanned words
              u32 fl_loc = 0xFFFFFFFFu;
              u32 w = max(search_w, cursor >> 5);
#pragma unroll 1
              for (; w < scanned; ++w) {
                u32 bits = win[w % (u32)kWinWords];
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
              if (((loc0 + nloc + 31u) >> 5) > scanned) { need_scan = true; pend_lo = loc0 >> 5; break; }
              pend_lo = 0xFFFFFFFFu;
              cursor = loc0 + nloc;
              u64 ex = 0, ez = 0;
#pragma unroll 1
              for (u32 i = lane; i < nloc; i += 32) {
                const u32 l = loc0 + i;
                if (!((win[(l >> 5) % (u32)kWinWords] >> (l & 31)) & 1u)) continue;
                const u64 lw = __ldg(locs + 2ull * l);
                const u32 nk = (u32)(lw >> 48) & 3;
                const double u = nk <= NK_DEP2 ? rng.uniform((u32)lw + 1) : 0.0;
                noise_letter(nk, (u32)(lw >> 32) & 0xff, (u32)(lw >> 40) & 0xff, u, ex, ez);
              }
              apply_error(warp_or64(ex), warp_or64(ez), nrec);
            }
            const bool more = scanned < P.nwords && __ldg(tables + P.wordpc_off + scanned) <= wpc;
            if (!more && !need_scan) break;
          }
          next_word_pc = scanned < P.nwords ? (u32)__ldg(tables + P.wordpc_off + scanned) : 0xFFFFFFFFu;
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
        // TF_RED: BUTTERFLY / GROW in the reduced form (global phase counted
        // in pn, see t_mix); word 12: bit 0 = sign of ss, bit 1 = T_DAG
        const bool red = (wfl & TF_RED) != 0;
        if (tcase == T_DIAG) {
          // beta == 0: pure phase per entry (ref state.py:120-126); the
          // factors have modulus 1, the norm is kept
#if GS_WIDE_SPARSE
          sp_phase(spc, dc, dmask, cadd(a, bx0), cadd(a, cneg(bx0)), ps, lane);
#else
          sweep_phase<kSmemChi, kG>(A, size, dc, dmask, cadd(a, bx0), cadd(a, cneg(bx0)), ps);
#endif
          ps = 1.0;
          gsync<kG>();
          mbytes += 32ull * cnt;
          continue;
        }
        const u32 cin = cnt;
        if (wkind == OP_GROW_LIMIT) {
          u32 nz = 0;
          const double2 bx1 = cneg(bx0);
          gbar_in<kG>();
#if GS_WIDE_SPARSE
          nz = sp_grow_count(spc, a, bx0, dc, dmask, ps, lane);
#else
#pragma unroll 1
          for (u32 j = gl; j < size; j += NT) {
            const double2 v = ldps(A, j, ps);
            const u32 s_ = dc ^ par32(j & dmask);
            nz += abs2(cadd(Z, cmul(a, v))) > kPrune2;
            nz += abs2(cadd(Z, cmul(s_ ? bx1 : bx0, v))) > kPrune2;
          }
#endif
          nz = group_sum_u32<kG>(nz, grp);
          status = (u64)nz > R.cap ? ST_OVERFLOW : ST_UNSUPPORTED;
          aux = (int)winstr;
          break;
        }
        // beta != 0: pair merge + prune (ref state.py:127-129, 294-306)
#if GS_WIDE_SPARSE
        if (ps != 1.0) sp_scale(spc, ps, lane);   // rare: right after a deferral
#else
        if (ps != 1.0) sweep_scale<kSmemChi, kG>(A, size, ps);   // rare: right after a deferral
#endif
        ps = 1.0;
        // TF_FUSEQ: the partner follows a noise insertion; fusable when no
        // location there fires for this shot: Philox -- its schedule has no
        // candidate up to the partner (fire_pc > its pc); SplitMix -- every
        // fire-bit word that can hold those locations is scanned
        // (next_word_pc > its pc; always true in Philox mode) and none fired
        if (tcase == T_BUTTERFLY &&
            ((wfl & TF_FUSE) || ((wfl & TF_FUSEQ) && fire_pc > wpc && next_word_pc > wpc))) {
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
          g1.ss = 0.0; g2.ss = 0.0;
          if (red) {   // the compiler fuses only pairs of the same form
            const u64 w12 = __ldg(op + 12), w122 = __ldg(op2 + 12);
            g1.ss = neg_if1(kTs, ((u32)w12 & 1u) ^ flip);
            g2.ss = neg_if1(kTs, ((u32)w122 & 1u) ^ flip2);
            pn = (pn + ((w12 & 2u) ? 15u : 1u) + ((w122 & 2u) ? 15u : 1u)) & 15u;
          }
          g2.a = make_double2(dbits(__ldg(op2 + 7)), dbits(__ldg(op2 + 8)));
          const double2 bxs2 = make_double2(dbits(__ldg(op2 + 9)), dbits(__ldg(op2 + 10)));
          g2.bx0 = flip2 ? cneg(bxs2) : bxs2;
          g2.cb = (u32)w62;
          g2.dmask = (u32)(w62 >> 32);
          g2.dc = par64(__ldg(op2 + 5) & c);
          mbytes += __ldg(op2 + 11);
          wpc += (u32)((h2 >> 8) & 0xff);
          hnext = __ldg(ops + wpc);
#if GS_WIDE_SPARSE
          // two single-gate passes (the fused pass's arithmetic); the
          // second only while the first stayed within the capacity
          SumNz2 r2;
          {
            const SumNz s1 = red ? sp_butterfly<true>(spc, g1, lane) : sp_butterfly<false>(spc, g1, lane);
            r2.nz1 = s1.nz;
            r2.nz = 0;
            r2.sum = 0.0;
            const u32 c1 = warp_sum_u32(s1.nz);
            if ((u64)c1 <= R.cap && c1 > 0) {
              const SumNz s2 = red ? sp_butterfly<true>(spc, g2, lane) : sp_butterfly<false>(spc, g2, lane);
              r2.nz = s2.nz;
              r2.sum = s2.sum;
            }
          }
#else
          const SumNz2 r2 = red ? sweep_butterfly2<kSmemChi, kG, true>(A, size >> 2, g1, g2)
                                : sweep_butterfly2<kSmemChi, kG, false>(A, size >> 2, g1, g2);
#endif
          gsync<kG>();
          const u32 cnt1 = group_sum_u32<kG>(r2.nz1, grp);
          mbytes += (u64)kEntryBytes * (cin + cnt1);
          if ((u64)cnt1 > R.cap) { status = ST_OVERFLOW; aux = (int)winstr; break; }
          if (cnt1 == 0) { status = ST_CORRUPT; aux = (int)winstr; break; }
          cnt = group_sum_u32<kG>(r2.nz, grp);
          nrm_l = r2.sum;
          nrm_lane0 = false;
          mbytes += (u64)kEntryBytes * (cnt1 + cnt);
          if ((u64)cnt > R.cap) { status = ST_OVERFLOW; aux = (int)instr2; break; }
          if (cnt == 0) { status = ST_CORRUPT; aux = (int)instr2; break; }
          continue;
        }
        Gate g;
        g.a = a; g.bx0 = bx0; g.cb = cb; g.dc = dc; g.dmask = dmask;
        g.ss = 0.0;
        if (red) {
          const u64 w12 = __ldg(op + 12);
          g.ss = neg_if1(kTs, ((u32)w12 & 1u) ^ flip);
          pn = (pn + ((w12 & 2u) ? 15u : 1u)) & 15u;
        }
        SumNz r;
#if GS_WIDE_SPARSE
        if (tcase == T_BUTTERFLY) {
          r = red ? sp_butterfly<true>(spc, g, lane) : sp_butterfly<false>(spc, g, lane);
        } else {
          r = red ? sp_grow<true>(spc, g, wk, lane) : sp_grow<false>(spc, g, wk, lane);
          kcur = wk + 1;
        }
#else
        if (tcase == T_BUTTERFLY) {
          r = red ? sweep_butterfly<kSmemChi, kG, true>(A, size >> 1, g)
                  : sweep_butterfly<kSmemChi, kG, false>(A, size >> 1, g);
        } else {
          r = red ? sweep_grow<kSmemChi, kG, true>(A, size, g) : sweep_grow<kSmemChi, kG, false>(A, size, g);
          kcur = wk + 1;
        }
#endif
        gsync<kG>();
        cnt = group_sum_u32<kG>(r.nz, grp);
        nrm_l = r.sum;
        nrm_lane0 = false;
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
          // a factor of exactly 1 changes no entry: any pending scale stays
          // pending instead of being applied by a pass now
          if (rs != 1.0) {
#if GS_WIDE_SPARSE
            if (ps != 1.0) sp_scale(spc, ps, lane);
#else
            if (ps != 1.0) sweep_scale<kSmemChi, kG>(A, size, ps);
#endif
            ps = rs;
          }
          nrm_u = __dmul_rn(__dmul_rn(kept, rs), rs);
          nrm_l = gl == 0 ? nrm_u : 0.0;
          nrm_lane0 = true;
        };
        const u32 cin = cnt;
        bool plus;
        if (mcase == M_DET) {
          // beta == 0: filter by eigenvalue (ref state.py:162-176)
          const u32 neg0 = (xi0 >> 1) ^ dc;
          double sp, sm;
          if (dmask == 0) {
            // every coordinate has eigenvalue (-1)^neg0: P+ is the norm
            const double nrm = nrm_lane0 ? nrm_u : group_sum<kG>(nrm_l, grp);
            sp = neg0 ? 0.0 : nrm;
            sm = neg0 ? nrm : 0.0;
          } else {
#if GS_WIDE_SPARSE
            const double2 part = sp_det_sums(spc, dmask, neg0, ps, lane);
#else
            const double2 part = sweep_det_sums<kSmemChi, kG>(A, size, dmask, neg0, ps);
#endif
            sp = group_sum<kG>(part.x, grp);
            sm = group_sum<kG>(part.y, grp);
          }
          plus = pick_plus(sp);
          const double chosen = plus ? sp : __dsub_rn(1.0, sp);
          if (chosen < 1e-12) { status = ST_CORRUPT; aux = (int)winstr; break; }
          const u32 want_neg = plus ? 0u : 1u;
          const double rs = inv_sqrt_norm(plus ? sp : sm);
          if (wfl & MF_COMPACT) {
            const u32 tau = want_neg ^ neg0;
#if GS_WIDE_SPARSE
            if (GS_WIDE_SPARSE) {
              cnt = sp_compact_move(spc, isq, dmask, tau, ps, lane);   // (warp total)
              ps = 1.0;
              defer_scale(rs, plus ? sp : sm);
            } else if (!kPP && GS_COMPACT_DEFER) {
#else
            if (!kPP && GS_COMPACT_DEFER) {
#endif
              // move only; the renormalisation rs is deferred (ldps), as the
              // ping-pong form's compactions of span pivots do
              const u32 nzm = sweep_compact_move<kSmemChi, kG>(A, size >> 1, isq, dmask, tau, ps);
              ps = 1.0;
              gsync<kG>();
              cnt = group_sum_u32<kG>(nzm, grp);
              defer_scale(rs, plus ? sp : sm);
            } else {
              SumNz r;
              if (kPP) {
                double2 *D = cur ? b0 : b1;
                r = sweep_compact_to<kG>(A, D, size >> 1, isq, dmask, tau, rs, ps);
                A = D;
                cur ^= 1u;
              } else {
                r = sweep_compact<kSmemChi, kG>(A, size >> 1, isq, dmask, tau, rs, ps);
              }
              ps = 1.0;
              gsync<kG>();
              cnt = group_sum_u32<kG>(r.nz, grp);
              nrm_l = r.sum;
              nrm_lane0 = false;
            }
            if (tau) c ^= vec;
            kcur = wk - 1;
          } else if ((plus ? sm : sp) == 0.0) {
            // the other eigenspace is empty: the filter is a pure
            // renormalisation
            defer_scale(rs, plus ? sp : sm);
          } else {
#if GS_WIDE_SPARSE
            const SumNz r = sp_filter(spc, dmask, neg0, want_neg, rs, ps, lane);
#else
            const SumNz r = sweep_filter<kSmemChi, kG>(A, size, dmask, neg0, want_neg, rs, ps);
#endif
            ps = 1.0;
            gsync<kG>();
            cnt = group_sum_u32<kG>(r.nz, grp);
            nrm_l = r.sum;
            nrm_lane0 = false;
          }
        } else {
          // beta != 0: pair-merge + tableau pivot (ref state.py:178-208)
          PivotGeo g;
          g.span = mcase == M_PIVOT_SPAN;
          g.npairs = g.span ? (size >> 1) : size;
          g.isq = isq; g.tmask = tmask; g.ct = (u32)(c >> t) & 1u; g.cb = cb;
          g.dc = dc; g.dmask = dmask;
          const double2 xpp = ipow(xi0);   // i^xi0, exact
#if GS_WIDE_SPARSE
          if (g.span) {
            // one pass (sp_pivot_both, as sweep_pivot_both): P+ and both
            // outcomes' lists, then chi continues at the chosen one
            u32 spn_p = 0, spn_m = 0;
            const PivotBoth pb = sp_pivot_both(spc, g, xpp, ps, spn_p, spn_m, lane);
#else
          if (kPP && g.span) {
            // one pass: P+ and both outcomes' merged, pruned, compacted
            // pairs (sweep_pivot_both), then chi continues at the chosen
            // half with the renormalisation deferred
            double2 *D = cur ? b0 : b1;
            const u32 half = size >> 1;
            const PivotBoth pb = sweep_pivot_both<kG>(A, D, g, xpp, ps);
#endif
            gsync<kG>();
            const double pp = __dmul_rn(0.5, group_sum<kG>(pb.pp, grp));
            plus = pick_plus(pp);
            const double chosen = plus ? pp : __dsub_rn(1.0, pp);
            if (chosen < 1e-12) { status = ST_CORRUPT; aux = (int)winstr; break; }
            const double sk = group_sum<kG>(plus ? pb.sump : pb.summ, grp);
            cnt = group_sum_u32<kG>(plus ? pb.nzp : pb.nzm, grp);
            if (cnt == 0) { status = ST_CORRUPT; aux = (int)winstr; break; }
            ps = 1.0;
#if GS_WIDE_SPARSE
            sp_take(spc, spc.cur ^ 1u, plus ? 0u : spc.cap2 >> 1, plus ? spn_p : spn_m);
#else
            A = D + (plus ? 0u : half);
            cur ^= 1u;
#endif
            kcur = wk - 1;
            defer_scale(inv_sqrt_norm(sk), sk);
          } else {
            // no span: every entry is either its pair's rep (w = v) or its
            // part (w = +-i^xi0 v, an exact rotation), so sum |w+|^2 is the
            // chi norm the writer passes track -- no read pass
            const double nrm0 = g.span ? 0.0 : (nrm_lane0 ? nrm_u : group_sum<kG>(nrm_l, grp));
#if GS_WIDE_SPARSE
            const double pp = __dmul_rn(0.5, nrm0);   // (no span here: span pivots took the branch above)
#else
            const double pp = __dmul_rn(0.5, g.span ? group_sum<kG>(sweep_pivot_p<kSmemChi, kG>(A, g, xpp, ps), grp)
                                                    : nrm0);
#endif
            plus = pick_plus(pp);
            const double chosen = plus ? pp : __dsub_rn(1.0, pp);
            if (chosen < 1e-12) { status = ST_CORRUPT; aux = (int)winstr; break; }
            if (!g.span && ps == 1.0) {
              // rotate the part entries only; norm and count carry over
#if GS_WIDE_SPARSE
              sp_pivot_part(spc, g, xpp, plus, lane);
#else
              sweep_pivot_part<kSmemChi, kG>(A, g, xpp, plus, size);
#endif
              gsync<kG>();
              defer_scale(inv_sqrt_norm(nrm0), nrm0);
            } else {
#if GS_WIDE_SPARSE
              const SumNz w = sp_pivot_w(spc, g, xpp, plus, ps, lane);
#else
              const SumNz w = sweep_pivot_w<kSmemChi, kG>(A, g, xpp, plus, ps);
#endif
              ps = 1.0;
              gsync<kG>();
              const double sk = group_sum<kG>(w.sum, grp);
              cnt = group_sum_u32<kG>(w.nz, grp);
              if (cnt == 0) { status = ST_CORRUPT; aux = (int)winstr; break; }
              const double rs = inv_sqrt_norm(sk);
              if (!GS_WIDE_SPARSE && g.span) {   // (sparse span pivots take the one-pass branch)
                const SumNz r = sweep_compact<kSmemChi, kG>(A, size >> 1, isq, tmask, g.ct, rs, 1.0);
                gsync<kG>();
                cnt = group_sum_u32<kG>(r.nz, grp);
                nrm_l = r.sum;
                nrm_lane0 = false;
                kcur = wk - 1;
              } else {
                defer_scale(rs, sk);
              }
            }
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
          if (rec_reg) {
            if (rb && lane == (slot >> 5)) rwl |= 1u << (slot & 31);
          } else if (lane == 0 && rb) recw[slot >> 5] |= 1u << (slot & 31);
          __syncwarp();
        }
        if ((wfl & MF_RESET) && bout) { sig_lo ^= __ldg(op + 15); sig_hi ^= __ldg(op + 16); }
        continue;
      }

      // @region wide: feedback/detector/end
      if (wkind == OP_FEEDBACK) {
        const u32 idx = (u32)__ldg(op + 1);
        if (rec_bit(idx)) {
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
        for (u32 i0 = 0; i0 < nidx; i0 += 32) {   // warp-uniform trips (shuffles)
          const u32 i = i0 + lane;
          const u32 idx = i < nidx ? (u32)__ldg(tables + off + i) : 0u;
          const u32 b = rec_bit(idx);
          if (i < nidx) bb ^= b;
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
    gsync<kG>();
    if (status == ST_RUNNING) {
      // survivor: hand it to the next (narrow) section's queue
      u32 o = 0;
      if (gl == 0) o = atomicAdd(S.n_out, 1u);
      o = group_bcast32<kG>(o, grp);
      u64 *q = S.q_out + (u64)o * SU;
      if (gl == 0) {
        q[Q_SL] = sl; q[Q_LO] = sig_lo; q[Q_HI] = sig_hi; q[Q_C] = c; q[Q_OBS] = obs;
        q[Q_MB] = mbytes; q[Q_PICK] = gpick; q[Q_SEED] = rng.seed;
        q[Q_CNTK] = (u64)cnt;
        q[Q_GEO] = (u64)gj | ((u64)gpos << 32);
        q[Q_FIRE] = fire_pc;
      }
      u32 *qr = reinterpret_cast<u32 *>(q + Q_HDR);
      if (rec_reg) {
        if (lane < P.rec_words32) qr[lane] = rwl;
      } else {
#pragma unroll 1
        for (u32 w = lane; leader && w < P.rec_words32; w += 32) qr[w] = recw[w];
      }
      double2 *qc = reinterpret_cast<double2 *>(q + Q_HDR + rec_u64(P.rec_words32));
#if !GS_WIDE_SPARSE
#pragma unroll 1
      for (u32 j = gl; j < (1u << kcur); j += NT) qc[j] = ldps(A, j, ps);
#endif
      (void)exit_pc;
    } else {
      if (kReg) {
        // lane i accumulates counter i (status, obs, mbytes are warp-uniform)
        const bool pres = status == ST_PRESERVED;
        u64 add = 0;
        switch (lane) {
          case WC_TOT: add = 1; break;
          case WC_MB: add = mbytes; break;
          case WC_PRES: add = pres; break;
          case WC_ERR: add = pres && obs; break;
          case WC_DISC: add = status == ST_DISCARDED; break;
          case WC_OVF: add = status == ST_OVERFLOW; break;
          case WC_COR: add = status == ST_CORRUPT; break;
          case WC_UNS: add = !pres && status != ST_DISCARDED && status != ST_OVERFLOW &&
                             status != ST_CORRUPT; break;
          default: break;
        }
        cntl += add;
      }
      if (gl == 0) {
        if (!kReg) wcnt[WC_TOT] += 1;
        if (!kReg) wcnt[WC_MB] += mbytes;
        if (status == ST_PRESERVED) {
          if (!kReg) wcnt[WC_PRES] += 1;
          if (obs) {
            if (!kReg) wcnt[WC_ERR] += 1;
#pragma unroll 1
            for (u64 o = obs; o; o &= o - 1)
              atomicAdd((unsigned long long *)&O.counters[GS_C_PER_OBS + (__ffsll((long long)o) - 1)], 1ull);
            if (O.witness) {
              const u32 wi = atomicAdd(O.witness_count, 1u);
              if (wi < O.witness_cap) O.witness[wi] = rng.shot;
            }
          }
        } else if (kReg) {
        } else if (status == ST_DISCARDED) wcnt[WC_DISC] += 1;
        else if (status == ST_OVERFLOW) wcnt[WC_OVF] += 1;
        else if (status == ST_CORRUPT) wcnt[WC_COR] += 1;
        else wcnt[WC_UNS] += 1;
      }
      if (O.mode != MODE_COUNTERS && leader) {
        if (lane == 0) {
          O.status[sl] = (u8)status;
          O.aux[sl] = aux;
          O.obs[sl] = obs;
        }
        const u32 rw64 = (P.nmeas + 63) / 64;
        if (rec_reg) {   // <= 32 words: rw64 <= 16, one round
          const u32 lo = __shfl_sync(FULL, rwl, (2 * lane) & 31);
          const u32 hi = __shfl_sync(FULL, rwl, (2 * lane + 1) & 31);
          if (lane < rw64) O.rec[sl * rw64 + lane] = ((u64)(2 * lane + 1 < P.rec_words32 ? hi : 0u) << 32) | lo;
        } else {
#pragma unroll 1
          for (u32 w = lane; w < rw64; w += 32) {
            const u32 lo = recw[2 * w];
            const u32 hi = (2 * w + 1 < P.rec_words32) ? recw[2 * w + 1] : 0u;
            O.rec[sl * rw64 + w] = ((u64)hi << 32) | lo;
          }
        }
        if (O.mode == MODE_DUMP) {
          if (lane == 0) {
            O.sig[2 * sl] = sig_lo;
            O.sig[2 * sl + 1] = sig_hi;
            O.cvec[sl] = c;
            O.dim[sl] = kcur;
          }
          const u64 stride = 1ull << P.max_dim;
#if GS_WIDE_SPARSE   // zero, then scatter the entries
#pragma unroll 1
          for (u32 j = lane; j < (1u << kcur); j += 32) O.amps[sl * stride + j] = make_double2(0.0, 0.0);
          __syncwarp();
#pragma unroll 1
          for (u32 i = lane; i < spc.n; i += 32)
            O.amps[sl * stride + spc.key[i]] = with_phase(pn, ldps(spc.amp, i, ps));
#else
#pragma unroll 1
          for (u32 j = lane; j < (1u << kcur); j += 32)   // leader warp
            O.amps[sl * stride + j] = with_phase(pn, ldps(A, j, ps));
#endif
        }
      }
    }
    gsync<kG>();
  }
  if (kReg) flush_counter_regs(O, cntl, lane);
  else flush_counters(O, wcnt, lane);
}
