// gs_kernels.cu -- B200 (sm_100a) shot-parallel generalized-stabilizer sampler.
//
// One translation unit, split for reading:
//   gs_common.cuh   enums, device program/run/output structs, RNG (SplitMix,
//                   Philox4x32-10, geometric gap search), SHA-1 seeding
//   gs_sweeps.cuh   warp-cooperative sweeps over the dense chi vector
//   gs_sparse.cuh   the sparse chi form: nonzero-entry list passes (GS_SPARSE)
//   gs_sections.cuh the lane-per-shot section kernel, slot queues, and
//   gs_wide.cuh     the warp/block-per-shot body, instantiated twice: dense
//                   wide_kernel and sparse_kernel
//   gs_plugin.cuh   the Pauli/tableau plugin kernels (ops.py boundary)
//   this file       host side: program upload, section plan, launch loop, C ABI
//
// The op stream is cut on the host into sections (see sections_of): narrow
// sections (every op has k <= kn) run one lane per shot in narrow_kernel,
// wide sections one warp per shot in wide_kernel; surviving shots pass from
// section to section through global slot queues.  The per-shot state is the
// static-frame state of compiler.py:
//   sig  : 2n tableau sign bits (destab word, stab word)    [ref tableau.py]
//   c    : u64 coset offset of the amplitude support        [ref state.py]
//   A    : dense complex128 amplitudes over 2^k coordinates [ref state.py]
//   rec  : measurement record bits
// Everything shot-invariant (x/z tableau trajectory, pivot rows, coordinate
// basis, draw offsets) was folded into the op stream on the host.
//
// Per-element arithmetic follows the reference's numpy forms:
//   complex product  (fma(ar,br,-(ai*bi)), fma(ar,bi,ai*br))
//   |v|^2            abs2: see gs_common.cuh                     np.abs()**2
//   prune            |v|^2 > kPrune2 (numpy abs()>1e-12)     ref state.py:298
//   renormalise      v * (1/sqrt(sum |v|^2))                ref state.py:311
// except the wide kernel's T updates (TF_RED, gs_sweeps.cuh t_mix), which
// factor T = e^{+-i pi/8} (c I + b' Z) and count the global phase instead of
// multiplying it in; amplitudes agree with the reference to a few ulps
// (tests: 1e-12 absolute), records and counters exactly.

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

#include "gs_common.cuh"
#include "gs_sweeps.cuh"
#include "gs_sparse.cuh"
#include "gs_sections.cuh"
#include "gs_plugin.cuh"

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
  // cross-stream ordering: recorded after every run, waited on by the next
  // run when it is issued on a different stream (engine scratch is shared)
  cudaEvent_t order_ev = nullptr;
  cudaStream_t last_stream = nullptr;
  bool has_last = false;
  // inter-section queue budget per queue (0: auto, sized on first use)
  u64 queue_budget = 0;
  // GS_SECTION_STATS: device accumulators [sec][GS_SEC_FIELDS] (+1 word: model
  // bytes already attributed), and the pending per-launch event pairs
  u64 *d_secstats = nullptr;
  size_t secstats_cap = 0;   // sections
  struct TimedLaunch { u32 sec; cudaEvent_t a, b; };
  std::vector<TimedLaunch> timed;
  std::vector<cudaEvent_t> spare_ev;
  std::vector<u64> sec_meta;  // per section: wide, pc0 of the last stats run
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
  CUDA_TRY(cudaEventCreateWithFlags(&e->order_ev, cudaEventDisableTiming));
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
  cudaFree(e->d_secstats);
  for (auto &t : e->timed) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
  for (cudaEvent_t ev : e->spare_ev) cudaEventDestroy(ev);
  if (e->order_ev) cudaEventDestroy(e->order_ev);
  if (e->ev0) cudaEventDestroy(e->ev0);
  if (e->ev1) cudaEventDestroy(e->ev1);
  if (e->stream) cudaStreamDestroy(e->stream);
  delete e;
  return GS_OK;
}

uint64_t gs_engine_launches(gs_engine *e) { return e ? e->launches : 0; }
double gs_engine_last_kernel_ms(gs_engine *e) { return e ? e->last_ms : 0.0; }

// copies are issued on the launch stream `st`, so they are ordered before
// the kernels that read them (the engine's stream is non-blocking: legacy
// stream copies would not be); the host vectors outlive the copies
static int upload(gs_engine *e, gs_program *p, cudaStream_t st) {
  if (p->dev == e->device) return GS_OK;
  if (p->dev >= 0) return fail(GS_ERR_ARG, "program already bound to another device");
  // one zero word past END: the interpreters prefetch the next header
  CUDA_TRY(cudaMalloc(&p->d_ops, (p->ops.size() + 1) * 8));
  CUDA_TRY(cudaMalloc(&p->d_tables, std::max<size_t>(p->tables.size(), 1) * 8));
  CUDA_TRY(cudaMalloc(&p->d_locs, std::max<size_t>(p->locs.size(), 1) * 8));
  CUDA_TRY(cudaMemsetAsync(p->d_ops + p->ops.size(), 0, 8, st));
  CUDA_TRY(cudaMemcpyAsync(p->d_ops, p->ops.data(), p->ops.size() * 8, cudaMemcpyHostToDevice, st));
  if (!p->tables.empty())
    CUDA_TRY(cudaMemcpyAsync(p->d_tables, p->tables.data(), p->tables.size() * 8, cudaMemcpyHostToDevice, st));
  if (!p->locs.empty())
    CUDA_TRY(cudaMemcpyAsync(p->d_locs, p->locs.data(), p->locs.size() * 8, cudaMemcpyHostToDevice, st));
  p->dev = e->device;
  return GS_OK;
}

// static section split of the op stream (see the kernels' header comment)
struct Section {
  u32 pc0, k0, nm0;
  bool wide;
  u32 pn0;   // reduced-T phase count on entry: TF_RED ops of earlier wide sections
  u32 kn;    // narrow sections: the chi rows they need, 4 or 5 (kn_max 5 only)
};

#ifndef GS_NARROW_KSPLIT
#define GS_NARROW_KSPLIT 30  // narrow sections of >= N ops also split where the 2^5-row need changes
#endif
#ifndef GS_NARROW_SPLIT
#define GS_NARROW_SPLIT 75  // split narrow sections every N ops (0: never) so the survivors of
                            // early discards re-pack into full warps (A/B: 51.2M at 75, 49.4M unsplit,
                            // 50.6M at 150, 50.3M at 40)
#endif

static void sections_of(const gs_program *p, bool wide_only, u32 kn, std::vector<Section> &out) {
  out.clear();
  const std::vector<u64> &ops = p->ops;
  // op starts, then for every op the length of the narrow run from it to the
  // next wide op (a k-split never leaves a short tail section)
  std::vector<u32> at;
  for (size_t pc = 0; pc < ops.size();) {
    at.push_back((u32)pc);
    const u32 kind = (u32)(ops[pc] & 0xff), len = (u32)((ops[pc] >> 8) & 0xff);
    if (kind == gs::OP_END || len == 0) break;
    pc += len;
  }
  auto hdr = [&](size_t i, u32 &kind, u32 &len, u32 &k, u32 &fl) {
    const u64 h = ops[at[i]];
    kind = (u32)(h & 0xff); len = (u32)((h >> 8) & 0xff);
    k = (u32)((h >> 16) & 0xff); fl = (u32)((h >> 24) & 0xff);
  };
  std::vector<u32> run(at.size() + 1, 0);
  for (size_t i = at.size(); i-- > 0;) {
    u32 kind, len, k, fl;
    hdr(i, kind, len, k, fl);
    run[i] = (wide_only || gs::op_is_wide(kind, k, fl, kn)) ? 0u : run[i + 1] + 1u;
  }
  size_t nm = 0;
  u32 nops = 0, pn = 0;
  bool prev5 = false;
  const u32 nn = p->info.num_noise;
  for (size_t i = 0; i < at.size(); ++i) {
    const u32 pc = at[i];
    u32 kind, len, k, fl;
    hdr(i, kind, len, k, fl);
    const bool wide = wide_only || gs::op_is_wide(kind, k, fl, kn);
    // needs5: a narrow op that needs 2^5 chi rows (wide at limit 4)
    const bool needs5 = !wide && kn > 4u && gs::op_is_wide(kind, k, fl, 4u);
    bool split = !wide && (GS_NARROW_SPLIT > 0) && nops >= (u32)GS_NARROW_SPLIT;
    // a 2^4-row narrow section of >= GS_NARROW_KSPLIT ops ends where the
    // ops start needing 2^5 rows (if >= 16 narrow ops follow), so the
    // k <= 4 stretch keeps the 20-warp layout instead of inheriting the
    // 12-warp one (the Table-2 d=5 injection + d=3 round)
    if (!wide && GS_NARROW_KSPLIT > 0 && !out.empty() && !out.back().wide && out.back().kn == 4u &&
        nops >= (u32)GS_NARROW_KSPLIT && needs5 && !prev5 && run[i] >= 16u)
      split = true;
    if (out.empty() || out.back().wide != wide || split) {
      while (nm < nn && (u32)p->tables[p->info.noise_off + 4 * nm] < pc) ++nm;
      out.push_back(Section{pc, k, (u32)nm, wide, pn, 4u});
      nops = 0;
    }
    // a narrow section needs 2^5 chi rows per lane only if one of its ops
    // would be wide at limit 4; the others keep the 20-warp/SM layout
    if (needs5) out.back().kn = kn;
    prev5 = needs5;
    ++nops;
    // the wide kernel runs TF_RED ops in the reduced form (gs_sweeps.cuh
    // t_mix); every shot entering a later section executed all of them
    if ((wide || GS_NARROW_RED) && kind == gs::OP_T && (fl & gs::TF_RED) && len > 12)
      pn = (pn + ((ops[pc + 12] & 2u) ? 15u : 1u)) & 15u;
  }
}

int gs_program_sections(const gs_program *p, uint32_t flags) {
  if (!p) return fail(GS_ERR_ARG, "null argument");
  std::vector<Section> secs;
  sections_of(p, (flags & (GS_WIDE_ONLY | GS_SPARSE)) != 0, gs::narrow_kn(flags), secs);
  return (int)secs.size();
}


extern "C++" {
// the sampling kernels: RNG mode (x chi placement for the wide kernel)
template <typename F>
static cudaError_t with_narrow_kernel(bool philox, bool k5, F f) {
  if (k5) return philox ? f(gs::narrow_kernel<true, true>) : f(gs::narrow_kernel<false, true>);
  return philox ? f(gs::narrow_kernel<true, false>) : f(gs::narrow_kernel<false, false>);
}
// gw = warps sharing one shot: 1 (warp per shot), 8 or GS_BLOCK_WARPS (16)
template <typename F>
static cudaError_t with_wide_kernel(bool smem_chi, bool philox, u32 gw, F f) {
  constexpr int G = GS_BLOCK_WARPS;
  if (gw == 8) {
    if (smem_chi) return philox ? f(gs::wide_kernel<true, true, 8>) : f(gs::wide_kernel<true, false, 8>);
    return philox ? f(gs::wide_kernel<false, true, 8>) : f(gs::wide_kernel<false, false, 8>);
  }
  if (gw > 1) {
    if (smem_chi) return philox ? f(gs::wide_kernel<true, true, G>) : f(gs::wide_kernel<true, false, G>);
    return philox ? f(gs::wide_kernel<false, true, G>) : f(gs::wide_kernel<false, false, G>);
  }
  if (smem_chi) return philox ? f(gs::wide_kernel<true, true, 1>) : f(gs::wide_kernel<true, false, 1>);
  return philox ? f(gs::wide_kernel<false, true, 1>) : f(gs::wide_kernel<false, false, 1>);
}

// the sparse-chi warp-per-shot kernel (GS_SPARSE)
template <typename F>
static cudaError_t with_sparse_kernel(bool philox, F f) {
  return philox ? f(gs::sparse_kernel<true>) : f(gs::sparse_kernel<false>);
}

struct KernelCfg {
  u32 wpb = 1, blocks = 1, warp_bytes = 0, chi_off = 0, rec_local = 0;
  size_t smem = 0;
};

// warps per block = the most resident warps per SM; grid = SMs x blocks/SM
template <typename W>
static int occupancy(gs_engine *e, u32 warp_bytes, u32 want_wpb, u32 max_wpb, W with,
                     KernelCfg &K) {
  u32 wpb = 1;
  int best = -1;
  for (u32 w = max_wpb; w >= 1; --w) {
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

static int launch_body(gs_engine *e, gs_program *p, const gs_run_params *r, gs::DevOut O,
                       cudaStream_t st, bool timed);
typedef gs_engine::TimedLaunch Engine_TimedLaunch;

static int launch(gs_engine *e, gs_program *p, const gs_run_params *r, gs::DevOut O,
                  cudaStream_t st, bool timed) {
  if (!e || !p || !r) return fail(GS_ERR_ARG, "null argument");
  if (r->capacity < 1) return fail(GS_ERR_ARG, "capacity must be >= 1");
  if ((r->flags & GS_RNG_PHILOX) && r->seeds)
    return fail(GS_ERR_ARG, "explicit seeds require the SplitMix RNG");
  CUDA_TRY(cudaSetDevice(e->device));
  // engine scratch is shared by every stream this engine runs on: order this
  // run after the previous one when the stream changes
  if (e->has_last && e->last_stream != st) CUDA_TRY(cudaStreamWaitEvent(st, e->order_ev, 0));
  int rc = upload(e, p, st);
  if (rc) return rc;
  rc = launch_body(e, p, r, O, st, timed);
  // recorded even after a failed launch, so a later run never overtakes work
  // already queued on this stream
  cudaError_t er = cudaEventRecord(e->order_ev, st);
  e->last_stream = st;
  e->has_last = true;
  if (rc) return rc;
  if (er != cudaSuccess) return fail(GS_ERR_CUDA, std::string("cudaEventRecord: ") + cudaGetErrorString(er));
  return GS_OK;
}

static int launch_body(gs_engine *e, gs_program *p, const gs_run_params *r, gs::DevOut O,
                       cudaStream_t st, bool timed) {
  int rc = GS_OK;
  const bool philox = (r->flags & GS_RNG_PHILOX) != 0;
  const bool sparse = (r->flags & GS_SPARSE) != 0;
  const bool wide_only = sparse || (r->flags & GS_WIDE_ONLY) != 0;
  if (sparse && r->capacity > 65536)
    return fail(GS_ERR_UNSUPPORTED, "GS_SPARSE: capacity above 65536 entries");
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
  P.kn = gs::narrow_kn(r->flags);
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
  sections_of(p, wide_only, P.kn, secs);
  bool any_narrow = false, any_wide = false;
  for (const Section &s : secs) (s.wide ? any_wide : any_narrow) = true;

  // launch shapes: narrow warps hold 32 shots' chi rows and record columns,
  // wide warps one shot's chi (shared memory when 2^max_dim entries fit)
  // chi of 2^13 entries or more: one block of warps per shot on two global
  // ping-pong buffers per block -- 8 warps and 2 blocks per SM at k = 13-14
  // (2 x 148 shots in flight stay L2-resident; A/B r02o: 1.2-1.7x over a
  // warp per shot at k = 13), 16 warps and 1 block per SM from k = 15 (r01bm
  // config-4 sweep: 1.4-5.5x over a warp per shot; 8 warps lose there).
  // GS_CHI_BLOCK forces the block form (16 warps, GS_BLOCK8: 8) with chi in
  // shared memory when it fits, GS_CHI_BLOCK | GS_CHI_GLOBAL on global memory
  const size_t chi = (size_t)16 << P.max_dim;
  const bool forced_block = (r->flags & GS_CHI_BLOCK) != 0;
  const bool block = !sparse && (forced_block ||
                     (!(r->flags & (GS_CHI_GLOBAL | GS_CHI_SMEM)) && P.max_dim >= GS_BLOCK_MIN_DIM));
  const u32 gwarps = !block ? 1u
                     : forced_block ? ((r->flags & GS_BLOCK8) ? 8u : (u32)GS_BLOCK_WARPS)
                     : (P.max_dim < 15 ? 8u : (u32)GS_BLOCK_WARPS);
  bool smem_chi;
  if (sparse || (r->flags & GS_CHI_GLOBAL)) smem_chi = false;
  else if (block) smem_chi = forced_block;   // decided below against the opt-in limit
  else if (r->flags & GS_CHI_SMEM) smem_chi = chi <= 64 * 1024;
  else smem_chi = chi <= 32 * 1024;
  const size_t nrec_b = (size_t)P.rec_words32 * 4 * 32, wrec_b = (size_t)P.rec_words32 * 4;
  KernelCfg KN4, KN5, KW;   // narrow launch shapes for sections needing 4 / 5 chi dims
  KN4.rec_local = KN5.rec_local = nrec_b <= 4096;
  KW.rec_local = wrec_b <= 4096;
  // the kn=5 build keeps counters and up to gs::kNarrowRecRegs record words
  // in registers (rec_local = 1 means "in registers" there): its slice is
  // the 16 KB of chi rows alone, in blocks of up to GS_NARROW_WARPS_K5 warps
  KN5.rec_local = P.rec_words32 <= gs::kNarrowRecRegs;
  for (u32 kn : {4u, 5u}) {
    bool used = false;
    for (const Section &sc : secs) used |= !sc.wide && sc.kn == kn;
    if (!used) continue;
    KernelCfg &KN = kn == 5 ? KN5 : KN4;
    const u32 wb = kn == 5 ? gs::narrow_bytes(5)
                           : (u32)((gs::kCntBytes + gs::narrow_bytes(kn) + (KN.rec_local ? nrec_b : 0) + 15) &
                                   ~(size_t)15);
    rc = occupancy(e, wb, r->warps_per_block, kn == 5 ? GS_NARROW_WARPS_K5 : 4,
                   [&](auto f) { return with_narrow_kernel(philox, kn == 5, f); }, KN);
    if (rc) return rc;
  }
  const u64 sp_stride = gs::sp_geometry(r->capacity).stride;   // sparse workspace per warp
  if (sparse) {
    // warp form layout without chi: counters and records in registers,
    // the SplitMix fire-bit ring in shared memory
    KW.rec_local = P.rec_words32 <= 32;
    KW.chi_off = 0;
    rc = occupancy(e, philox ? 0u : (u32)gs::kWinBytes, r->warps_per_block, GS_WIDE_WARPS,
                   [&](auto f) { return with_sparse_kernel(philox, f); }, KW);
    if (rc) return rc;
    const u64 max_warps = ((u64)GS_SPARSE_GB << 30) / sp_stride;
    if ((u64)KW.blocks * KW.wpb > max_warps) KW.blocks = (u32)std::max<u64>(1, max_warps / KW.wpb);
  }
  if (any_wide && !block && !sparse) {
    // warp form: counters and up to 32 record words in registers
    // (rec_local = 1 means "in registers" here), the SplitMix fire-bit
    // ring in shared memory, then chi
    KW.rec_local = P.rec_words32 <= 32;
    size_t base = philox ? 0 : gs::kWinBytes;
    KW.chi_off = (u32)base;
    const u32 wb = (u32)(base + (smem_chi ? chi : 0));
    rc = occupancy(e, wb, r->warps_per_block, GS_WIDE_WARPS,
                   [&](auto f) { return with_wide_kernel(smem_chi, philox, 1u, f); }, KW);
    if (rc) return rc;
    if (!smem_chi) {   // bound the global chi scratch
      const u64 max_warps = ((u64)8 << 30) / chi;
      if ((u64)KW.blocks * KW.wpb > max_warps) KW.blocks = (u32)std::max<u64>(1, max_warps / KW.wpb);
    }
  }
  if (any_wide && block) {
    // [per-warp slices][group scratch: 2 x 32 u64][chi]
    const size_t base = gs::kCntBytes + gs::kWinBytes + (KW.rec_local ? ((wrec_b + 15) & ~(size_t)15) : 0);
    const size_t head = (size_t)gwarps * base + 64 * sizeof(u64);
    if (smem_chi && head + chi > e->smem_optin) smem_chi = false;
    KW.wpb = gwarps;
    KW.warp_bytes = (u32)base;
    KW.chi_off = (u32)head;
    KW.smem = head + (smem_chi ? chi : 0);
    int per = 0;
    CUDA_TRY(with_wide_kernel(smem_chi, philox, gwarps, [&](auto kern) {
      cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)KW.smem);
      return err != cudaSuccess ? err
                                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, gwarps * 32, KW.smem);
    }));
    if (per < 1) return fail(GS_ERR_UNSUPPORTED, "block-per-shot state exceeds the SM");
    KW.blocks = (u32)(e->num_sms * per);
    if (!smem_chi) {
      const u64 max_blocks = ((u64)8 << 30) / (3 * chi);   // two 1.5-chi buffers per block
      if ((u64)KW.blocks > max_blocks) KW.blocks = (u32)std::max<u64>(1, max_blocks);
    }
  }
  if (r->blocks) { KN4.blocks = KN5.blocks = r->blocks; KW.blocks = r->blocks; }
  const u64 nwarps = std::max({(u64)KN4.blocks * KN4.wpb, (u64)KN5.blocks * KN5.wpb,
                               (u64)KW.blocks * KW.wpb});
  if (sparse) {
    rc = ensure_buf(&e->d_chi, &e->chi_bytes, (size_t)KW.blocks * KW.wpb * sp_stride);
    if (rc) return rc;
  } else if (!smem_chi && any_wide) {
    rc = ensure_buf(&e->d_chi, &e->chi_bytes, (size_t)KW.blocks * (block ? 3 : KW.wpb) * chi);
    if (rc) return rc;
  }
  if (!KN4.rec_local || !KN5.rec_local || !KW.rec_local) {
    rc = ensure_buf(&e->d_rec, &e->rec_bytes, (size_t)nwarps * nrec_b);
    if (rc) return rc;
  }
  // queues between sections: fixed slots, chunks of at most `chunk` shots
  const u64 slot_b = 8ull * (gs::Q_HDR + gs::rec_u64(P.rec_words32) + 2 * (1u << P.kn));
  u64 chunk = r->shot_count ? r->shot_count : 1;
#ifndef GS_QUEUE_GB
#define GS_QUEUE_GB 8   // per section queue: one chunk for a 2^24-shot step (A/B +0.4 % over 2 GB)
#endif
  if (!e->queue_budget) {   // auto: min(8 GiB, 1/16 of the free device memory)
    size_t fr = 0, tot = 0;
    CUDA_TRY(cudaMemGetInfo(&fr, &tot));
    e->queue_budget = std::max<u64>(64ull << 20, std::min<u64>((u64)GS_QUEUE_GB << 30, fr / 16));
  }
  const u64 qbudget = e->queue_budget;   // bytes per queue
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
  const bool stats = (r->flags & GS_SECTION_STATS) != 0;
  if (stats) {
    if (secs.size() > e->secstats_cap) {   // (re)size: accumulations restart
      cudaFree(e->d_secstats);
      e->d_secstats = nullptr;
      e->secstats_cap = 0;
      const size_t cap = std::max<size_t>(64, secs.size());
      CUDA_TRY(cudaMalloc(&e->d_secstats, (cap * 4 + 1) * 8));
      CUDA_TRY(cudaMemsetAsync(e->d_secstats, 0, (cap * 4 + 1) * 8, st));
      e->secstats_cap = cap;
    }
    e->sec_meta.assign(2 * secs.size(), 0);
    for (size_t i = 0; i < secs.size(); ++i) {
      e->sec_meta[2 * i] = secs[i].wide;
      e->sec_meta[2 * i + 1] = secs[i].pc0;
    }
  }
  u64 *d_mbprev = stats ? e->d_secstats + 4 * e->secstats_cap : nullptr;
  auto grab_event = [&](cudaEvent_t *ev) -> int {
    if (!e->spare_ev.empty()) { *ev = e->spare_ev.back(); e->spare_ev.pop_back(); return GS_OK; }
    CUDA_TRY(cudaEventCreate(ev));
    return GS_OK;
  };
  if (r->shot_count) {
    if (timed) CUDA_TRY(cudaEventRecord(e->ev0, st));
    for (u64 first = 0; first < r->shot_count; first += chunk) {
      const u64 count = std::min(chunk, r->shot_count - first);
      CUDA_TRY(cudaMemsetAsync(e->d_work, 0, sizeof(unsigned long long) * (secs.size() + 2), st));
      if (stats) {
        gs::mb_snapshot_kernel<<<1, 1, 0, st>>>(O.counters + GS_C_MODEL_BYTES, d_mbprev);
        CUDA_TRY(cudaGetLastError());
        e->launches += 1;
      }
      for (size_t i = 0; i < secs.size(); ++i) {
        gs::DevSec S;
        S.pc0 = secs[i].pc0;
        S.k0 = secs[i].k0;
        S.nm0 = secs[i].nm0;
        S.pc_end = i + 1 < secs.size() ? secs[i + 1].pc0 : 0xFFFFFFFFu;   // the next section's first op
        S.first = first;
        S.count = count;
        S.q_in = i ? e->d_queue[(i - 1) & 1] : nullptr;
        S.n_in = i ? d_qn + ((i - 1) & 1) : nullptr;
        S.q_out = i + 1 < secs.size() ? e->d_queue[i & 1] : nullptr;
        S.n_out = d_qn + (i & 1);
        S.work = e->d_work + i;
        S.pn0 = secs[i].pn0;
        S.kn = secs[i].kn;
        if (i >= 1 && i + 1 < secs.size())   // the queue written here was read by section i-1
          CUDA_TRY(cudaMemsetAsync(d_qn + (i & 1), 0, sizeof(u32), st));
        Engine_TimedLaunch tl{(u32)i, nullptr, nullptr};
        if (stats) {
          if (grab_event(&tl.a) || grab_event(&tl.b)) return GS_ERR_CUDA;
          CUDA_TRY(cudaEventRecord(tl.a, st));
        }
        if (secs[i].wide) {
          gs::DevOut Ow = O;
          Ow.warp_bytes = KW.warp_bytes;
          Ow.rec_local = KW.rec_local;
          Ow.chi_off = KW.chi_off;
          auto go = [&](auto kern) {
            kern<<<KW.blocks, KW.wpb * 32, KW.smem, st>>>(P, R, Ow, S);
            return cudaGetLastError();
          };
          if (sparse) CUDA_TRY(with_sparse_kernel(philox, go));
          else CUDA_TRY(with_wide_kernel(smem_chi, philox, gwarps, go));
        } else {
          const KernelCfg &KN = secs[i].kn == 5 ? KN5 : KN4;
          gs::DevOut On = O;
          On.warp_bytes = KN.warp_bytes;
          On.rec_local = KN.rec_local;
          On.chi_off = 0;
          CUDA_TRY(with_narrow_kernel(philox, secs[i].kn == 5, [&](auto kern) {
            kern<<<KN.blocks, KN.wpb * 32, KN.smem, st>>>(P, R, On, S);
            return cudaGetLastError();
          }));
        }
        e->launches += 1;
        if (stats) {
          CUDA_TRY(cudaEventRecord(tl.b, st));
          e->timed.push_back({tl.sec, tl.a, tl.b});
          const u64 nq = secs.size() > 1 ? chunk : 0;
          const u32 grid = (u32)std::max<u64>(1, std::min<u64>((u64)e->num_sms * 4, (nq + 255) / 256));
          gs::section_stats_kernel<<<grid, 256, 0, st>>>(
              S.q_in, S.n_in, count, S.q_out, S.n_out, (u32)(slot_b / 8),
              O.counters + GS_C_MODEL_BYTES, d_mbprev, e->d_secstats + 4 * i);
          CUDA_TRY(cudaGetLastError());
          e->launches += 1;
        }
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

int gs_engine_section_stats(gs_engine *e, uint64_t *out, uint32_t cap, uint32_t *n, int reset) {
  if (!e || !n || (cap && !out)) return fail(GS_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(e->device));
  CUDA_TRY(cudaDeviceSynchronize());   // the timed runs may sit on any stream
  const size_t nsec = e->sec_meta.size() / 2;
  std::vector<u64> dev(4 * std::max<size_t>(nsec, 1), 0);
  if (nsec && e->d_secstats)
    CUDA_TRY(cudaMemcpy(dev.data(), e->d_secstats, nsec * 4 * 8, cudaMemcpyDeviceToHost));
  std::vector<double> ns(nsec, 0.0);
  std::vector<u64> nl(nsec, 0);
  for (auto &t : e->timed) {
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, t.a, t.b));
    if (t.sec < nsec) { ns[t.sec] += 1e6 * (double)ms; nl[t.sec] += 1; }
  }
  *n = (uint32_t)nsec;
  for (size_t i = 0; i < nsec && i < cap; ++i) {
    uint64_t *o = out + i * GS_SEC_FIELDS;
    o[GS_SEC_SHOTS_IN] = dev[4 * i];
    o[GS_SEC_SHOTS_OUT] = dev[4 * i + 1];
    o[GS_SEC_MODEL_BYTES] = dev[4 * i + 2];
    o[GS_SEC_DEVICE_NS] = (uint64_t)llround(ns[i]);
    o[GS_SEC_LAUNCHES] = nl[i];
    o[GS_SEC_WIDE] = e->sec_meta[2 * i];
    o[GS_SEC_PC0] = e->sec_meta[2 * i + 1];
  }
  if (reset) {
    if (e->d_secstats) {
      // legacy-stream memset: finish it before a launch on a non-blocking stream
      CUDA_TRY(cudaMemset(e->d_secstats, 0, (e->secstats_cap * 4 + 1) * 8));
      CUDA_TRY(cudaDeviceSynchronize());
    }
    for (auto &t : e->timed) { e->spare_ev.push_back(t.a); e->spare_ev.push_back(t.b); }
    e->timed.clear();
  }
  return GS_OK;
}

int gs_engine_set_queue_budget(gs_engine *e, uint64_t bytes_per_queue) {
  if (!e) return fail(GS_ERR_ARG, "null argument");
  e->queue_budget = bytes_per_queue;
  return GS_OK;
}

int gs_engine_trim(gs_engine *e) {
  if (!e) return fail(GS_ERR_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(e->device));
  CUDA_TRY(cudaDeviceSynchronize());
  cudaFree(e->d_queue[0]); e->d_queue[0] = nullptr; e->queue_bytes[0] = 0;
  cudaFree(e->d_queue[1]); e->d_queue[1] = nullptr; e->queue_bytes[1] = 0;
  cudaFree(e->d_chi); e->d_chi = nullptr; e->chi_bytes = 0;
  cudaFree(e->d_rec); e->d_rec = nullptr; e->rec_bytes = 0;
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
