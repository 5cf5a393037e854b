/*
 * gstab_sm100.h -- C ABI of the B200 (sm_100a) generalized-stabilizer shot
 * sampler (libgstab_sm100a.so).
 *
 * Drop-in boundary for the reference's shot engine
 * (/root/reference/pkg/src/gstab/sampler.py):
 *
 *   gs_run_counters  replaces run_batch -> _run_chunk -> run_shot
 *                    (ref sampler.py:348-382, 302-331, 169-255): counters of
 *                    SamplerConfig.shots shots, overflow reruns with capacity
 *                    doubling folded into one pass (ref sampler.py:306-316).
 *   gs_run_records   replaces run_shot(..., keep_record=True) per shot
 *                    (ref sampler.py:169-255): status, discarded detector /
 *                    overflow instruction, record bits, observables.
 *   gs_dump_shots    replaces the observer snapshot of GenStabState after an
 *                    instruction (ref oracle.py:246-262, state.py:52-80).
 *   gs_anticommute_mask / gs_conj_gate_rows / gs_mul_rows / gs_parity_pm
 *                    batched device versions of the reference kernel plugin
 *                    API (ref _kernels.pyx:28-139, _kernels_py.py:20-110).
 *
 * The program words come from paper_2512_23037_b200/compiler.py (static
 * frame).  Conventions: return 0 on success, <0 on error
 * with a thread-local message from gs_last_error(); OVERFLOW / DISCARDED /
 * CORRUPT are per-shot statuses, not errors.  Host arrays are caller-owned
 * and copied; device buffers and handles are library-owned.  One engine per
 * device and host thread; calls are host-synchronous except *_async.
 */
#ifndef GSTAB_SM100_H
#define GSTAB_SM100_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_ABI_VERSION 3

/* error codes */
#define GS_OK 0
#define GS_ERR_ARG (-1)
#define GS_ERR_CUDA (-2)
#define GS_ERR_NOMEM (-3)
#define GS_ERR_UNSUPPORTED (-4)

/* run flags */
#define GS_POSTSELECT 1u   /* discard on the first firing detector      */
#define GS_RNG_PHILOX 2u   /* Philox4x32-10 streams (else SHA-1+SplitMix) */
#define GS_CHI_GLOBAL 4u   /* force chi buffers into global memory (test) */
#define GS_CHI_SMEM 16u    /* force chi buffers into shared memory (test) */
#define GS_WIDE_ONLY 32u   /* run every op warp-per-shot (A/B, test)     */
#define GS_CHI_BLOCK 64u   /* wide sections: one block of 16 warps per
                              shot, chi in shared memory when it fits (the
                              default from chi dimension 13: 8 warps at
                              13-14, 16 from 15, on global memory)       */
#define GS_SECTION_STATS 128u /* per-section device time (CUDA events on
                              the launch stream) and model bytes / shots
                              (a small reduction launch after each
                              section); read with gs_engine_section_stats */
#define GS_NARROW_K5 256u  /* lane-per-shot sections up to chi dimension 5
                              (default 4; only sections holding a k = 5 op
                              use the 2^5-row layout): a pure performance
                              choice, the results are identical either way */
#define GS_BLOCK8 512u     /* with GS_CHI_BLOCK: 8 warps per shot (test)   */
#define GS_SPARSE 1024u    /* sparse chi: the whole program warp per shot
                              on a list of the nonzero entries (program
                              max_dim <= 30, capacity <= 65536) -- for
                              supports far below 2^k, e.g. T gates that
                              cancel; results as the dense forms'        */

/* per-shot status codes (gs_run_records) */
#define GS_ST_PRESERVED 1
#define GS_ST_DISCARDED 2
#define GS_ST_OVERFLOW 3
#define GS_ST_CORRUPT 4
#define GS_ST_UNSUPPORTED 5

/* counter vector layout (int64) */
#define GS_C_TOTAL 0
#define GS_C_PRESERVED 1
#define GS_C_DISCARDED 2
#define GS_C_OVERFLOW 3
#define GS_C_CORRUPT 4
#define GS_C_UNSUPPORTED 5
#define GS_C_ERROR_SHOTS 6
#define GS_C_MODEL_BYTES 7
#define GS_C_PER_OBS 8       /* + observable id, num_obs entries */

typedef struct gs_program gs_program;
typedef struct gs_engine gs_engine;

typedef struct {
  uint32_t num_qubits;       /* 1..64                                    */
  uint32_t num_measurements; /* record bits per shot                     */
  uint32_t num_detectors;
  uint32_t num_obs;          /* distinct observable keys (<= 64)         */
  uint32_t max_dim;          /* static chi dimension k_max (<= 30)       */
  uint32_t num_locations;    /* noise locations                          */
  uint32_t num_noise;        /* noise instructions (tables[noise_off..]) */
  uint32_t num_words;        /* ceil(num_locations / 32)                 */
  uint64_t noise_off;        /* tables offset: 4 words per noise instr.  */
  uint64_t wordpc_off;       /* tables offset: insertion pc per word     */
  /* Philox mode: fired noise locations come from geometric skipping over a
     Bernoulli(p_max) candidate process (thinned to each location's p) */
  uint64_t geo_off;          /* tables offset: gap table T[0..geo_len)   */
  uint32_t geo_len;          /* num_locations of the full program + 1    */
  uint32_t noise_uniform;    /* 1: every location has p == p_max        */
  uint64_t acc_off;          /* tables offset: per-location thinning
                                thresholds (used when !noise_uniform)    */
} gs_program_info;

typedef struct {
  uint64_t master_seed;
  uint64_t shot_begin;       /* global index of the first shot           */
  uint64_t shot_count;
  uint64_t capacity;         /* entry_capacity * 2^doublings (effective) */
  uint32_t flags;            /* GS_POSTSELECT | GS_RNG_PHILOX | ...      */
  uint32_t warps_per_block;  /* 0 = auto                                 */
  uint32_t blocks;           /* 0 = auto (persistent grid)               */
  uint32_t chunk_shots;      /* shots per section pass, 0 = auto (test)  */
  const uint64_t *seeds;     /* optional host per-shot seeds (SplitMix)  */
} gs_run_params;

/* program (host copy; uploaded to the engine's device on first use) */
int gs_program_create(const gs_program_info *info, const uint64_t *ops,
                      size_t n_ops, const uint64_t *tables, size_t n_tables,
                      const uint64_t *locs, size_t n_locs, gs_program **out);
int gs_program_destroy(gs_program *prog);
/* number of narrow/wide sections (= sampling launches per chunk of shots)
   the program runs as under `flags` (GS_WIDE_ONLY); <0 on error */
int gs_program_sections(const gs_program *prog, uint32_t flags);

int gs_engine_create(int device, gs_engine **out);
int gs_engine_destroy(gs_engine *eng);

/* counters: host vector of GS_C_PER_OBS + num_obs int64 (overwritten) */
int gs_run_counters(gs_engine *eng, gs_program *prog, const gs_run_params *p,
                    int64_t *counters);
/* counters plus up to witness_cap global shot indices of preserved shots
   whose observables flipped (logical-error witnesses, paper §V-B); the
   total number found is returned in *witness_count (may exceed the cap).
   Order is nondeterministic; callers sort. */
int gs_run_counters_witness(gs_engine *eng, gs_program *prog,
                            const gs_run_params *p, int64_t *counters,
                            uint64_t *witness, uint32_t witness_cap,
                            uint32_t *witness_count);
/* async variant: accumulates (+=) into a DEVICE int64 vector on `stream`
   (cudaStream_t); lets NCCL reduce the counters in place */
int gs_run_counters_async(gs_engine *eng, gs_program *prog,
                          const gs_run_params *p, int64_t *counters_dev,
                          void *stream);

/* records: status[shots], aux[shots] (discarded detector / overflow
   instruction / -1), record_bits[shots][ceil(num_measurements/64)],
   obs_bits[shots] (bit i = observable id i) */
int gs_run_records(gs_engine *eng, gs_program *prog, const gs_run_params *p,
                   uint8_t *status, int32_t *aux, uint64_t *record_bits,
                   uint64_t *obs_bits);

/* dumps: as records plus final sign vector sig[shots][2] (destab, stab),
   coset offset c[shots], amplitudes amps[shots][2^max_dim][2] (re, im) and
   the dimension dim[shots] in force when the shot stopped */
int gs_dump_shots(gs_engine *eng, gs_program *prog, const gs_run_params *p,
                  uint8_t *status, int32_t *aux, uint64_t *record_bits,
                  uint64_t *obs_bits, uint64_t *sig, uint64_t *c,
                  double *amps, uint32_t *dim);

/* kernel plugin API, batched over `batch` independent row sets (ref
   _kernels.pyx).  Host arrays; rows are `rows` per batch entry.
   anticommute: out_mask[batch][2] (128-bit row mask, lo word first). */
int gs_anticommute_mask(gs_engine *eng, const uint64_t *xs, const uint64_t *zs,
                        uint32_t rows, uint32_t batch, const uint64_t *qx,
                        const uint64_t *qz, uint64_t *out_mask);
int gs_conj_gate_rows(gs_engine *eng, uint64_t *xs, uint64_t *zs, uint8_t *ph,
                      uint32_t rows, uint32_t batch, const uint32_t *code,
                      const uint64_t *m1, const uint64_t *m2);
int gs_mul_rows(gs_engine *eng, uint64_t *xs, uint64_t *zs, uint8_t *ph,
                uint32_t rows, uint32_t batch, const uint8_t *sel,
                const uint64_t *px, const uint64_t *pz, const uint32_t *pe);
int gs_parity_pm(gs_engine *eng, const uint64_t *idx, size_t count,
                 uint64_t mask, double *out);

/* per-section statistics accumulated by GS_SECTION_STATS runs since the
   last read (reset = 1 clears them): out[i * GS_SEC_FIELDS + f] for section
   i < *n (at most `cap` sections written), fields below.  Synchronizes with
   the streams the timed launches ran on. */
#define GS_SEC_SHOTS_IN 0     /* shots that entered the section            */
#define GS_SEC_SHOTS_OUT 1    /* shots it handed to the next section       */
#define GS_SEC_MODEL_BYTES 2  /* SURVEY §8(d) state-touch bytes it executed */
#define GS_SEC_DEVICE_NS 3    /* summed launch durations (CUDA events), ns */
#define GS_SEC_LAUNCHES 4     /* launches of the section                   */
#define GS_SEC_WIDE 5         /* 1: wide_kernel (warp/block per shot)      */
#define GS_SEC_PC0 6          /* first op word of the section              */
#define GS_SEC_FIELDS 7
int gs_engine_section_stats(gs_engine *eng, uint64_t *out, uint32_t cap,
                            uint32_t *n, int reset);

/* inter-section queue budget in bytes per queue (two queues); 0 = auto:
   min(8 GiB, 1/16 of the device memory free when first sized).  A run
   larger than the budget is split into chunks (results are identical). */
int gs_engine_set_queue_budget(gs_engine *eng, uint64_t bytes_per_queue);
/* free the engine's scratch (queues, global chi/record buffers) after the
   pending work; the next run re-allocates what it needs */
int gs_engine_trim(gs_engine *eng);

/* Streams: synchronous calls run on the engine's own stream; *_async calls
   on the caller's.  Launches are ordered across streams by the engine (an
   event recorded after each run is waited on by the next run's stream), so
   mixing the two is safe; concurrent calls from several host threads on
   one engine are not supported (the Python Engine serialises its calls
   with a lock, so its process-wide engines are thread-safe). */

/* diagnostics */
const char *gs_last_error(void);
int gs_abi_version(void);
/* number of gs kernels this engine launched since creation */
uint64_t gs_engine_launches(gs_engine *eng);
/* device time (ms) of the last gs_run_* sampling kernel, CUDA events */
double gs_engine_last_kernel_ms(gs_engine *eng);

#ifdef __cplusplus
}
#endif
#endif /* GSTAB_SM100_H */
