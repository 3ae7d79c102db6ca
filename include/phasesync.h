/*
 * phasesync.h -- C ABI of libphasesync_cuda.so, the sm_100a PLV / iPLV / ciPLV
 * hot path (arXiv 1710.08037 reformulation: Hilbert -> unit phasors ->
 * Hermitian Gram Z Z^H -> fused PLV-family epilogue).
 *
 * The reference (/root/reference) defines this boundary only as SPEC text: the
 * `bindings` module, SPEC.md:519-564 (ArrayView :524-527, py_analytic_signal
 * :530-537, py_plv / py_iplv / py_ciplv :538-544, errors "mapped 1:1" :533,
 * GIL released :554, no state :548).  Each entry point below names the
 * reference operation it replaces.  No torch types cross this ABI: plain
 * pointers, sizes and strides; device pointers unless stated otherwise.
 *
 * Errors: every function returns a ps_status; nothing throws or aborts across
 * the ABI.  PS_E_SHAPE -> ShapeError (errors.py:32), PS_E_ALL_MASKED ->
 * AllSamplesMaskedError (errors.py:12), PS_E_EMPTY_WINDOW ->
 * EmptyEffectiveWindowError (errors.py:20); device/library failures map to
 * RuntimeError subclasses.  ps_last_error() returns a thread-local message.
 */
#ifndef PHASESYNC_H_
#define PHASESYNC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PS_ABI_VERSION 8

typedef enum ps_status {
  PS_OK = 0,
  PS_E_SHAPE = 1,         /* ShapeError                 errors.py:32 */
  PS_E_ALL_MASKED = 2,    /* AllSamplesMaskedError      errors.py:12 */
  PS_E_EMPTY_WINDOW = 3,  /* EmptyEffectiveWindowError  errors.py:20 */
  PS_E_INVALID = 4,       /* ValueError (bad argument combination)    */
  PS_E_UNSUPPORTED = 5,   /* UnsupportedError (valid per SPEC, not built) */
  PS_E_CUDA = 6,          /* CudaError                                */
  PS_E_CUFFT = 7,         /* CudaError (cuFFT)                        */
  PS_E_OOM = 8,           /* MemoryError                              */
  PS_E_INTERNAL = 9,      /* RuntimeError                             */
  PS_E_SIGNAL_TOO_SHORT = 10, /* SignalTooShortError (n_samples <= order + 1) */
  PS_E_WINDOW_TOO_LONG = 11,  /* WindowTooLongError (window_len > n_samples) */
  PS_E_EMPTY_BAND = 12        /* EmptyBandError (no bin in the band)        */
} ps_status;

typedef enum ps_dtype { PS_F32 = 0, PS_F64 = 1, PS_C64 = 2, PS_C128 = 3 } ps_dtype;

/* What the input array holds. */
typedef enum ps_input_kind {
  PS_INPUT_REAL = 0,      /* RealEpochs: Hilbert + normalise + Gram        */
  PS_INPUT_ANALYTIC = 1,  /* AnalyticEpochs: normalise + Gram              */
  PS_INPUT_PHASOR = 2     /* PhasorEpochs: Gram (zeros are masked samples) */
} ps_input_kind;

typedef enum ps_precision {
  PS_PREC_SPLIT_F16X3 = 0, /* tcgen05 kind::f16, hi/lo split, 3 products, fp32 out */
  PS_PREC_FP64 = 1         /* DMMA f64 operands and accumulation, fp64 out       */
} ps_precision;

typedef enum ps_trial_reduce {
  PS_TRIALS_MEAN = 0,  /* mean over trials of per-trial metrics (default) */
  PS_TRIALS_NONE = 1,  /* one matrix per trial (PAPER.md:281-287 plv(:,:,t))        */
  PS_TRIALS_POOL = 2,  /* one Gram over all R*T observations                         */
  PS_TRIALS_SUM = 3    /* sum over trials of per-trial metrics (ABI v8): the partial sums
                          of a (band, trial)-sharded call, combined across ranks by
                          ps_reduce_partials, which divides by the global trial count */
} ps_trial_reduce;

enum {
  PS_METRIC_PLV = 1,    /* (1/T)|z_i z_j^H|            Eq 7, */
  PS_METRIC_IPLV = 2,   /* (1/T)|Im z_i z_j^H|         Eq 13 */
  PS_METRIC_CIPLV = 4,  /* |Im|/sqrt(1-Re^2)           Eq 14 */
  PS_METRIC_CRE = 8,    /* signed Re (1/T) z_i z_j^H (coherency real part)  */
  PS_METRIC_CIM = 16    /* signed Im (1/T) z_i z_j^H (antisymmetric)        */
};

typedef struct ps_ctx ps_ctx;

/* Band-pass front end for real input (decisions :121-122):
 * reflection padding of pad_samples per side, zero-phase two-pass FIR (forward,
 * reverse, forward, reverse; zero initial state), analytic signal of the padded
 * record, then trim ("prior to the removal of the padding").
 * taps: HOST pointer to n_taps = order + 1 coefficients (design_bandpass_fir).
 * Requires n_samples > n_taps (SignalTooShort) and pad_samples < n_samples. */
typedef struct ps_fir {
  const double* taps;
  int64_t n_taps;
  int64_t pad_samples;
} ps_fir;

/* Input/output description for one call.  Shapes follow the reference
 * ArrayView [n_signals x n_samples x n_trials] plus an optional
 * leading band axis.  Strides are in ELEMENTS (complex elements for c64/c128)
 * and may describe any layout; samples need not be contiguous (a
 * non-unit sample stride costs one packing copy, reported in
 * ps_plv_result.input_copied -- SPEC.md:526,551 copy-on-mismatch). */
typedef struct ps_plv_args {
  const void* input;           /* device pointer (host pointer for *_host entry) */
  int32_t dtype;               /* ps_dtype */
  int32_t input_kind;          /* ps_input_kind */
  int64_t n_bands, n_signals, n_samples, n_trials;
  int64_t stride_band, stride_signal, stride_sample, stride_trial;
  double amp_floor;            /* SPEC.md:123 default 1e-6 */
  uint32_t metrics;            /* PS_METRIC_* bitmask */
  int32_t precision;           /* ps_precision */
  int32_t trial_reduce;        /* ps_trial_reduce */
  /* Outputs, one per requested metric: dense row-major [n_bands][n_signals]
   * [n_signals] (MEAN/POOL) or [n_bands][n_trials][n_signals][n_signals]
   * (NONE); float for SPLIT, double for FP64.  Symmetric (CIM: antisymmetric)
   * with the SPEC diagonal rules applied. */
  void* out_plv;
  void* out_iplv;
  void* out_ciplv;
  void* out_cre;
  void* out_cim;
  /* Output-tile sharding across devices: this call computes
   * only tiles t with t % shard_count == shard_index; other entries of DEVICE
   * outputs are left untouched.  The host-output entry points stage the
   * outputs in device memory and copy whole matrices back, so there the
   * entries owned by other shards are written as 0 (the shards' host
   * matrices sum to the full result); with PS_LAYOUT_UPPER on the streamed
   * host path a shard owns whole row bands and writes only those rows.
   * shard_count = 1 computes everything. */
  int32_t shard_index;
  int32_t shard_count;
  void* stream;                /* cudaStream_t (NULL = legacy default stream) */
  /* PS_MODE_OVER_SAMPLES (Eq 7, default) or PS_MODE_OVER_TRIALS (Eq 8,
   * time-resolved: one matrix per sample from the Gram over trials, SPEC.md:
   * 153-157,173,186-189).  Over trials, outputs are [n_bands][n_samples][N][N]
   * and trial_reduce is ignored. */
  int32_t mode;
  /* PS_LAYOUT_FULL (default): both triangles written (symmetric; CIM
   * antisymmetric).  PS_LAYOUT_UPPER: only entries (i, j) with i <= j of each
   * [N][N] slot are written -- the output BASELINE configs[4] asks for ("the
   * 20,000 x 20,000 upper triangle for each metric"); the strictly lower
   * triangle is left as the caller allocated it (device outputs); the host
   * entry point does not transfer it except inside the diagonal blocks of its
   * copy-out, which read 0 there.  Halves output writes and D2H bytes. */
  int32_t out_layout;
  /* Optional band-pass front end (real input only; NULL = input is already
   * band-limited, the configs' case). */
  const ps_fir* fir;
} ps_plv_args;

enum { PS_MODE_OVER_SAMPLES = 0, PS_MODE_OVER_TRIALS = 1 };
enum { PS_LAYOUT_FULL = 0, PS_LAYOUT_UPPER = 1 };

typedef struct ps_plv_result {
  int64_t n_observations;      /* T used for normalisation (R*T for POOL) */
  int64_t n_masked_samples;    /* total samples masked by the amplitude guard */
  int64_t n_refined_pairs;     /* ill-conditioned ciPLV pairs recomputed in FP64 */
  int32_t input_copied;        /* 1 if the input layout forced a packing copy */
  int32_t n_kernel_launches;   /* kernels of this library launched by the call */
  float ms_hilbert;            /* reserved (0): the Hilbert stage is interleaved with, and
                                  counted in, ms_normalize */
                               /* device time per stage (ps_ctx_set_timing): */
  float ms_normalize;
  float ms_gram;
  float ms_finish;
  /* Host entry point only: bytes actually moved over the host link by the
   * call (the pipelined path transfers one triangle's column blocks and
   * mirrors the rest on the host). */
  int64_t h2d_bytes;
  int64_t d2h_bytes;
  /* Gram arithmetic of the call (ABI v7): 0 = split fp16 x 3, four real
   * products (12 UMMAs per K step); 1 = split fp16 x 3, three-product Gauss
   * form (9 UMMAs); 2 = FP64 DMMA. */
  int32_t gram_variant;
  /* Split path (ABI v8): off-diagonal pairs whose |Re| rounds to 1 in fp32
   * while |Im| > 4e-6 -- the ciPLV denominator 1 - Re^2 is below the split
   * arithmetic's resolution there, so ciPLV (reported as 0) is indeterminate
   * and the caller should use PS_PREC_FP64 for them (SPEC.md:259 singularity
   * rule applies to |Re| >= 1 - 1e-12 only).  0 in FP64 mode. */
  int32_t n_indeterminate_ciplv;
} ps_plv_result;

/* ABI version check (PS_ABI_VERSION). */
int ps_abi_version(void);

/* Thread-local description of the last error on this thread. */
const char* ps_last_error(void);

/* Context: owns cuFFT plans, workspace and per-device state for `device`.
 * Results are never cached.  One context per thread, or
 * external locking. */
ps_status ps_ctx_create(int device, ps_ctx** out);
ps_status ps_ctx_destroy(ps_ctx* ctx);
/* Enable per-stage CUDA-event timing (fills ms_* in ps_plv_result). */
ps_status ps_ctx_set_timing(ps_ctx* ctx, int enable);

/* Replaces bindings.py_plv / py_iplv / py_ciplv and
 * connectivity.plv_matrix / iplv / ciplv: all requested
 * PLV-family metrics from ONE Gram per trial.  Device pointers; synchronises
 * `stream` before returning so the status reflects device-side checks
 * (AllSamplesMasked, EmptyEffectiveWindow).  result may be NULL. */
ps_status ps_plv_family(ps_ctx* ctx, const ps_plv_args* args, ps_plv_result* result);

/* Device path with a staged input (multi-GPU input distribution):
 * the signal rows [stage_cols[s], stage_cols[s+1]) of every (band, trial)
 * unit become valid on the device once ready_events[s] (a cudaEvent_t, NULL =
 * already valid) completes -- e.g. after an NCCL broadcast of that chunk from
 * the rank holding the input.  Normalisation of a chunk and the Gram tiles
 * whose columns fall in stage s start as soon as their rows have arrived, so
 * the transfer of later chunks overlaps compute ("growing square").
 * stage_cols: n_stages + 1 increasing signal indices, 0 ... n_signals, interior
 * ones multiples of 256.  Trial means use one trial group per band. */
ps_status ps_plv_family_staged(ps_ctx* ctx, const ps_plv_args* args, ps_plv_result* result, int32_t n_stages,
                               const int64_t* stage_cols, void* const* ready_events);

/* Same contract with HOST input/output pointers (pinned memory recommended):
 * host->device copy, compute, device->host copy, all inside the call.  This is
 * the entry point a host binding (ctypes / cgo / JNI) uses for plain arrays. */
ps_status ps_plv_family_host(ps_ctx* ctx, const ps_plv_args* args, ps_plv_result* result);

/* DEVICE input (valid in args->stream's order, e.g. assembled on every rank by
 * an NCCL all-gather of per-rank host slices), HOST outputs: compute and
 * device->host copy inside the call, the copy-out streamed while the Gram
 * runs.  With PS_LAYOUT_UPPER and shard_count > 1 each shard owns whole row
 * bands and writes only those rows of the host matrices (ABI v6). */
ps_status ps_plv_family_to_host(ps_ctx* ctx, const ps_plv_args* args, ps_plv_result* result);

/* Replaces signalprep.analytic_signal / bindings.py_analytic_signal
 * (SPEC.md:76-84, :530-537): out = x + i H{x}, Re(out) == x bit-exactly.
 * Input real (f32 or f64) with the strides of args; output interleaved
 * complex (c64 for f32, c128 for f64), dense [n_bands][n_trials][n_signals]
 * [n_samples].  Uses only: input, dtype, n_*, stride_*, stream. */
ps_status ps_analytic_signal(ps_ctx* ctx, const ps_plv_args* args, void* out);

/* Replaces signalprep.filter_two_pass: zero-phase two-pass
 * FIR of real input with reflection padding, trimmed back to the input shape.
 * Uses args->fir (required) and the input fields of args; output real of the
 * input precision, dense [n_bands][n_trials][n_signals][n_samples]. */
ps_status ps_filter_two_pass(ps_ctx* ctx, const ps_plv_args* args, void* out);

/* Welch coherence family over all pairs (Eq 12; SURVEY 8(f)
 * #3).  Segments of window_len samples advancing by window_len - overlap within
 * each trial (segments of all trials pooled), symmetric Hamming
 * taper, spectrum X_n,s(k) per bin.  For every bin k in the band
 * (low <= 2 pi k / window_len <= high) the normalised
 * cross-spectrum C_ij(k) = sum_s X_i X_j^* / sqrt(sum_s |X_i|^2 sum_s |X_j|^2)
 * is one Gram over segments, and the outputs of args are reinterpreted:
 *   out_plv  -> COH  = |C|          (coherence_welch, magnitude)
 *   out_iplv -> ICOH = |Im C|       (imaginary_coherency)
 *   out_cre / out_cim -> Re C, Im C (signed coherency);  out_ciplv -> |Im C| / sqrt(1 - Re C^2)
 * aggregated over the band's bins by `reduce` (band_coherence):
 * MEAN / MAX -> [n_bands][N][N], NONE -> [n_bands][n_bins][N][N] (one matrix
 * per bin, ascending k).  Pairs with zero power at a bin get 0 there; the COH
 * diagonal is 1.  Real input only; n_trials = trials, precision as usual. */
typedef enum ps_band_reduce { PS_BAND_MEAN = 0, PS_BAND_MAX = 1, PS_BAND_NONE = 2 } ps_band_reduce;
typedef struct ps_welch {
  int64_t window_len;
  int64_t overlap;
  double band_low;   /* radians per sample, 0 <= low <= high <= pi */
  double band_high;
  int32_t reduce;    /* ps_band_reduce */
  int32_t reserved0;
} ps_welch;
ps_status ps_coherence(ps_ctx* ctx, const ps_plv_args* args, const ps_welch* welch, ps_plv_result* result);
/* Number of bins the band selects (host helper): k0 (first bin) in *first_bin. */
int64_t ps_welch_bins(int64_t window_len, double band_low, double band_high, int64_t* first_bin);

/* Replaces signalprep.normalize_phasors: z = a/|a| with the
 * amplitude-floor mask (masked samples exactly 0+0i).  Input complex (c64 /
 * c128) or real (then the analytic signal is formed first); output complex of
 * the input precision, dense [n_bands][n_trials][n_signals][n_samples];
 * mask_out (optional, uint8, same dense layout) gets 1 where masked. */
ps_status ps_normalize_phasors(ps_ctx* ctx, const ps_plv_args* args, void* out, uint8_t* mask_out);

/* Combines the partial metric sums of a (band, trial)-sharded computation
 * (PS_TRIALS_SUM) in a FIXED order ("deterministic tree order"):
 *   out[e] = (parts[0][e] + parts[1][e] + ... + parts[n_parts-1][e]) / divisor
 * summed left to right, part p at parts + p * part_stride elements; n elements.
 * dtype PS_F32 or PS_F64; device pointers; out may not alias parts.  Used
 * after an all-to-all that gives every rank the P partials of its output row
 * slice (paper_1710_08037_b200/sharding.py reduce_trial_partials). */
ps_status ps_reduce_partials(ps_ctx* ctx, const void* parts, int32_t n_parts, int64_t part_stride, int64_t n,
                             double divisor, int32_t dtype, void* out, void* stream);

/* Output-tile gather (SURVEY 8(e) "gathering the output only if the caller
 * asks"): ps_shard_pack copies the upper-triangle tiles shard `shard_index` of
 * `shard_count` owns (the rule of ps_pair_shard) out of a [N][N] matrix into
 * a dense buffer of ps_shard_tiles() tiles x tile_rows x tile_cols elements
 * (tile order = the library's enumeration); ps_shard_unpack writes the owned
 * entries (i <= j) of such a buffer, received from shard `shard_index`, into a
 * [N][N] matrix, plus the mirror (j, i) when `mirror` is 1 (negated when
 * `mirror` is -1, the antisymmetric signed imaginary part).  dtype PS_F32 (split
 * outputs) or PS_F64 (fp64 outputs); device pointers. */
int64_t ps_shard_tiles(int64_t n_signals, int32_t precision, int32_t shard_count, int32_t shard_index,
                       int32_t* tile_rows, int32_t* tile_cols);
ps_status ps_shard_pack(ps_ctx* ctx, int64_t n_signals, int32_t precision, int32_t shard_count, int32_t shard_index,
                        const void* matrix, void* packed, void* stream);
ps_status ps_shard_unpack(ps_ctx* ctx, int64_t n_signals, int32_t precision, int32_t shard_count,
                          int32_t shard_index, const void* packed, void* matrix, int32_t mirror, void* stream);

/* Host-only helpers (no GPU needed): the output-tile sharding rule of
 * ps_plv_args.shard_index / shard_count.  ps_tile_count returns the number of
 * upper-triangle output tiles for n_signals at `precision`; ps_pair_shard the
 * shard that writes pair (i, j) (and its mirror) for shard_count shards. */
int64_t ps_tile_count(int64_t n_signals, int32_t precision);
int32_t ps_pair_shard(int64_t n_signals, int32_t precision, int32_t shard_count, int64_t i, int64_t j);

#ifdef __cplusplus
}
#endif
#endif /* PHASESYNC_H_ */
