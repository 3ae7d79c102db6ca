// Internal declarations shared by the host layer (capi.cu) and the kernels.
// Data layout in HBM:
//   rows      = n_bands * n_trials * n_signals; row r = (b*R + t)*N + n
//   pitch     = Tp = roundup(T, 8) elements (16-byte TMA stride rule)
//   split     : fp16 planes [4][rows][Tp] = {re_hi, re_lo, im_hi, im_lo}
//   fp64      : f64 planes  [2][rows][Tp] = {re, im}
//   rowstat   : per row {min |a|, max |a|} as order-preserving unsigned bits
//   maskcount : per row number of masked samples (int32)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ps {

enum DevFlags : int {
  FLAG_ALL_MASKED = 1,
  FLAG_EMPTY_WINDOW = 2,
  FLAG_NONFINITE = 4,
  FLAG_TIMEOUT = 8,
  FLAG_ANY_MASKED = 16,
};

// Device-visible status words (one small device allocation per context).
struct DevStatus {
  int flags;                 // DevFlags
  int n_fix_rows;            // rows that needed the exact-median path
  unsigned long long n_masked;
  unsigned long long n_illcond;   // ciPLV pairs flagged ill-conditioned
  unsigned long long n_indeterminate;  // split: |Re| rounds to 1 with |Im| > tol (ciPLV reported 0)
  int pad[8];
};

// Where the (possibly strided) source samples of row r live.
struct SrcDesc {
  const void* ptr;           // base pointer of the source (input or packed copy)
  int kind;                  // 0 real, 1 complex (analytic), 2 complex (phasor)
  int is_double;             // scalar type of the source
  long long N, R, B, T;
  long long s_sig, s_samp, s_trial, s_band;   // element strides
  const void* hbuf;          // H{x} for real input: [rows_in_chunk][T] scalar
  long long h_row0;          // first row held in hbuf
  long long h_ld;            // hbuf row stride (elements; T unless band-pass padded)
  const void* h_scale;       // per-row factor on hbuf values ([rows_in_chunk], hbuf type), nullptr = 1
  int gauss_planes;          // split output for the Gauss Gram: planes 4..7 (S, D hi / lo) are
                             // written by the vectorised normaliser and zeroed by the fixup
};

// An ill-conditioned ciPLV value of the split path queued for exact FP64
// recomputation (slot / pair / units of one epilogue round + the value the
// epilogue emitted).  Sorted on the host before the refine kernel runs, so
// corrections are applied in a fixed order (deterministic output).
struct RefineEntry {
  int slot, i, j, u0, nu;
  float approx;
};

// One Gram work item: band b, trial group g (trials [g*Rg, min(R,(g+1)*Rg))),
// row panel I (BM rows), column panel J (BN cols).
struct Item { int b, g, I, J; };

struct GramParams {
  int N, T, R, B;
  int Tp;
  int rows;                  // B*R*N
  int Rg;                    // trials per group
  int G;                     // groups per band
  int pool;                  // 1: K runs over all R*T observations
  int n_items;
  const Item* items;
  // outputs (nullptr = not requested); element type float (split) / double (fp64)
  // Each output is an array of [N][N] slots; the slot written by a round is
  //   slot_mode 0: b*R + r     (per trial, PS_TRIALS_NONE)
  //   slot_mode 1: b           (per band: MEAN with one group, or POOL)
  //   slot_mode 2: b*G + g     (per trial group, reduced afterwards)
  void* out_plv; void* out_iplv; void* out_ciplv; void* out_cre; void* out_cim;
  int slot_mode;
  int mean_div;                // divisor applied at the last round of a slot (1 = none)
  // masks
  const int* maskcount;        // [rows]
  const void* planes;          // planes base (for masked-overlap scan)
  long long plane_stride;      // elements between planes
  DevStatus* status;
  // timing / debug
  float illcond_tol;           // flag ciPLV pairs whose predicted error > tol
  RefineEntry* refine;         // queue of flagged pairs (nullptr: count only)
  int refine_cap;
  int kc_blocks;               // split kernel: K blocks per TMEM accumulation chunk (drain period)
  int debug_flags;             // experiments only (PS_DEBUG_EPI): 1 = skip the metric emission
  int upper_only;              // PS_LAYOUT_UPPER: the final outputs hold i <= j only (refinement skips mirrors)
  int slot_upper;              // the Gram writes only i <= j of its output slots (no mirror (j, i) stores):
                               // PS_LAYOUT_UPPER, and trial-group partial-sum slots, whose reduce mirrors
  // Producer lockstep (split kernel): every producer publishes each group of
  // lock_group issued K blocks in lock_cnt[group] and may not run more than
  // lock_lag groups ahead of the slowest producer, so the CTAs that share an
  // operand panel stream it through L2 together (one DRAM read per panel
  // slice instead of one per CTA).  lock_cnt == nullptr disables it.
  int* lock_cnt;
  int lock_group;
  int lock_lag;
  int lock_rounds;             // rounds per item (uniform across items when enabled)
  // Streamed copy-out (split kernel, pipelined host path): item n belongs to
  // output sub-block item_sb[n]; every epilogue warp that finished emitting an
  // item fences its stores and counts in sb_cnt[sb]; the arrival that reaches
  // sb_need[sb] publishes sb_flag[sb] = 1 into mapped host memory, so the host
  // ships that block while the kernel keeps running.  sb_cnt == nullptr: off.
  int* sb_cnt;
  const int* item_sb;
  const int* sb_need;
  volatile int* sb_flag;
  // Per-pair observation counts (K7 mask-count Gram): written by
  // the count kernel ([slots][N][N] int32, slot = b*R + r, or b for pool),
  // read by the metric epilogues in place of the plane scan when samples are
  // masked.  nullptr: no count pass ran.
  int* cnt;
  // PS_GRAM_PROF=1 (diagnostics): cycles the pipeline roles spent blocked,
  // summed over CTAs: [0] MMA issuer on operand stages (full), [1] MMA issuer
  // on accumulation buffers (tempty), [2] MMA issuer total, [3] producer on
  // free stages (empty), [4] producer total.  nullptr: off.
  unsigned long long* prof;
  // split kernel producer: L2 prefetch distance in K blocks (0 = off); the
  // operand slices of block kb + prefetch_blocks are pulled into L2 while
  // block kb is loaded into shared memory (hides DRAM latency the few
  // shared-memory stages cannot)
  int prefetch_blocks;
};

// ---- launchers (return cudaError_t) --------------------------------------
cudaError_t launch_pack_real(const SrcDesc& src, long long row0, long long nrows,
                             void* dst, int dst_double, cudaStream_t st);
// packing copy scaled per row by a power of two (odd T: cuFFT pairs rows)
cudaError_t launch_pack_real_scaled(const SrcDesc& src, long long row0, long long nrows, void* dst, void* inv_scale,
                                    int dst_double, cudaStream_t st);
// in-place per-row power-of-two scaling of [rows][L] (stride ld) / its undo
cudaError_t launch_scale_rows(void* y, long long nrows, long long L, long long ld, void* inv_scale, int undo,
                              int is_double, cudaStream_t st);
cudaError_t launch_hilbert_spectrum(void* spec, long long nrows, int T, int is_double,
                                    cudaStream_t st);
// even T: the multiplier between two half-length complex transforms
// ([nrows][T / 2] complex, in place; see hilbert_halfspec_kernel)
cudaError_t launch_hilbert_halfspec(void* spec, long long nrows, int T, int is_double, cudaStream_t st);
// fmt: 0 split fp16 planes, 1 f64 planes, 2 complex interleaved (compute type)
// cdouble: compute in double although the source is float
// *gauss_done (optional) = 1 when the Gauss planes 4..7 were written too
// (vectorised path with src.gauss_planes), else 0
cudaError_t launch_normalize_fmt(const SrcDesc& src, long long row0, long long nrows, void* out, int fmt,
                                 int cdouble, int pitch, long long plane_stride, unsigned long long* rowstat,
                                 long long rows_total, DevStatus* status, cudaStream_t st, int* gauss_done = nullptr);
cudaError_t launch_fixup_fmt(const SrcDesc& src, long long row0, long long nrows, void* out, int fmt,
                             int cdouble, int pitch, long long plane_stride, const unsigned long long* rowstat,
                             long long rows_total, int* maskcount, double amp_floor, DevStatus* status,
                             cudaStream_t st);
// Fused Hilbert + normalise (real fp32 rows, T = 4096, split planes): writes
// planes and row min/max; H lands in src.hbuf only for rows the fixup inspects.
// With src.gauss_planes it also writes the Gauss-Gram S / D planes (*gauss_done = 1).
bool hilbert_fused_supported(const SrcDesc& src, int fmt, int cdouble, int pitch);
cudaError_t launch_hilbert_fused(const SrcDesc& src, long long row0, long long nrows, void* out, int pitch,
                                 long long plane_stride, unsigned long long* rowstat, long long rows_total,
                                 double amp_floor, DevStatus* status, cudaStream_t st, int* gauss_done);
// Band-pass front end (two-pass FIR evaluated spectrally on length Lf)
cudaError_t launch_reflect_pad(const SrcDesc& src, long long row0, long long nrows, long long pad, long long L,
                               long long Lf, void* xp, int dst_double, cudaStream_t st);
cudaError_t launch_spectrum_mul(void* spec, long long nrows, long long nb, const void* Hf, int conj, double scale,
                                int is_double, cudaStream_t st);
cudaError_t launch_zero_tail(void* y, long long nrows, long long L, long long Lf, int is_double, cudaStream_t st);
cudaError_t launch_trim_rows(const void* y, long long nrows, long long ld, long long pad, long long T, void* out,
                             int is_double, cudaStream_t st);
// *dst = *src on the device (dst may be mapped pinned host memory)
cudaError_t launch_copy_u64(const unsigned long long* src, unsigned long long* dst, cudaStream_t st);
// Welch coherence front end: tapered segments, per-bin normalised Gram operand
// rows, and the max-over-bins band reduction
cudaError_t launch_welch_segments(const SrcDesc& src, long long rows, int nseg, int W, int hop, const double* win,
                                  void* seg, int dst_double, cudaStream_t st);
cudaError_t launch_coherence_planes(const void* spec, int spec_double, int nbW, long long B, long long R, long long N,
                                    int nseg, int k0, int nb, int K, int Kp, void* planes, long long ps, int split,
                                    cudaStream_t st);
// upper_n = N for PS_LAYOUT_UPPER (strictly lower entries skipped), 0 = all
cudaError_t launch_band_max(const void* ws, long long B, long long nb, long long nn, void* out, int is_double,
                            cudaStream_t st, long long upper_n);
cudaError_t launch_analytic_out(const SrcDesc& src, long long row0, long long nrows,
                                void* out, cudaStream_t st);
// Eq 8 (over trials): planes [P][B*R][N][Tp] -> [P][B*T][N][Rp] + masked-trial counts
cudaError_t launch_transpose_trials(const void* src, long long sps, int Tp, void* dst, long long dps, int Rp, int B,
                                    int R, int N, int T, int split, int* maskcount_dst, cudaStream_t st);
// Trial-group reduce: out_m[b] = sum_g ws_m[b][g] scaled by 1 / R, from slots
// holding only i <= j (GramParams::slot_upper); upper = 1 writes i <= j of the
// outputs, upper = 0 both triangles (the mirror through shared-memory tiles,
// negated for the antisymmetric signed Im output, m = 4).
cudaError_t launch_group_reduce(const void* ws, int G, int N, int B, int n_outputs, void* const* outs, int R,
                                int is_double, cudaStream_t st, int upper);
// K7: per-pair observation counts from the unmasked-indicator plane (same
// items / tiles / cluster layout as the split Gram; p.cnt receives the counts)
cudaError_t launch_gram_count(const void* tmapA, const void* tmapB, const GramParams& p, int groups, cudaStream_t st);
// unmasked indicator u(t) (fp16 0 / 1, padding 0) of every plane row
cudaError_t launch_indicator_plane(const void* planes, long long plane_stride, int split, long long rows, int Tp,
                                   int T, void* ind, int ind_pitch, cudaStream_t st);
cudaError_t launch_gram_split(const void* tmapA, const void* tmapB, const void* tmapB2, bool gauss,
                              const GramParams& p, int grid, cudaStream_t st);
// Gauss-Gram planes 4..7 (S, D hi / lo) from planes 0..3, flat elements [e0, e1)
cudaError_t launch_gauss_planes(void* planes, long long plane_stride, long long e0, long long e1, cudaStream_t st);
cudaError_t launch_gram_f64(const GramParams& p, int grid, cudaStream_t st);
// Exact FP64 recomputation of queued ciPLV pairs.  groups[g]..groups[g+1]
// index a run of entries (sorted by slot, i, j, u0) sharing one output
// location; `overwrite` = the slot holds a single round (else the mean over
// `div` rounds gets (exact - approx) / div added).
cudaError_t launch_refine(const GramParams& p, const RefineEntry* entries, const int* groups, int n_groups,
                          int n_entries, double* exact, int overwrite, int div, cudaStream_t st);
// Same, with the queue ordered on the device (entries modified in place:
// slot /= slot_div; sorted copy in `sorted`, group starts in `groups`,
// n + 1 ints).  ib = bits of the signal index; the packed key needs
// bits(slot) + 2 ib <= 64.
size_t refine_sort_ws_bytes(int n);
// (flat output index, final ciPLV value) of queued refine entries (split outputs)
cudaError_t launch_refine_pick(const RefineEntry* entries, int n, const float* out, long long N, long long* idx,
                               float* val, cudaStream_t st);
cudaError_t launch_refine_sorted(const GramParams& p, RefineEntry* entries, int n, int slot_div, int ib, int key_bits,
                                 void* ws, size_t ws_bytes, RefineEntry* sorted, double* exact, int* groups, int overwrite,
                                 int div, cudaStream_t st);

// multi-GPU combine / gather (shard_kernels.cu)
cudaError_t launch_reduce_partials(const void* parts, int P, long long stride, long long n, double div, int is_double,
                                   void* out, cudaStream_t st);
cudaError_t launch_shard_pack(const void* M, long long N, const void* tiles, int n_tiles, int bm, int bn, int is_double,
                              void* packed, cudaStream_t st);
cudaError_t launch_shard_unpack(const void* packed, long long N, const void* tiles, int n_tiles, int bm, int bn,
                                int is_double, void* M, int mirror, cudaStream_t st);

// split Gram variant: 2 = CTA pair (cta_group::2, 256-row panels), 1 = single
// CTA (128-row panels).  PS_CTA_GROUP=1 selects the latter.
int split_cta_group();
int split_panel_rows();   // rows of one execution panel (= UMMA M)
int split_b_box_rows();   // J-panel rows staged per CTA
int split_epi_arrivals(); // epilogue warps per CTA group (arrivals per item on GramParams::sb_cnt)
// Gauss Gram operand feed: false (default) = TMA streams the precomputed
// S / D planes 4..7 too; true (PS_GAUSS_CONV=1, experiment, slower) = TMA
// streams the 4 split planes {Zr, Zi} hi / lo and the epilogue warps form
// S / D in shared memory
bool gauss_smem_convert();

// tile geometry of the two Gram kernels (ownership / sharding granularity)
constexpr int kSplitBM = 256;
constexpr int kSplitBN = 128;
constexpr int kSplitBK = 32;
constexpr int kF64BM = 64;
constexpr int kF64BN = 64;

}  // namespace ps
