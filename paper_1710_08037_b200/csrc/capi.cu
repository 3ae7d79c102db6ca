// Host side of libphasesync_cuda.so: the C ABI declared in include/phasesync.h.
//
// Owns per-context resources only (cuFFT plans, growable device workspace,
// cached TMA descriptors and work-item tables); results are never cached
// (SPEC.md:548).  Every entry point validates its arguments, launches the
// sm_100a pipeline on the caller's stream, synchronises that stream and maps
// device-side status flags to ps_status codes ("errors mapped 1:1").
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <atomic>
#include <memory>
#include <chrono>
#include <thread>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/phasesync.h"
#include "ps_internal.h"

using namespace ps;

namespace {

thread_local std::string g_last_error;

ps_status fail(ps_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

#define PS_CUDA(call)                                                                                   \
  do {                                                                                                  \
    cudaError_t e_ = (call);                                                                            \
    if (e_ != cudaSuccess)                                                                              \
      return fail(e_ == cudaErrorMemoryAllocation ? PS_E_OOM : PS_E_CUDA,                               \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                                  \
  } while (0)

#define PS_CUFFT(call)                                                                                  \
  do {                                                                                                  \
    cufftResult r_ = (call);                                                                            \
    if (r_ != CUFFT_SUCCESS) return fail(PS_E_CUFFT, std::string(#call) + ": cufft error " + std::to_string((int)r_)); \
  } while (0)

#define PS_TRY(expr)                 \
  do {                               \
    ps_status s_ = (expr);           \
    if (s_ != PS_OK) return s_;      \
  } while (0)

struct Buf {
  void* p = nullptr;
  size_t n = 0;
};

using PlanKey = std::tuple<int, long long, long long, int, int>;  // T, batch, idist, double, dir

struct TmapKey {
  const void* base;
  long long T, N, U, pitch;
  bool gauss;
  bool operator<(const TmapKey& o) const {
    return std::tie(base, T, N, U, pitch, gauss) < std::tie(o.base, o.T, o.N, o.U, o.pitch, o.gauss);
  }
};
struct Tmaps {
  CUtensorMap a, b, b2;  // A panel, B panel (planes 0..), B panel planes 4..7 (Gauss)
};

}  // namespace

struct ps_ctx {
  int device = 0;
  int num_sms = 148;
  size_t total_mem = 0;  // device memory (cudaDeviceProp.totalGlobalMem)
  bool timing = false;
  std::mutex mu;
  std::map<PlanKey, cufftHandle> plans;
  Buf xw, spec, hbuf, planes, rowstat, maskcount, items, gws, hin, hout, refine, refine_sorted, planes_t, maskcount_t;
  Buf fir_taps, fir_spec;  // band-pass front end: padded taps, filter spectrum (double)
  Buf cohws;               // coherence: per-bin matrices before the max-over-bins reduction
  Buf lockbuf;             // Gram producer lockstep counters (one launch at a time per ctx)
  Buf hscale;              // per-row factors restoring H after scaled packing (odd T)
  Buf sortws;              // device-side ordering of the ciPLV refinement queue
  Buf shardtiles;          // (I, J) of the tiles one shard owns (ps_shard_pack / unpack)
  Buf ind, cntws, cntitems;  // K7: unmasked-indicator plane, per-pair counts, count-pass items
  Buf profbuf;               // PS_GRAM_PROF counters
  std::vector<cudaEvent_t> tev;  // timing events of the staged path (2 per stage)
  DevStatus* d_status = nullptr;
  DevStatus* h_status = nullptr;  // pinned
  std::map<TmapKey, Tmaps> tmaps;
  std::vector<Item> h_items;
  Item* h_items_pinned = nullptr;
  size_t h_items_cap = 0;
  cudaEvent_t ev[8] = {};
  int launches = 0;
  // host (e2e) pipeline: copy-in / compute / refine / copy-out streams
  cudaStream_t s_in = nullptr, s_comp = nullptr, s_ref = nullptr, s_out = nullptr, s_prep = nullptr;
  std::vector<cudaEvent_t> evpool;
  unsigned long long* h_cnt = nullptr;  // mapped pinned per-stage refine-queue counters
  unsigned long long* d_cnt = nullptr;  // device alias of h_cnt
  int h_cnt_cap = 0;
  // streamed copy-out of the pipelined host path (upper layout)
  Buf sbinfo;                    // device: item_sb[items] | sb_need[sb] | sb_cnt[sb]
  Buf rpick;                     // device: (index, value) of refined ciPLV entries
  std::vector<int> h_sbinfo;     // host staging of item_sb | sb_need
  int* h_sbflag = nullptr;       // mapped pinned per-sub-block ready flags
  int* d_sbflag = nullptr;       // device alias of h_sbflag
  int h_sbflag_cap = 0;
};

namespace {

ps_status ensure(Buf& b, size_t bytes) {
  if (bytes <= b.n) return PS_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.n = 0;
  size_t want = std::max(bytes, (size_t)256);
  cudaError_t e = cudaMalloc(&b.p, want);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(PS_E_OOM, "cudaMalloc(" + std::to_string(want) + " bytes) failed: " + cudaGetErrorString(e));
  }
  b.n = want;
  return PS_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

long long round_up(long long a, long long b) { return (a + b - 1) / b * b; }

struct Geometry {
  long long B, N, T, R, rows;
  bool cdouble;   // compute type of the Hilbert / normalise stage
  bool split;     // split fp16 planes vs fp64 planes
  bool complex_in;
  int in_double;  // input scalar is double
  long long pitch;
  long long plane_stride;
  // split Gram as the 3-product (Gauss) complex product: planes 4..7 hold
  // S = Zr + Zi and D = Zr - Zi (hi / lo) next to {Re hi, Re lo, Im hi, Im lo}
  bool gauss = false;
  int nplanes() const { return split ? (gauss ? 8 : 4) : 2; }
  size_t plane_bytes() const { return (size_t)nplanes() * plane_stride * (split ? 2 : 8); }
};

ps_status validate(const ps_plv_args* a, Geometry& g) {
  if (!a) return fail(PS_E_INVALID, "args is NULL");
  if (!a->input) return fail(PS_E_INVALID, "input pointer is NULL");
  if (a->n_bands < 1 || a->n_signals < 1 || a->n_trials < 1)
    return fail(PS_E_SHAPE, "expected axes [n_signals x n_samples x n_trials] with n_signals >= 1, n_trials >= 1 "
                            "(SPEC.md:31)");
  if (a->n_samples < 2) return fail(PS_E_SHAPE, "n_samples must be >= 2 (SPEC.md:31)");
  if (a->dtype < PS_F32 || a->dtype > PS_C128) return fail(PS_E_INVALID, "unknown dtype");
  const bool cplx = a->dtype == PS_C64 || a->dtype == PS_C128;
  if (a->input_kind == PS_INPUT_REAL && cplx)
    return fail(PS_E_INVALID, "real input_kind requires a real dtype (f32/f64)");
  if (a->input_kind != PS_INPUT_REAL && !cplx)
    return fail(PS_E_INVALID, "analytic/phasor input_kind requires a complex dtype (c64/c128)");
  if (a->input_kind < 0 || a->input_kind > 2) return fail(PS_E_INVALID, "unknown input_kind");
  if (a->precision != PS_PREC_SPLIT_F16X3 && a->precision != PS_PREC_FP64)
    return fail(PS_E_INVALID, "unknown precision");
  if (a->trial_reduce < 0 || a->trial_reduce > 3) return fail(PS_E_INVALID, "unknown trial_reduce");
  if (a->mode != PS_MODE_OVER_SAMPLES && a->mode != PS_MODE_OVER_TRIALS) return fail(PS_E_INVALID, "unknown mode");
  if (a->out_layout != PS_LAYOUT_FULL && a->out_layout != PS_LAYOUT_UPPER)
    return fail(PS_E_INVALID, "unknown out_layout");
  if (!(a->amp_floor >= 0.0)) return fail(PS_E_INVALID, "amp_floor must be >= 0");
  if (a->n_signals > (1 << 30) || a->n_samples > (1LL << 31) - 1)
    return fail(PS_E_SHAPE, "n_signals / n_samples exceed the supported range");
  if (a->fir) {
    if (a->input_kind != PS_INPUT_REAL) return fail(PS_E_INVALID, "the band-pass front end applies to real input");
    if (!a->fir->taps || a->fir->n_taps < 1) return fail(PS_E_INVALID, "fir: taps missing");
    if (a->fir->pad_samples < 0) return fail(PS_E_INVALID, "fir: pad_samples must be >= 0");
    if (a->n_samples <= a->fir->n_taps)
      return fail(PS_E_SIGNAL_TOO_SHORT, "n_samples must exceed order + 1 (SPEC.md:69)");
    if (a->fir->pad_samples >= a->n_samples)
      return fail(PS_E_SIGNAL_TOO_SHORT, "reflection padding needs pad_samples < n_samples (SPEC.md:122)");
    if (a->n_samples + 2 * a->fir->pad_samples + a->fir->n_taps > (1LL << 30))
      return fail(PS_E_SHAPE, "padded record length exceeds the supported range");
  }
  g.B = a->n_bands;
  g.N = a->n_signals;
  g.T = a->n_samples;
  g.R = a->n_trials;
  g.rows = g.B * g.R * g.N;
  g.complex_in = cplx;
  g.in_double = (a->dtype == PS_F64 || a->dtype == PS_C128) ? 1 : 0;
  g.split = a->precision == PS_PREC_SPLIT_F16X3;
  g.cdouble = g.in_double || !g.split;
  g.pitch = g.split ? round_up(g.T, 8) : round_up(g.T, 16);
  g.plane_stride = g.rows * g.pitch;
  return PS_OK;
}

SrcDesc make_src(const ps_plv_args* a, const Geometry& g, const void* ptr) {
  SrcDesc s;
  s.ptr = ptr;
  s.kind = a->input_kind;
  s.is_double = g.in_double;
  s.N = g.N;
  s.R = g.R;
  s.B = g.B;
  s.T = g.T;
  s.s_sig = a->stride_signal;
  s.s_samp = a->stride_sample;
  s.s_trial = a->stride_trial;
  s.s_band = a->stride_band;
  s.hbuf = nullptr;
  s.h_row0 = 0;
  s.h_ld = g.T;
  s.h_scale = nullptr;
  s.gauss_planes = 0;
  return s;
}

// Rows directly consumable by a single batched cuFFT plan: sample stride 1,
// dtype == compute type and row r at offset r * stride_signal.
bool fft_direct(const ps_plv_args* a, const Geometry& g) {
  if (a->stride_sample != 1) return false;
  if ((bool)g.in_double != g.cdouble) return false;
  const long long s = a->stride_signal;
  if (s < g.T) return false;
  if (g.R > 1 && a->stride_trial != g.N * s) return false;
  if (g.B > 1 && a->stride_band != g.R * g.N * s) return false;
  return true;
}

ps_status get_plan(ps_ctx* c, int T, long long batch, long long idist, bool dbl, int dir, cufftHandle* out) {
  PlanKey k{T, batch, idist, dbl ? 1 : 0, dir};
  auto it = c->plans.find(k);
  if (it != c->plans.end()) {
    *out = it->second;
    return PS_OK;
  }
  cufftHandle h;
  PS_CUFFT(cufftCreate(&h));
  long long n[1] = {T};
  long long nb = T / 2 + 1;
  size_t ws = 0;
  cufftResult r;
  if (dir == 2) {  // C2C / Z2Z of length T / 2: rows of distance idist (complex elements) -> dense rows
    long long m[1] = {T / 2};
    long long inembed[1] = {idist}, onembed[1] = {T / 2};
    r = cufftMakePlanMany64(h, 1, m, inembed, 1, idist, onembed, 1, T / 2, dbl ? CUFFT_Z2Z : CUFFT_C2C, batch, &ws);
  } else if (dir == 0) {  // R2C / D2Z: input real rows of distance idist, output half spectra
    long long inembed[1] = {idist}, onembed[1] = {nb};
    r = cufftMakePlanMany64(h, 1, n, inembed, 1, idist, onembed, 1, nb, dbl ? CUFFT_D2Z : CUFFT_R2C, batch, &ws);
  } else {         // C2R / Z2D: half spectra -> dense real rows of length T
    long long inembed[1] = {nb}, onembed[1] = {T};
    r = cufftMakePlanMany64(h, 1, n, inembed, 1, nb, onembed, 1, T, dbl ? CUFFT_Z2D : CUFFT_C2R, batch, &ws);
  }
  if (r != CUFFT_SUCCESS) {
    cufftDestroy(h);
    return fail(PS_E_CUFFT, "cufftMakePlanMany64 failed: " + std::to_string((int)r));
  }
  c->plans[k] = h;
  *out = h;
  return PS_OK;
}

// Which chain takes real rows of even length T.  cuFFT's R2C / C2R run as a
// half-length complex transform plus a split / merge pass each for most
// lengths, and the half-length complex chain with the collapsed multiplier
// saves two of the five passes (C2, T = 10000: 2.54 -> 1.91 ms).  For powers
// of two cuFFT has single symmetric kernels (8 B/sample each); measured per
// 67 M samples (tools/hilbert_probe.py, R2C chain / half-length chain, ms):
// T = 512 0.95 / 0.73, 2048 0.50 / 0.47, 8192 0.61 / 0.57, 16384 0.57 / 0.51,
// 32768 0.72 / 0.60, 65536 0.75 / 0.76, 131072 1.00 / 0.80 -- the half-length
// chain everywhere except T = 65536 (C3), a tie it loses by 2%.
// PS_HILBERT_CHAIN=r2c / half forces one (A/B, tests of both).
bool hilbert_half_chain(long long T) {
  const char* s = std::getenv("PS_HILBERT_CHAIN");  // read per call: tests switch it
  const int forced = (s && std::string(s) == "r2c") ? 0 : (s && std::string(s) == "half") ? 1 : -1;
  if (T % 2 != 0 || T < 4) return false;
  if (forced >= 0) return forced == 1;
  return T != 65536;
}

long long hilbert_chunk_rows(const Geometry& g) {
  const long long target = 1LL << 27;  // samples per chunk (bounds spectrum + H workspace)
  long long rc = target / g.T;
  rc = std::max(1LL, std::min(rc, g.rows));
  return rc;
}

// H{x} of nr real rows of even length L at `in` (row distance idist reals,
// even; base aligned like the complex type) into c->hbuf (dense rows of L):
// C2C of length L / 2 -> collapsed multiplier -> C2C (hilbert_halfspec_kernel).
// c->spec must hold nr * L / 2 complex values.
ps_status hilbert_half_exec(ps_ctx* c, long long L, long long nr, const void* in, long long idist, bool dbl,
                            cudaStream_t st) {
  const long long M = L / 2;
  cufftHandle fw, iv;
  PS_TRY(get_plan(c, (int)L, nr, idist / 2, dbl, 2, &fw));
  PS_TRY(get_plan(c, (int)L, nr, M, dbl, 2, &iv));
  PS_CUFFT(cufftSetStream(fw, st));
  if (dbl) {
    PS_CUFFT(cufftExecZ2Z(fw, (cufftDoubleComplex*)const_cast<void*>(in), (cufftDoubleComplex*)c->spec.p, CUFFT_FORWARD));
  } else {
    PS_CUFFT(cufftExecC2C(fw, (cufftComplex*)const_cast<void*>(in), (cufftComplex*)c->spec.p, CUFFT_FORWARD));
  }
  PS_CUDA(launch_hilbert_halfspec(c->spec.p, nr, (int)L, dbl ? 1 : 0, st));
  c->launches++;
  PS_CUFFT(cufftSetStream(iv, st));
  if (dbl) {
    PS_CUFFT(cufftExecZ2Z(iv, (cufftDoubleComplex*)c->spec.p, (cufftDoubleComplex*)c->hbuf.p, CUFFT_INVERSE));
  } else {
    PS_CUFFT(cufftExecC2C(iv, (cufftComplex*)c->spec.p, (cufftComplex*)c->hbuf.p, CUFFT_INVERSE));
  }
  return PS_OK;
}

// Hilbert stage for rows [row0, row0+nr): leaves H{x} (compute type) in c->hbuf.
// For odd T cuFFT's batched R2C transforms two rows as one complex sequence,
// so a row's rounding error scales with its partner's magnitude: the rows are
// then packed with a per-row power-of-two scale first and *h_scale receives
// the per-row factors that restore H (SrcDesc::h_scale; nullptr otherwise).
ps_status hilbert_chunk(ps_ctx* c, const ps_plv_args* a, const Geometry& g, const SrcDesc& src, long long row0,
                        long long nr, cudaStream_t st, bool* copied, const void** h_scale) {
  const size_t es = g.cdouble ? 8 : 4;
  const long long nb = g.T / 2 + 1;
  PS_TRY(ensure(c->spec, (size_t)nr * nb * 2 * es));
  PS_TRY(ensure(c->hbuf, (size_t)nr * g.T * es));
  const void* in = nullptr;
  long long idist = g.T;
  *h_scale = nullptr;
  if (g.T % 2 == 1) {
    PS_TRY(ensure(c->xw, (size_t)nr * g.T * es));
    PS_TRY(ensure(c->hscale, (size_t)nr * es));
    PS_CUDA(launch_pack_real_scaled(src, row0, nr, c->xw.p, c->hscale.p, g.cdouble ? 1 : 0, st));
    c->launches++;
    in = c->xw.p;
    *h_scale = c->hscale.p;
  } else if (fft_direct(a, g) && a->stride_signal % 2 == 0 &&
             (reinterpret_cast<uintptr_t>(static_cast<const char*>(src.ptr) + (size_t)row0 * a->stride_signal * es) %
              (2 * es)) == 0) {
    // (cuFFT wants real input rows aligned like its complex type: a view that
    // starts an odd number of elements into its buffer is packed instead)
    in = static_cast<const char*>(src.ptr) + (size_t)row0 * a->stride_signal * es;
    idist = a->stride_signal;
  } else {
    PS_TRY(ensure(c->xw, (size_t)nr * g.T * es));
    PS_CUDA(launch_pack_real(src, row0, nr, c->xw.p, g.cdouble ? 1 : 0, st));
    c->launches++;
    in = c->xw.p;
    *copied = true;
  }
  if (hilbert_half_chain(g.T)) {
    // Even T: the row re-read as T / 2 complex samples, one C2C each way and
    // the collapsed multiplier in between (hilbert_halfspec_kernel): cuFFT's
    // own R2C / C2R do the same half-length transforms plus a split / merge
    // pass each, which with the -i sgn(k) pass made three passes of this one.
    // (in is aligned and idist even: direct rows passed the check above, packed rows are dense)
    return hilbert_half_exec(c, g.T, nr, in, idist, g.cdouble, st);
  }
  cufftHandle fwd, inv;
  PS_TRY(get_plan(c, (int)g.T, nr, idist, g.cdouble, 0, &fwd));
  PS_TRY(get_plan(c, (int)g.T, nr, g.T, g.cdouble, 1, &inv));
  PS_CUFFT(cufftSetStream(fwd, st));
  PS_CUFFT(cufftSetStream(inv, st));
  if (g.cdouble) {
    PS_CUFFT(cufftExecD2Z(fwd, (cufftDoubleReal*)in, (cufftDoubleComplex*)c->spec.p));
  } else {
    PS_CUFFT(cufftExecR2C(fwd, (cufftReal*)in, (cufftComplex*)c->spec.p));
  }
  PS_CUDA(launch_hilbert_spectrum(c->spec.p, nr, (int)g.T, g.cdouble ? 1 : 0, st));
  c->launches++;
  if (g.cdouble) {
    PS_CUFFT(cufftExecZ2D(inv, (cufftDoubleComplex*)c->spec.p, (cufftDoubleReal*)c->hbuf.p));
  } else {
    PS_CUFFT(cufftExecC2R(inv, (cufftComplex*)c->spec.p, (cufftReal*)c->hbuf.p));
  }
  return PS_OK;
}

// ---- band-pass front end (DESIGN.md 8(f) #1) -------
// Record of length L = T + 2 pad (reflection padded), filtered by the two-pass
// FIR evaluated spectrally on Lf >= L + n_taps - 1 (no wrap-around), then the
// analytic signal of the padded record (length-L Hilbert), trimmed to T.
struct FirGeom {
  long long P = 0, L = 0, Lf = 0, nt = 0;
};

long long next_fast_len(long long n) {  // smallest EVEN 2^a 3^b 5^c 7^d >= n
  // (even: cuFFT's odd-length R2C pairs two rows of the batch into one complex
  // transform, which would couple the rounding error of rows of unequal scale)
  for (long long m = std::max(n + (n & 1), 2LL);; m += 2) {
    long long r = m;
    for (long long f : {2LL, 3LL, 5LL, 7LL})
      while (r % f == 0) r /= f;
    if (r == 1) return m;
  }
}

FirGeom fir_geom(const ps_plv_args* a, const Geometry& g) {
  FirGeom f;
  f.P = a->fir->pad_samples;
  f.nt = a->fir->n_taps;
  f.L = g.T + 2 * f.P;
  f.Lf = next_fast_len(f.L + f.nt - 1);
  return f;
}

long long prep_chunk_rows(const ps_plv_args* a, const Geometry& g) {
  if (a->fir) {
    const long long rc = (1LL << 27) / fir_geom(a, g).Lf;
    return std::max(1LL, std::min(rc, g.rows));
  }
  return hilbert_chunk_rows(g);
}

// Call-scope preparation of the real-input stage: size the workspace once
// for the largest chunk (no reallocation between pipelined stages) and, with
// a band-pass front end, the filter spectrum Hf = FFT_Lf(taps) in double.
ps_status prep_begin(ps_ctx* c, const ps_plv_args* a, const Geometry& g, cudaStream_t st) {
  if (a->input_kind != PS_INPUT_REAL) return PS_OK;
  const size_t es = g.cdouble ? 8 : 4;
  const long long rc = std::min(prep_chunk_rows(a, g), g.rows);
  PS_TRY(ensure(c->hscale, (size_t)rc * es));
  if (!a->fir) {
    PS_TRY(ensure(c->spec, (size_t)rc * (g.T / 2 + 1) * 2 * es));
    PS_TRY(ensure(c->hbuf, (size_t)rc * g.T * es));
    PS_TRY(ensure(c->xw, (size_t)rc * g.T * es));
    return PS_OK;
  }
  const FirGeom f = fir_geom(a, g);
  PS_TRY(ensure(c->xw, (size_t)rc * f.Lf * es));
  PS_TRY(ensure(c->spec, (size_t)rc * (f.Lf / 2 + 1) * 2 * es));
  PS_TRY(ensure(c->hbuf, (size_t)rc * f.L * es));
  PS_TRY(ensure(c->fir_taps, (size_t)f.Lf * sizeof(double)));
  PS_TRY(ensure(c->fir_spec, (size_t)(f.Lf / 2 + 1) * 2 * sizeof(double)));
  PS_CUDA(cudaMemsetAsync(c->fir_taps.p, 0, (size_t)f.Lf * sizeof(double), st));
  PS_CUDA(cudaMemcpyAsync(c->fir_taps.p, a->fir->taps, (size_t)f.nt * sizeof(double), cudaMemcpyHostToDevice, st));
  cufftHandle h;
  PS_TRY(get_plan(c, (int)f.Lf, 1, f.Lf, true, 0, &h));
  PS_CUFFT(cufftSetStream(h, st));
  PS_CUFFT(cufftExecD2Z(h, (cufftDoubleReal*)c->fir_taps.p, (cufftDoubleComplex*)c->fir_spec.p));
  return PS_OK;
}

// Band-pass stage for rows [row0, row0+nr): c->xw rows (stride Lf) hold the
// filtered padded record; with `hilbert`, c->hbuf rows (stride L) hold its
// Hilbert transform.  *fs describes the trimmed (x_f, H) pair for the
// normalisation kernels (row r -> xw[(r - row0) * Lf + P + t]).
ps_status bandpass_chunk(ps_ctx* c, const ps_plv_args* a, const Geometry& g, const SrcDesc& src, long long row0,
                         long long nr, bool hilbert, cudaStream_t st, SrcDesc* fs) {
  const FirGeom f = fir_geom(a, g);
  const size_t es = g.cdouble ? 8 : 4;
  const int dbl = g.cdouble ? 1 : 0;
  const long long nbf = f.Lf / 2 + 1;
  PS_CUDA(launch_reflect_pad(src, row0, nr, f.P, f.L, f.Lf, c->xw.p, dbl, st));
  cufftHandle fwd, inv;
  PS_TRY(get_plan(c, (int)f.Lf, nr, f.Lf, g.cdouble, 0, &fwd));
  PS_TRY(get_plan(c, (int)f.Lf, nr, f.Lf, g.cdouble, 1, &inv));
  PS_CUFFT(cufftSetStream(fwd, st));
  PS_CUFFT(cufftSetStream(inv, st));
  auto r2c = [&](cufftHandle h, void* in) -> cufftResult {
    return dbl ? cufftExecD2Z(h, (cufftDoubleReal*)in, (cufftDoubleComplex*)c->spec.p)
               : cufftExecR2C(h, (cufftReal*)in, (cufftComplex*)c->spec.p);
  };
  auto c2r = [&](cufftHandle h, void* out) -> cufftResult {
    return dbl ? cufftExecZ2D(h, (cufftDoubleComplex*)c->spec.p, (cufftDoubleReal*)out)
               : cufftExecC2R(h, (cufftComplex*)c->spec.p, (cufftReal*)out);
  };
  const double inv_lf = 1.0 / (double)f.Lf;
  // pass 1: y1 = h * xp, truncated to L samples (zero initial state)
  PS_CUFFT(r2c(fwd, c->xw.p));
  PS_CUDA(launch_spectrum_mul(c->spec.p, nr, nbf, c->fir_spec.p, 0, inv_lf, dbl, st));
  PS_CUFFT(c2r(inv, c->xw.p));
  PS_CUDA(launch_zero_tail(c->xw.p, nr, f.L, f.Lf, dbl, st));
  // pass 2 on the reversed record == correlation with h: spectrum * conj(Hf)
  PS_CUFFT(r2c(fwd, c->xw.p));
  PS_CUDA(launch_spectrum_mul(c->spec.p, nr, nbf, c->fir_spec.p, 1, inv_lf, dbl, st));
  PS_CUFFT(c2r(inv, c->xw.p));
  c->launches += 5;
  const bool odd = (f.L & 1) != 0;
  if (hilbert && hilbert_half_chain(f.L)) {
    // even L that is not a power of two: the filtered records (row distance
    // Lf, even) re-read as L / 2 complex samples (see hilbert_chunk)
    PS_TRY(hilbert_half_exec(c, f.L, nr, c->xw.p, f.Lf, g.cdouble, st));
  } else if (hilbert) {  // analytic signal of the padded record (length L), before the trim
    cufftHandle fl, il;
    PS_TRY(get_plan(c, (int)f.L, nr, f.Lf, g.cdouble, 0, &fl));
    PS_TRY(get_plan(c, (int)f.L, nr, f.L, g.cdouble, 1, &il));
    PS_CUFFT(cufftSetStream(fl, st));
    PS_CUFFT(cufftSetStream(il, st));
    if (odd) {  // odd L: rows scaled by powers of two around the paired R2C (see hilbert_chunk)
      PS_TRY(ensure(c->hscale, (size_t)nr * es));
      PS_CUDA(launch_scale_rows(c->xw.p, nr, f.L, f.Lf, c->hscale.p, 0, dbl, st));
    }
    PS_CUFFT(r2c(fl, c->xw.p));
    PS_CUDA(launch_hilbert_spectrum(c->spec.p, nr, (int)f.L, dbl, st));
    PS_CUFFT(c2r(il, c->hbuf.p));
    if (odd) PS_CUDA(launch_scale_rows(c->xw.p, nr, f.L, f.Lf, c->hscale.p, 1, dbl, st));
    c->launches += odd ? 3 : 1;
  }
  SrcDesc s = src;
  s.ptr = static_cast<const char*>(c->xw.p) + (f.P - row0 * f.Lf) * (long long)es;
  s.kind = 0;
  s.is_double = dbl;
  s.s_sig = f.Lf;
  s.s_samp = 1;
  s.s_trial = g.N * f.Lf;
  s.s_band = g.R * g.N * f.Lf;
  s.hbuf = static_cast<const char*>(c->hbuf.p) + f.P * (long long)es;
  s.h_row0 = row0;
  s.h_ld = f.L;
  s.h_scale = (hilbert && odd) ? c->hscale.p : nullptr;
  *fs = s;
  return PS_OK;
}

// PS_HILBERT=cufft forces the cuFFT chain where the fused kernel applies
bool hilbert_fused_enabled() {
  static const bool on = [] {
    const char* s = std::getenv("PS_HILBERT");
    return !(s && std::string(s) == "cufft");
  }();
  return on;
}

ps_status reset_status(ps_ctx* c, cudaStream_t st) {
  PS_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(DevStatus), st));
  return PS_OK;
}

// Re-read the device status after the FP64 refinement (its kernels add to
// the indeterminate-ciPLV count); the flags were checked before it ran.
ps_status refresh_status(ps_ctx* c, cudaStream_t st) {
  PS_CUDA(cudaMemcpyAsync(c->h_status, c->d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
  PS_CUDA(cudaStreamSynchronize(st));
  return PS_OK;
}

ps_status read_status(ps_ctx* c, cudaStream_t st) {
  PS_CUDA(cudaMemcpyAsync(c->h_status, c->d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
  PS_CUDA(cudaStreamSynchronize(st));
  const int f = c->h_status->flags;
  if (f & FLAG_TIMEOUT) return fail(PS_E_INTERNAL, "device pipeline timeout");
  if (f & FLAG_NONFINITE) return fail(PS_E_INVALID, "input contains non-finite values (SPEC.md:32)");
  if (f & FLAG_ALL_MASKED)
    return fail(PS_E_ALL_MASKED, "every sample of some signal/trial fell below the amplitude floor");
  if (f & FLAG_EMPTY_WINDOW) return fail(PS_E_EMPTY_WINDOW, "all samples are masked for at least one signal pair");
  return PS_OK;
}

// Per-call row state: amplitude min/max (order-preserving bits) and masked
// counts.  Must run (stream-ordered) before any prepare_rows of the call.
ps_status init_row_state(ps_ctx* c, const Geometry& g, cudaStream_t st) {
  PS_TRY(ensure(c->rowstat, (size_t)g.rows * 2 * sizeof(unsigned long long)));
  PS_TRY(ensure(c->maskcount, (size_t)g.rows * sizeof(int)));
  unsigned long long* rs = static_cast<unsigned long long*>(c->rowstat.p);
  PS_CUDA(cudaMemsetAsync(rs, 0xFF, (size_t)g.rows * sizeof(unsigned long long), st));
  PS_CUDA(cudaMemsetAsync(rs + g.rows, 0, (size_t)g.rows * sizeof(unsigned long long), st));
  return PS_OK;
}

// Normalisation of rows [row_lo, row_hi) into `out` (fmt 0/1: planes, fmt 2:
// dense complex rows relative to `out`).  Real input goes through the cuFFT
// Hilbert stage in bounded row chunks first.
ps_status prepare_rows(ps_ctx* c, const ps_plv_args* a, const Geometry& g, const void* in_ptr, void* out, int fmt,
                       long long pitch, long long plane_stride, long long row_lo, long long row_hi, cudaStream_t st,
                       bool* copied) {
  unsigned long long* rs = static_cast<unsigned long long*>(c->rowstat.p);
  SrcDesc src = make_src(a, g, in_ptr);
  const size_t ces = g.cdouble ? 8 : 4;
  auto out_at = [&](long long row0) -> void* {
    if (fmt != 2) return out;
    return static_cast<char*>(out) + (size_t)row0 * g.T * 2 * ces;
  };
  const long long rc = a->input_kind == PS_INPUT_REAL ? prep_chunk_rows(a, g) : (row_hi - row_lo);
  const bool bandpass = a->input_kind == PS_INPUT_REAL && a->fir;
  // Gauss Gram: the vectorised normaliser writes the S / D planes in the same
  // pass; any chunk that took another route gets them from gauss_planes_kernel
  const bool want_gauss = g.gauss && fmt == 0 && !gauss_smem_convert();
  src.gauss_planes = want_gauss ? 1 : 0;
  bool gauss_all = true;
  const bool fused = a->input_kind == PS_INPUT_REAL && !bandpass && hilbert_fused_enabled() &&
                     hilbert_fused_supported(src, fmt, g.cdouble ? 1 : 0, (int)pitch);
  for (long long row0 = row_lo; row0 < row_hi; row0 += rc) {
    const long long nr = std::min(rc, row_hi - row0);
    if (bandpass) {  // Hf was computed by prep_begin for this call
      SrcDesc fs;
      PS_TRY(bandpass_chunk(c, a, g, src, row0, nr, true, st, &fs));
      int gd = 0;
      PS_CUDA(launch_normalize_fmt(fs, row0, nr, out_at(row0), fmt, g.cdouble, (int)pitch, plane_stride, rs, g.rows,
                                   c->d_status, st, &gd));
      gauss_all = gauss_all && gd;
      PS_CUDA(launch_fixup_fmt(fs, row0, nr, out_at(row0), fmt, g.cdouble, (int)pitch, plane_stride, rs, g.rows,
                               static_cast<int*>(c->maskcount.p), a->amp_floor, c->d_status, st));
      c->launches += 2;
      continue;
    }
    if (fused) {
      // one kernel: FFT -> multiplier -> IFFT -> normalise; H is kept (in
      // hbuf) only for rows the exact-median fixup will inspect
      PS_TRY(ensure(c->hbuf, (size_t)nr * g.T * sizeof(float)));
      src.hbuf = c->hbuf.p;
      src.h_row0 = row0;
      int gd = 0;
      PS_CUDA(launch_hilbert_fused(src, row0, nr, out, (int)pitch, plane_stride, rs, g.rows, a->amp_floor,
                                   c->d_status, st, &gd));
      gauss_all = gauss_all && gd;
      PS_CUDA(launch_fixup_fmt(src, row0, nr, out, fmt, 0, (int)pitch, plane_stride, rs, g.rows,
                               static_cast<int*>(c->maskcount.p), a->amp_floor, c->d_status, st));
      c->launches += 2;
      continue;
    }
    if (a->input_kind == PS_INPUT_REAL) {
      PS_TRY(hilbert_chunk(c, a, g, src, row0, nr, st, copied, &src.h_scale));
      src.hbuf = c->hbuf.p;
      src.h_row0 = row0;
    }
    int gd = 0;
    PS_CUDA(launch_normalize_fmt(src, row0, nr, out_at(row0), fmt, g.cdouble, (int)pitch, plane_stride, rs, g.rows,
                                 c->d_status, st, &gd));
    gauss_all = gauss_all && gd;
    PS_CUDA(launch_fixup_fmt(src, row0, nr, out_at(row0), fmt, g.cdouble, (int)pitch, plane_stride, rs, g.rows,
                             static_cast<int*>(c->maskcount.p), a->amp_floor, c->d_status, st));
    c->launches += 2;
  }
  if (want_gauss && !gauss_all) {  // S = Zr + Zi, D = Zr - Zi planes of the Gauss Gram (after any masking)
    PS_CUDA(launch_gauss_planes(out, plane_stride, row_lo * pitch, row_hi * pitch, st));
    c->launches++;
  }
  return PS_OK;
}

// Normalisation of all rows.
ps_status prepare_phasors(ps_ctx* c, const ps_plv_args* a, const Geometry& g, const void* in_ptr, void* out,
                          int fmt, long long pitch, long long plane_stride, cudaStream_t st, bool* copied) {
  PS_TRY(init_row_state(c, g, st));
  PS_TRY(prep_begin(c, a, g, st));
  return prepare_rows(c, a, g, in_ptr, out, fmt, pitch, plane_stride, 0, g.rows, st, copied);
}

// Upper-triangle tile list (tiles that contain at least one pair i <= j).
void build_tiles(long long N, int bm, int bn, std::vector<std::pair<int, int>>& tiles) {
  tiles.clear();
  const int nj = (int)((N + bn - 1) / bn), ni = (int)((N + bm - 1) / bm);
  for (int J = 0; J < nj; ++J) {
    const long long jmax = std::min<long long>((long long)J * bn + bn, N) - 1;
    for (int I = 0; I < ni; ++I)
      if ((long long)I * bm <= jmax) tiles.emplace_back(I, J);
  }
}

int choose_groups(long long items_per_group, int R, int num_slots, size_t ws_bytes_per_group, size_t ws_budget) {
  // Trial groups: items = tiles x bands x G, each running Rg = ceil(R / G)
  // trials back to back.  Time ~ waves(items) x Rg.  Rounds after the first
  // of a group read-modify-write the partial sums (measured ~25% slower per
  // round on C4), so among near-optimal choices prefer the most groups whose
  // partial-sum workspace fits the budget.
  auto cost = [&](int G, int Rg) {
    const long long items = items_per_group * G;
    const long long waves = (items + num_slots - 1) / num_slots;
    return (double)waves * (1.0 + 1.25 * (Rg - 1));  // first round of an item 1, RMW rounds 1.25
  };
  int best_g = 1;
  double best = cost(1, R);
  for (int G = 2; G <= R; ++G) {
    const int Rg = (R + G - 1) / G;
    if ((R + Rg - 1) / Rg != G) continue;
    if ((size_t)G * ws_bytes_per_group > ws_budget) break;
    const double c = cost(G, Rg);
    if (c <= best * 1.02) {
      best = std::min(best, c);
      best_g = G;
    }
  }
  return best_g;
}

}  // namespace

template <typename S>
__global__ void mask_from_zero_kernel(const S* z, size_t n, uint8_t* m) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    m[e] = (z[2 * e] == S(0) && z[2 * e + 1] == S(0)) ? 1 : 0;
}

static cudaError_t ps_mask_from_zero(const void* z, int is_double, size_t n, uint8_t* m, cudaStream_t st) {
  const int grid = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
  if (is_double) mask_from_zero_kernel<double><<<grid, 256, 0, st>>>((const double*)z, n, m);
  else mask_from_zero_kernel<float><<<grid, 256, 0, st>>>((const float*)z, n, m);
  return cudaGetLastError();
}

namespace {

// Everything one ps_plv_family call needs after validation: work items (by
// stage), kernel parameters, TMA descriptors, output routing.
struct Call {
  Geometry g;
  void* outs[5] = {};   // final device outputs (nullptr = metric not requested)
  int shard_count = 1, shard_index = 0;
  bool pool = false;
  int G = 1, slot_mode = 1, mean_div = 1, Rg = 1;
  // divisor of the trial-group reduction: R (trial mean) or 1 (PS_TRIALS_SUM)
  int reduce_div = 1;
  bool trial_sum = false;
  std::vector<int> stage_off;  // item offsets of the stages (size n_stages + 1)
  GramParams p;
  const CUtensorMap* ta = nullptr;
  const CUtensorMap* tb = nullptr;
  const CUtensorMap* tb2 = nullptr;
  long long nn = 0;
  size_t oes = 4;
  long long slots = 1;  // output slots per metric
  std::vector<std::pair<int, int>> mine;  // ownership tiles of this call (plan_call)
};

// The 3-product (Gauss) split Gram: 9 UMMAs per K step instead of 12
// (gram_tc.cu), same 256 x 128 tiles, one accumulation buffer.  It pays where
// the Gram dominates and rounds are long: complex (analytic / phasor) input
// with >= 8192 samples per round (C5: Gram -7%, step -5%); with real input
// or short trials the extra S / D plane pass outweighs it (measured C2-C4).
// PS_GAUSS=1 forces it for every split over-samples call, PS_GAUSS=0 never.
int gauss_mode() {
  static const int m = [] {
    const char* s = std::getenv("PS_GAUSS");
    return s ? (std::atoi(s) != 0 ? 1 : 0) : -1;  // -1: automatic
  }();
  return m;
}

void decide_gauss(const ps_plv_args* a, Call& k) {
  const bool eligible = k.g.split && a->mode == PS_MODE_OVER_SAMPLES;
  const long long round_len = a->trial_reduce == PS_TRIALS_POOL ? k.g.T * k.g.R : k.g.T;
  // complex input: rounds >= 8192 samples (C5).  Real input, whose S / D
  // planes now come out of the normaliser at 8 B / sample more writes: where
  // the Gram dominates the normalisation by enough -- N >= 2048 signals and
  // rounds >= 8192 (C3: step 17.7 -> 16.7 ms; C2, N = 1200: 6.3 -> 6.5 ms, not
  // taken; profiles/r02_gauss_real_input.txt)
  const bool automatic =
      round_len >= 8192 && (a->input_kind != PS_INPUT_REAL || (k.g.N >= 2048 && !a->fir));
  const int m = gauss_mode();
  k.g.gauss = eligible && (m == 1 || (m == -1 && automatic));
}

int kc_blocks_default() {
  // TMEM accumulation chunk (drain period) in 32-sample K blocks; see gram_tc.cu
  static const int kcb = [] {
    const char* s = std::getenv("PS_KC_BLOCKS");
    return s ? std::max(1, std::atoi(s)) : 4;
  }();
  return kcb;
}

// Supertile of the item raster order within a stage: SI row panels x SJ
// column panels, and the order inside it (0: J-major, 1: I-major).  The 74
// items in flight at a time share their operand panels through L2; what a
// wave fetches from DRAM is (rows of its A panels + rows of its B panels) x
// T, so the raster shapes a wave to cover few 256-row A panels and more
// 128-row B panels.  PS_RASTER="SI[,SJ[,order]]" (experiments).
struct Raster {
  int si = 12, sj = 12, order = 0;
};
// Defaults per Gram variant: the Gauss Gram streams 8 planes (16 B per row
// sample), so a wave's DRAM traffic is twice the 4-product's: it takes 8 row
// panels x 12 column panels, I-major (a wave of 74 items spans ~6 A panels and
// ~12 B panels; C5 Gram 53.1 -> 50.2 ms), the 4-product keeps the square
// 12 x 12 J-major raster (C3 13.7 ms against 14.7 with the Gauss shape;
// profiles/r02_raster_lockstep.txt, r02_sweep_variants.txt)
Raster raster_shape(bool gauss) {
  static const bool has_env = std::getenv("PS_RASTER") != nullptr;
  if (!has_env) {
    Raster d;
    if (gauss) {
      d.si = 8;
      d.sj = 12;
      d.order = 1;
    }
    return d;
  }
  static const Raster r = [] {
    Raster x;
    const char* s = std::getenv("PS_RASTER");
    if (s) {
      x.si = x.sj = std::max(1, std::atoi(s));
      const char* c = std::strchr(s, ',');
      if (c) {
        x.sj = std::max(1, std::atoi(c + 1));
        c = std::strchr(c + 1, ',');
        if (c) x.order = std::atoi(c + 1) != 0 ? 1 : 0;
      }
    }
    return x;
  }();
  return r;
}
int raster_tiles() { return raster_shape(false).si; }

// Row panels per streamed output band in the final row stage.
int row_band_last(int row_band) {
  static const int v = [] {
    const char* s = std::getenv("PS_SB_BAND_LAST");
    return s ? std::max(1, std::atoi(s)) : 0;
  }();
  // never wider than an ownership band (a sharded call owns whole bands)
  return v > 0 ? std::min(v, std::max(1, row_band)) : std::max(1, row_band / 2);
}

// Work items, grouped by stage: stage s holds the tiles whose column panel
// starts in [cols[s], cols[s+1]) (one stage covering everything when `cols` is
// empty).  Ownership (sharding) uses the canonical J-major tile enumeration
// of ps_pair_shard -- except on the streamed host path (row stages), which
// deals whole row bands; within a stage items run in 12 x 12 supertile raster
// order (column stages) or band by band (row stages).
ps_status plan_call(ps_ctx* c, const ps_plv_args* a, Call& k, const std::vector<long long>& cols, bool force_g1,
                    cudaStream_t st, int row_band = 0) {
  const Geometry& g = k.g;
  const int bm = g.split ? kSplitBM : kF64BM;
  const int bn = g.split ? kSplitBN : kF64BN;
  std::vector<std::pair<int, int>> tiles;
  build_tiles(g.N, bm, bn, tiles);
  std::vector<std::pair<int, int>> mine;
  if (row_band > 0 && k.shard_count > 1) {
    // streamed host path, sharded: whole row bands per shard (so each shard
    // ships long contiguous rows), dealt largest-work-first to the least
    // loaded shard (band work ~ rows x (N - i)); deterministic for every shard
    const long long band_rows = (long long)row_band * bm;
    const int n_bands = (int)((g.N + band_rows - 1) / band_rows);
    std::vector<std::pair<long long, int>> work(n_bands);
    for (int b = 0; b < n_bands; ++b) {
      const long long r0 = b * band_rows, r1 = std::min<long long>(r0 + band_rows, g.N);
      work[b] = {(r1 - r0) * (g.N - (r0 + r1) / 2), b};
    }
    std::stable_sort(work.begin(), work.end(),
                     [](const std::pair<long long, int>& x, const std::pair<long long, int>& y) { return x.first > y.first; });
    std::vector<long long> load(k.shard_count, 0);
    std::vector<int> owner(n_bands, 0);
    for (const auto& wb : work) {
      const int r = (int)(std::min_element(load.begin(), load.end()) - load.begin());
      owner[wb.second] = r;
      load[r] += wb.first;
    }
    for (const auto& t : tiles)
      if (owner[(int)(((long long)t.first * bm) / band_rows)] == k.shard_index) mine.push_back(t);
  } else {
    for (size_t t = 0; t < tiles.size(); ++t)
      if ((int)(t % k.shard_count) == k.shard_index) mine.push_back(tiles[t]);
  }
  k.mine = mine;
  const int n_stages = cols.empty() ? 1 : (int)cols.size() - 1;
  // Column stages (row_band == 0): stage s holds the tiles whose column panel
  // starts in [cols[s], cols[s+1]).  Row stages (row_band > 0, the streamed
  // copy-out of the upper layout): stage s holds the tiles whose row panel
  // starts in [cols[n-1-s], cols[n-s]) -- the last signals come first, and a
  // finished row band is final over the whole upper part of its rows.
  auto stage_of = [&](const std::pair<int, int>& t) -> int {
    if (cols.empty()) return 0;
    const long long x0 = row_band > 0 ? (long long)t.first * bm : (long long)t.second * bn;
    int s = 0;
    while (s + 1 < n_stages && x0 >= cols[s + 1]) ++s;
    return row_band > 0 ? n_stages - 1 - s : s;
  };
  const int S = row_band > 0 ? row_band : raster_tiles();
  // row stages: the final stage uses bands of half the size (its last band's
  // Gram + copy-out is the tail of the call)
  auto band_of = [&](int stage) { return stage == n_stages - 1 ? row_band_last(row_band) : S; };
  // row stages: bands of S row panels, J-major within a band (a finished band
  // is one output block of full upper rows); the in-flight window (~74
  // consecutive items: ~74/S column panels x S row panels) stays L2-sized.
  // Column stages: S x S supertile raster.
  const Raster rs = raster_shape(g.gauss);
  std::stable_sort(mine.begin(), mine.end(), [&](const std::pair<int, int>& x, const std::pair<int, int>& y) {
    const int sx = stage_of(x), sy = stage_of(y);
    if (row_band > 0) {
      const int bx = band_of(sx), by = band_of(sy);
      return std::make_tuple(sx, x.first / bx, x.second, x.first) < std::make_tuple(sy, y.first / by, y.second, y.first);
    }
    const int ix = rs.order ? x.first : x.second, jx = rs.order ? x.second : x.first;
    const int iy = rs.order ? y.first : y.second, jy = rs.order ? y.second : y.first;
    return std::make_tuple(sx, x.second / rs.sj, x.first / rs.si, ix, jx) <
           std::make_tuple(sy, y.second / rs.sj, y.first / rs.si, iy, jy);
  });
  k.pool = a->trial_reduce == PS_TRIALS_POOL;
  if (k.pool || g.R == 1) {
    k.G = 1;
    k.slot_mode = 1;
  } else if (a->trial_reduce == PS_TRIALS_NONE) {
    k.G = (int)g.R;
    k.slot_mode = 0;
  } else {
    // concurrent work slots = CTA groups (pairs for the cta_group::2 kernel);
    // items per group = tiles in 128-row halves for the single-CTA variant
    const int slots = c->num_sms / (g.split ? split_cta_group() : 1);
    const long long per_group = (long long)mine.size() * g.B * (g.split ? kSplitBM / split_panel_rows() : 1);
    // partial-sum workspace budget from the device's total memory (fixed per
    // device: the trial-group choice -- and with it the summation order --
    // does not depend on what else happens to be allocated, and no
    // cudaMemGetInfo on the call path: it can stall for tens of ms while
    // another process queries the driver, e.g. nvidia-smi)
    const size_t ws_per_group = (size_t)g.B * g.N * g.N * (g.split ? 4 : 8) * 5;  // worst case: 5 metrics
    const size_t ws_budget = std::min<size_t>(c->total_mem / 6, (size_t)24 << 30);
    k.G = (k.shard_count > 1 || force_g1) ? 1 : choose_groups(per_group, (int)g.R, slots, ws_per_group, ws_budget);
    static const int g_env = [] {
      const char* s = std::getenv("PS_GROUPS");  // experiment override
      return s ? std::atoi(s) : 0;
    }();
    if (g_env > 0 && k.shard_count == 1 && !force_g1) k.G = std::min<int>(g_env, (int)g.R);
    k.slot_mode = k.G == 1 ? 1 : 2;
    k.trial_sum = a->trial_reduce == PS_TRIALS_SUM;
    k.mean_div = (k.G == 1 && !k.trial_sum) ? (int)g.R : 1;
    k.reduce_div = k.trial_sum ? 1 : (int)g.R;
  }
  k.Rg = (int)((g.R + k.G - 1) / k.G);
  k.slots = (a->trial_reduce == PS_TRIALS_NONE && !k.pool) ? g.B * g.R : g.B;
  // Split path: ownership tiles are 256 x 128; the single-CTA variant runs
  // each as two 128-row halves (halves wholly below the diagonal dropped).
  const int exec_rows = g.split ? split_panel_rows() : kF64BM;
  const int sub = g.split ? kSplitBM / exec_rows : 1;
  std::vector<Item>& items = c->h_items;
  items.clear();
  k.stage_off.assign(1, 0);
  size_t t0 = 0;
  for (int s = 0; s < n_stages; ++s) {
    size_t t1 = t0;
    while (t1 < mine.size() && stage_of(mine[t1]) == s) ++t1;
    for (int b = 0; b < g.B; ++b)
      for (int gi = 0; gi < k.G; ++gi)
        for (size_t t = t0; t < t1; ++t)
          for (int hs = 0; hs < sub; ++hs) {
            const int I = mine[t].first * sub + hs;
            const long long jmax = std::min<long long>((long long)mine[t].second * bn + bn, g.N) - 1;
            if ((long long)I * exec_rows > jmax || (long long)I * exec_rows >= g.N) continue;
            items.push_back(Item{b, gi, I, mine[t].second});
          }
    k.stage_off.push_back((int)items.size());
    t0 = t1;
  }
  const size_t ibytes = std::max<size_t>(items.size(), 1) * sizeof(Item);
  if (c->h_items_cap < ibytes) {
    if (c->h_items_pinned) cudaFreeHost(c->h_items_pinned);
    c->h_items_pinned = nullptr;
    c->h_items_cap = 0;
    PS_CUDA(cudaMallocHost(&c->h_items_pinned, ibytes));
    c->h_items_cap = ibytes;
  }
  // calls are synchronous: the previous call finished with the pinned staging
  if (!items.empty()) std::memcpy(c->h_items_pinned, items.data(), items.size() * sizeof(Item));
  PS_TRY(ensure(c->items, ibytes));
  if (!items.empty())
    PS_CUDA(cudaMemcpyAsync(c->items.p, c->h_items_pinned, items.size() * sizeof(Item), cudaMemcpyHostToDevice, st));

  GramParams& p = k.p;
  std::memset(&p, 0, sizeof(p));
  p.N = (int)g.N;
  p.T = (int)g.T;
  p.R = (int)g.R;
  p.B = (int)g.B;
  p.Tp = (int)g.pitch;
  p.rows = (int)g.rows;
  p.Rg = k.Rg;
  p.G = k.G;
  p.pool = k.pool ? 1 : 0;
  p.items = static_cast<const Item*>(c->items.p);
  p.slot_mode = k.slot_mode;
  p.mean_div = k.mean_div;
  p.maskcount = static_cast<const int*>(c->maskcount.p);
  p.planes = c->planes.p;
  p.plane_stride = g.plane_stride;
  p.status = c->d_status;
  p.illcond_tol = 4e-6f;  // 2.5x margin below the 1e-5 split-path tolerance
  // the Gauss Gram drains a single accumulation buffer: longer chunks (its
  // error at 512 samples matches the 4-product Gram's at 128, accuracy probe)
  // PS_KC_BLOCKS (experiments) is capped at the longest chunk whose measured
  // error stays inside the 1e-5 split budget (profiles/r01_accuracy_probe_kc,
  // r02_accuracy_probe_gauss_kc: 4-product kc 4 = 128 samples, Gauss kc 16 =
  // 512 samples); PS_KC_UNSAFE=1 lifts the cap for accuracy probes only
  {
    const int kc_max = g.gauss ? 16 : 4;
    static const bool unsafe = std::getenv("PS_KC_UNSAFE") != nullptr;
    const int want = std::getenv("PS_KC_BLOCKS") ? kc_blocks_default() : kc_max;
    p.kc_blocks = unsafe ? want : std::min(want, kc_max);
  }
  p.upper_only = a->out_layout == PS_LAYOUT_UPPER ? 1 : 0;
  // trial-group partial sums are written as upper triangles; the group reduce
  // produces the mirror (half the slot stores and reduce reads)
  p.slot_upper = (p.upper_only || k.slot_mode == 2) ? 1 : 0;
  static const int dbg = [] {
    const char* s = std::getenv("PS_DEBUG_EPI");
    return s ? std::atoi(s) : 0;
  }();
  p.debug_flags = dbg;
  if (g.split && k.outs[2]) {
    const int cap = 1 << 22;  // queued ill-conditioned ciPLV (pair, round) entries
    PS_TRY(ensure(c->refine, (size_t)cap * sizeof(RefineEntry)));
    p.refine = static_cast<RefineEntry*>(c->refine.p);
    p.refine_cap = cap;
  }
  k.oes = g.split ? 4 : 8;
  k.nn = g.N * g.N;
  void* kouts[5];
  std::memcpy(kouts, k.outs, sizeof(kouts));
  if (k.slot_mode == 2) {
    // trial-group partial sums, reduced in a fixed order afterwards
    const size_t per = (size_t)g.B * k.G * k.nn * k.oes;
    PS_TRY(ensure(c->gws, per * 5));
    for (int m = 0; m < 5; ++m) kouts[m] = kouts[m] ? static_cast<char*>(c->gws.p) + m * per : nullptr;
  }
  p.out_plv = kouts[0];
  p.out_iplv = kouts[1];
  p.out_ciplv = kouts[2];
  p.out_cre = kouts[3];
  p.out_cim = kouts[4];
  if (g.split) {
    TmapKey key{c->planes.p, g.T, g.N, g.B * g.R, g.pitch, g.gauss};
    auto it = c->tmaps.find(key);
    if (it == c->tmaps.end()) {
      auto enc = encode_fn();
      if (!enc) return fail(PS_E_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
      Tmaps tm{};
      cuuint64_t dims[4] = {(cuuint64_t)g.T, (cuuint64_t)g.N, (cuuint64_t)(g.B * g.R), (cuuint64_t)g.nplanes()};
      cuuint64_t strides[3] = {(cuuint64_t)g.pitch * 2, (cuuint64_t)(g.N * g.pitch * 2),
                               (cuuint64_t)(g.plane_stride * 2)};
      // boxes: A = 128 rows x {4 planes | Gauss: 6 planes Zr, Zi, S}; B = the
      // CTA's share of the J panel x {4 planes | Gauss: 2 planes Zr (+ b2: S, D)}
      const cuuint32_t brows = (cuuint32_t)split_b_box_rows();
      // (Gauss with the smem S / D conversion streams the 4-plane boxes)
      const bool gs_planes = g.gauss && !gauss_smem_convert();
      cuuint32_t boxA[4] = {(cuuint32_t)kSplitBK, 128u, 1, gs_planes ? 6u : 4u};
      cuuint32_t boxB[4] = {(cuuint32_t)kSplitBK, brows, 1, gs_planes ? 2u : 4u};
      cuuint32_t boxB2[4] = {(cuuint32_t)kSplitBK, brows, 1, 4u};
      cuuint32_t estr[4] = {1, 1, 1, 1};
      const CUtensorMapSwizzle swz = kSplitBK == 16   ? CU_TENSOR_MAP_SWIZZLE_32B
                                     : kSplitBK == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                      : CU_TENSOR_MAP_SWIZZLE_128B;
      auto encode = [&](CUtensorMap* m, cuuint32_t* box) {
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, c->planes.p, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      };
      const CUresult r1 = encode(&tm.a, boxA), r2 = encode(&tm.b, boxB);
      const CUresult r3 = gs_planes ? encode(&tm.b2, boxB2) : CUDA_SUCCESS;
      if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS || r3 != CUDA_SUCCESS)
        return fail(PS_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r1) + "/" +
                                   std::to_string((int)r2) + "/" + std::to_string((int)r3));
      if (c->tmaps.size() > 64) c->tmaps.clear();
      it = c->tmaps.emplace(key, tm).first;
    }
    k.ta = &it->second.a;
    k.tb = &it->second.b;
    k.tb2 = g.gauss && !gauss_smem_convert() ? &it->second.b2 : nullptr;
  }
  return PS_OK;
}

// K7 mask-count Gram (SPEC.md:260 per-pair effective T): when the
// normalisation masked any sample, T_ij = sum_t u_i(t) u_j(t) for every pair
// of the call's tiles comes from one tcgen05 product of the 0/1 indicator
// planes (gram_tc.cu, MK variant) -- exact -- and the metric epilogues read it
// (interior fast path kept) instead of scanning both rows' planes.  Runs after
// plan_call, before the Gram; the host reads the mask flag first (one short
// synchronisation; the pipelined host paths keep the plane scan).
ps_status mask_count_pass(ps_ctx* c, Call& k, cudaStream_t st) {
  const Geometry& g = k.g;
  const long long ip = round_up(g.T, 16);  // E4M3 bytes, 16-byte rows for TMA
  PS_TRY(ensure(c->ind, (size_t)g.rows * ip));
  PS_CUDA(launch_indicator_plane(c->planes.p, g.plane_stride, g.split ? 1 : 0, g.rows, (int)g.pitch, (int)g.T,
                                 c->ind.p, (int)ip, st));
  c->launches++;
  const long long cslots = k.pool ? g.B : g.B * g.R;
  PS_TRY(ensure(c->cntws, (size_t)cslots * g.N * g.N * sizeof(int)));
  // count tiles: the split geometry's ownership tiles (fp64 calls: all of them)
  std::vector<std::pair<int, int>> tiles;
  if (g.split) tiles = k.mine;
  else build_tiles(g.N, kSplitBM, kSplitBN, tiles);
  const int exec_rows = split_panel_rows();
  const int sub = kSplitBM / exec_rows;
  const int units = k.pool ? 1 : (int)g.R;
  std::vector<Item> items;
  for (int b = 0; b < g.B; ++b)
    for (int gi = 0; gi < units; ++gi)
      for (const auto& t : tiles)
        for (int hs = 0; hs < sub; ++hs) {
          const int I = t.first * sub + hs;
          const long long jmax = std::min<long long>((long long)t.second * kSplitBN + kSplitBN, g.N) - 1;
          if ((long long)I * exec_rows > jmax || (long long)I * exec_rows >= g.N) continue;
          items.push_back(Item{b, gi, I, t.second});
        }
  if (items.empty()) return PS_OK;
  PS_TRY(ensure(c->cntitems, items.size() * sizeof(Item)));
  // pageable source: staged before the call returns
  PS_CUDA(cudaMemcpyAsync(c->cntitems.p, items.data(), items.size() * sizeof(Item), cudaMemcpyHostToDevice, st));
  GramParams pc;
  std::memset(&pc, 0, sizeof(pc));
  pc.N = (int)g.N;
  pc.T = (int)g.T;
  pc.R = (int)g.R;
  pc.B = (int)g.B;
  pc.Tp = (int)ip;
  pc.rows = (int)g.rows;
  pc.Rg = 1;
  pc.G = units;
  pc.pool = k.pool ? 1 : 0;
  pc.items = static_cast<const Item*>(c->cntitems.p);
  pc.n_items = (int)items.size();
  pc.status = c->d_status;
  pc.kc_blocks = 16;  // 16 x 128-sample stages per drain (exact for integer counts)
  pc.cnt = static_cast<int*>(c->cntws.p);
  auto enc = encode_fn();
  if (!enc) return fail(PS_E_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  CUtensorMap ta, tb;
  cuuint64_t dims[4] = {(cuuint64_t)g.T, (cuuint64_t)g.N, (cuuint64_t)(g.B * g.R), 1};
  cuuint64_t strides[3] = {(cuuint64_t)ip, (cuuint64_t)(g.N * ip), (cuuint64_t)(g.rows * ip)};
  // 128 one-byte samples per stage row: the 128B swizzle of the MK kernel
  cuuint32_t boxA[4] = {(cuuint32_t)(4 * kSplitBK), 128u, 1, 1};
  cuuint32_t boxB[4] = {(cuuint32_t)(4 * kSplitBK), (cuuint32_t)split_b_box_rows(), 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  static_assert(kSplitBK == 32, "the fp8 count operand rows are 128 bytes (4 x kSplitBK samples)");
  const CUresult r1 = enc(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, c->ind.p, dims, strides, boxA, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const CUresult r2 = enc(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, c->ind.p, dims, strides, boxB, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS)
    return fail(PS_E_CUDA, "cuTensorMapEncodeTiled (indicator plane) failed");
  const int grid = std::min(pc.n_items, c->num_sms / split_cta_group());
  PS_CUDA(launch_gram_count(&ta, &tb, pc, grid, st));
  c->launches++;
  k.p.cnt = pc.cnt;
  return PS_OK;
}

// Did the normalisation mask any sample?  (reads the device flag; syncs `st`)
ps_status any_masked(ps_ctx* c, cudaStream_t st, bool* out) {
  PS_CUDA(cudaMemcpyAsync(c->h_status, c->d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
  PS_CUDA(cudaStreamSynchronize(st));
  *out = (c->h_status->flags & FLAG_ANY_MASKED) != 0;
  return PS_OK;
}

static bool k7_enabled() {
  static const bool on = std::getenv("PS_NO_K7") == nullptr;  // PS_NO_K7=1: plane scan (A/B experiments)
  return on;
}

ps_status launch_stage(ps_ctx* c, Call& k, int s, cudaStream_t st) {
  GramParams p = k.p;
  const int i0 = k.stage_off[s], i1 = k.stage_off[s + 1];
  p.items = k.p.items + i0;
  if (p.item_sb) p.item_sb += i0;
  p.n_items = i1 - i0;
  if (p.n_items <= 0) return PS_OK;
  const int cta_per_group = k.g.split ? split_cta_group() : 1;
  const int grid = std::min(p.n_items, c->num_sms / cta_per_group);
  // producer lockstep (GramParams::lock_cnt): needs the same number of K
  // blocks in every item; PS_LOCKSTEP="group,lag" in K blocks ("0" = off)
  // (group, lag) in K blocks: the Gauss Gram's 8-plane working set takes the
  // tighter window (16, 2); the 4-product (32, 2) (profiles/r02_raster_lockstep.txt)
  static const std::pair<int, int> lk_env = [] {
    const char* s = std::getenv("PS_LOCKSTEP");
    int g = -1, l = 2;
    if (s) {
      g = std::atoi(s);
      const char* comma = std::strchr(s, ',');
      if (comma) l = std::max(1, std::atoi(comma + 1));
    }
    return std::make_pair(g, l);
  }();
  const std::pair<int, int> lk = lk_env.first >= 0 ? lk_env : std::make_pair(k.g.gauss ? 16 : 32, 2);
  p.lock_cnt = nullptr;
  const bool uniform = k.pool || (k.g.R % k.Rg) == 0;
  if (k.g.split && lk.first > 0 && uniform) {
    const long long rounds = k.pool ? k.g.R : k.Rg;
    const long long nk = (k.g.T + kSplitBK - 1) / kSplitBK;
    const long long per_cta = (long long)((p.n_items + grid - 1) / grid) * rounds * nk;
    const long long ngroups = per_cta / lk.first + 2;
    // sized generously once: a reallocation would synchronise the device and
    // break the overlap of the pipelined host path's stages
    PS_TRY(ensure(c->lockbuf, (size_t)std::max<long long>(ngroups, 1 << 16) * sizeof(int)));
    PS_CUDA(cudaMemsetAsync(c->lockbuf.p, 0, (size_t)ngroups * sizeof(int), st));
    p.lock_cnt = static_cast<int*>(c->lockbuf.p);
    p.lock_group = lk.first;
    p.lock_lag = lk.second;
    p.lock_rounds = (int)rounds;
  }
  static const bool prof = std::getenv("PS_GRAM_PROF") != nullptr;  // diagnostics: pipeline wait cycles
  if (prof && k.g.split) {
    PS_TRY(ensure(c->profbuf, 8 * sizeof(unsigned long long)));
    PS_CUDA(cudaMemsetAsync(c->profbuf.p, 0, 8 * sizeof(unsigned long long), st));
    p.prof = static_cast<unsigned long long*>(c->profbuf.p);
  }
  static const int pf = [] {
    const char* e = std::getenv("PS_PREFETCH");  // L2 prefetch distance (K blocks); 0 = off
    return e ? std::max(0, std::atoi(e)) : 0;
  }();
  p.prefetch_blocks = pf;
  if (k.g.split) PS_CUDA(launch_gram_split(k.ta, k.tb, k.tb2, k.g.gauss, p, grid, st));
  else PS_CUDA(launch_gram_f64(p, grid, st));
  c->launches++;
  if (p.prof) {
    unsigned long long h[8];
    PS_CUDA(cudaMemcpyAsync(h, p.prof, sizeof(h), cudaMemcpyDeviceToHost, st));
    PS_CUDA(cudaStreamSynchronize(st));
    const double mt = (double)std::max<unsigned long long>(h[2], 1), pt = (double)std::max<unsigned long long>(h[4], 1);
    std::fprintf(stderr,
                 "[gram-prof] variant %s items %d grid %d: MMA issuer blocked on operands %.1f%%, on TMEM buffers "
                 "%.1f%%; producer blocked on free stages %.1f%%; epilogue warps blocked on accumulators %.1f%%, "
                 "emitting %.1f%%\n",
                 k.g.gauss ? "gauss" : "4prod", p.n_items, grid, 100.0 * h[0] / mt, 100.0 * h[1] / mt,
                 100.0 * h[3] / pt, 100.0 * h[5] / std::max<unsigned long long>(h[7], 1),
                 100.0 * h[6] / std::max<unsigned long long>(h[7], 1));
  }
  return PS_OK;
}

// Exact FP64 refinement of queued ill-conditioned ciPLV entries [lo, hi):
// copied to the host, sorted (deterministic application order), grouped by
// output location and recomputed by refine_kernel on stream `st`.
ps_status refine_range(ps_ctx* c, Call& k, unsigned long long lo, unsigned long long hi, cudaStream_t st) {
  if (hi <= lo || !k.g.split || !k.outs[2]) return PS_OK;
  if (hi > (unsigned long long)k.p.refine_cap)
    return fail(PS_E_UNSUPPORTED,
                "more than " + std::to_string(k.p.refine_cap) + " ill-conditioned ciPLV pair-rounds (" +
                    std::to_string(hi) +
                    "; |Re| within ~1e-3 of 1 for a large share of pairs): the split path cannot meet 1e-5 for "
                    "them cheaply -- use precision='fp64' for this input");
  const bool single_round = k.pool || k.g.R == 1 || k.slot_mode == 0;
  {  // device-side ordering when the packed (slot, i, j) key fits 64 bits
    auto bits = [](long long v) {
      int b = 1;
      while ((1LL << b) < v) ++b;
      return b;
    };
    const int ib = bits(k.g.N), sb = bits(std::max<long long>(k.slots, 2));
    if (sb + 2 * ib <= 64 && hi - lo < (1ULL << 30)) {
      const int n = (int)(hi - lo);
      const size_t ebytes = (size_t)round_up((long long)n * (long long)sizeof(RefineEntry), 256);
      const size_t xbytes = (size_t)round_up((long long)n * 8, 256);
      PS_TRY(ensure(c->refine_sorted, ebytes + xbytes + (size_t)(n + 1) * sizeof(int) + 256));
      const size_t wsb = refine_sort_ws_bytes(n);
      PS_TRY(ensure(c->sortws, wsb));
      RefineEntry* d_ent = static_cast<RefineEntry*>(c->refine_sorted.p);
      double* d_exact = reinterpret_cast<double*>(static_cast<char*>(c->refine_sorted.p) + ebytes);
      int* d_grp = reinterpret_cast<int*>(static_cast<char*>(c->refine_sorted.p) + ebytes + xbytes);
      GramParams pr = k.p;
      pr.out_ciplv = k.outs[2];
      PS_CUDA(launch_refine_sorted(pr, static_cast<RefineEntry*>(c->refine.p) + lo, n, k.slot_mode == 2 ? k.G : 1, ib,
                                   sb + 2 * ib, c->sortws.p, c->sortws.n, d_ent, d_exact, d_grp, single_round ? 1 : 0,
                                   k.trial_sum ? -(int)k.g.R : (int)k.g.R, st));
      c->launches += 8;
      PS_CUDA(cudaStreamSynchronize(st));
      return PS_OK;
    }
  }
  std::vector<RefineEntry> ent(hi - lo);
  PS_CUDA(cudaMemcpyAsync(ent.data(), static_cast<RefineEntry*>(c->refine.p) + lo, ent.size() * sizeof(RefineEntry),
                          cudaMemcpyDeviceToHost, st));
  PS_CUDA(cudaStreamSynchronize(st));
  if (k.slot_mode == 2)
    for (auto& e : ent) e.slot /= k.G;  // workspace slot b*G+g -> final output slot b
  std::sort(ent.begin(), ent.end(), [](const RefineEntry& x, const RefineEntry& y) {
    return std::tie(x.slot, x.i, x.j, x.u0) < std::tie(y.slot, y.i, y.j, y.u0);
  });
  std::vector<int> groups;
  for (size_t q = 0; q < ent.size(); ++q)
    if (q == 0 || ent[q].slot != ent[q - 1].slot || ent[q].i != ent[q - 1].i || ent[q].j != ent[q - 1].j)
      groups.push_back((int)q);
  const int n_groups = (int)groups.size();
  groups.push_back((int)ent.size());
  const size_t ebytes = (size_t)round_up((long long)(ent.size() * sizeof(RefineEntry)), 16);
  const size_t xbytes = ent.size() * sizeof(double);
  PS_TRY(ensure(c->refine_sorted, ebytes + xbytes + groups.size() * sizeof(int) + 64));
  RefineEntry* d_ent = static_cast<RefineEntry*>(c->refine_sorted.p);
  double* d_exact = reinterpret_cast<double*>(static_cast<char*>(c->refine_sorted.p) + ebytes);
  int* d_grp = reinterpret_cast<int*>(static_cast<char*>(c->refine_sorted.p) + ebytes + xbytes);
  PS_CUDA(cudaMemcpyAsync(d_ent, ent.data(), ent.size() * sizeof(RefineEntry), cudaMemcpyHostToDevice, st));
  PS_CUDA(cudaMemcpyAsync(d_grp, groups.data(), groups.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  GramParams pr = k.p;
  pr.out_ciplv = k.outs[2];
  PS_CUDA(launch_refine(pr, d_ent, d_grp, n_groups, (int)ent.size(), d_exact, single_round ? 1 : 0,
                        k.trial_sum ? -(int)k.g.R : (int)k.g.R, st));
  c->launches += 2;
  // host vectors must outlive the async copies
  PS_CUDA(cudaStreamSynchronize(st));
  return PS_OK;
}

ps_status setup_outputs(const ps_plv_args* a, Call& k) {
  if (a->metrics == 0) return fail(PS_E_INVALID, "no metric requested");
  void* outs[5] = {a->out_plv, a->out_iplv, a->out_ciplv, a->out_cre, a->out_cim};
  for (int m = 0; m < 5; ++m) {
    const bool want = (a->metrics >> m) & 1u;
    if (want && !outs[m]) return fail(PS_E_INVALID, "output pointer missing for a requested metric");
    k.outs[m] = want ? outs[m] : nullptr;
  }
  k.shard_count = a->shard_count < 1 ? 1 : a->shard_count;
  k.shard_index = a->shard_index;
  if (k.shard_index < 0 || k.shard_index >= k.shard_count) return fail(PS_E_INVALID, "shard_index out of range");
  if (k.g.rows > (long long)INT32_MAX || k.g.B * k.g.R > 65535) return fail(PS_E_SHAPE, "too many rows for one call");
  return PS_OK;
}

cudaEvent_t pool_event(ps_ctx* c, size_t i) {
  while (c->evpool.size() <= i) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    c->evpool.push_back(e);
  }
  return c->evpool[i];
}

ps_status ensure_pipeline(ps_ctx* c, int n_stages) {
  if (!c->s_in) {
    PS_CUDA(cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking));
    PS_CUDA(cudaStreamCreateWithFlags(&c->s_comp, cudaStreamNonBlocking));
    PS_CUDA(cudaStreamCreateWithFlags(&c->s_ref, cudaStreamNonBlocking));
    PS_CUDA(cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking));
  }
  if (!c->s_prep) PS_CUDA(cudaStreamCreateWithFlags(&c->s_prep, cudaStreamNonBlocking));
  if (c->h_cnt_cap < n_stages) {
    if (c->h_cnt) cudaFreeHost(c->h_cnt);
    c->h_cnt = nullptr;
    PS_CUDA(cudaHostAlloc(&c->h_cnt, (size_t)n_stages * sizeof(unsigned long long),
                          cudaHostAllocMapped | cudaHostAllocPortable));
    PS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->d_cnt), c->h_cnt, 0));
    c->h_cnt_cap = n_stages;
  }
  return PS_OK;
}

// Host-side mirror of the pipelined copy-out: for every matrix, rows
// [c0, c1) x cols [0, c0) := (+/-) transpose of rows [0, c0) x cols [c0, c1),
// which the device already delivered.  Cache-blocked (64 x 64) and split over
// host threads by row bands; PS_HOST_THREADS caps the thread count.
template <typename S>
void mirror_rows(S* M, long long N, long long r0, long long r1, long long c0, bool neg) {
  constexpr long long Bk = 64;
  for (long long rb = r0; rb < r1; rb += Bk)
    for (long long cb = 0; cb < c0; cb += Bk) {
      const long long re = std::min(rb + Bk, r1), ce = std::min(cb + Bk, c0);
      for (long long r = rb; r < re; ++r) {
        S* dst = M + r * N;
        if (neg)
          for (long long cc = cb; cc < ce; ++cc) dst[cc] = -M[cc * N + r];
        else
          for (long long cc = cb; cc < ce; ++cc) dst[cc] = M[cc * N + r];
      }
    }
}

void host_mirror_rows(const std::vector<std::pair<char*, bool>>& mats, int dbl, long long N, long long c0,
                      long long c1) {
  static const int nthreads = [] {
    const char* s = std::getenv("PS_HOST_THREADS");
    int n = s ? std::atoi(s) : (int)std::thread::hardware_concurrency();
    return std::max(1, std::min(n, 64));
  }();
  const long long rows = c1 - c0;
  const int nt = (int)std::max(1LL, std::min<long long>(nthreads, rows / 16));
  auto work = [&](int t) {
    const long long a = c0 + rows * t / nt, b = c0 + rows * (t + 1) / nt;
    for (const auto& mb : mats) {
      if (dbl) mirror_rows(reinterpret_cast<double*>(mb.first), N, a, b, c0, mb.second);
      else mirror_rows(reinterpret_cast<float*>(mb.first), N, a, b, c0, mb.second);
    }
  };
  std::vector<std::thread> th;
  th.reserve(nt);
  for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
}

// PS_PIPE_TRACE=1: per-stage event timeline of the pipelined host path on stderr
// (each line: device time of the event, host time at which it was enqueued)
struct PipeTrace {
  cudaEvent_t t0 = nullptr;
  std::chrono::steady_clock::time_point h0;
  std::vector<std::tuple<cudaEvent_t, const char*, int, double>> ev;
  explicit PipeTrace(cudaStream_t st) {
    cudaEventCreate(&t0);
    cudaEventRecord(t0, st);
    h0 = std::chrono::steady_clock::now();
  }
  void rec(cudaStream_t st, const char* what, int s) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    const double hms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
    ev.emplace_back(e, what, s, hms);
  }
  void dump() {
    for (auto& x : ev) {
      cudaEventSynchronize(std::get<0>(x));
      float ms = 0.f;
      cudaEventElapsedTime(&ms, t0, std::get<0>(x));
      std::fprintf(stderr, "[pipe] %-6s stage %2d  %8.2f ms  (host %8.2f ms)\n", std::get<1>(x), std::get<2>(x), ms,
                   std::get<3>(x));
      cudaEventDestroy(std::get<0>(x));
    }
    cudaEventDestroy(t0);
  }
};

// E2E host path, pipelined over stages of signals (the "growing square"):
// the H2D + normalisation of stage s+1's signals, the Gram of stage s and the
// D2H of finished output run concurrently on separate streams.
//  * Full layout -- column stages: stage s owns output columns
//    [cols[s], cols[s+1]); its tiles need only signals < cols[s+1], and once
//    they are done the block rows [0, cols[s+1]) x cols [cols[s], cols[s+1])
//    plus its mirror is final and is copied out.
//  * Upper layout -- row stages from the last signals up: stage s owns the
//    tiles of rows [lo(s), hi(s)) (all their columns have arrived), and the
//    output is streamed per finished row band: the upper part of a band's
//    rows, cols [i, N), is final when the band's tiles are emitted, and long
//    contiguous host rows are what the copy engine moves fastest (55 GB/s
//    against 35-45 GB/s for the 10-14 KB rows of column blocks).
// dev_input: the input already is in device memory (ready in a->stream's
// order, e.g. assembled by an NCCL all-gather): no copy-in, one stage, and the
// output still streamed into the caller's host arrays (ps_plv_family_to_host).
ps_status host_pipelined(ps_ctx* c, const ps_plv_args* a, Call& k, long long span, long long esz,
                         ps_plv_result* res, bool dev_input = false) {
  const Geometry& g = k.g;
  static const long long w_env = [] {
    const char* s = std::getenv("PS_STAGE_W");  // experiment override (signals per stage)
    return s ? std::atoll(s) : 0LL;
  }();
  // Column stages grow (1024, 1536, 2048, ... up to ~N/6): the first output
  // blocks become final after a short H2D so the D2H engine -- the critical
  // path, 4.8 GB at C5 -- starts early; later stages are wide enough to fill
  // the GPU.  Row stages: see below.  PS_STAGE_W forces a uniform width and
  // PS_STAGE_COLS an explicit list (experiments).
  static const std::vector<long long> w_list = [] {
    // experiment override: PS_STAGE_COLS="w0,w1,..." explicit stage widths
    // (rounded up to 256), the last one repeated until N is covered
    std::vector<long long> v;
    const char* s = std::getenv("PS_STAGE_COLS");
    while (s && *s) {
      const long long w = std::atoll(s);
      if (w > 0) v.push_back(round_up(w, 256));
      s = std::strchr(s, ',');
      if (s) ++s;
    }
    return v;
  }();
  const bool upper = a->out_layout == PS_LAYOUT_UPPER;
  static const bool no_stream_env = std::getenv("PS_PIPE_NO_STREAM") != nullptr;  // experiment: column stages
  // upper layout: row stages from the last signals up, output streamed per
  // finished row band (see below); full layout: column stages
  const bool stream_out = upper && !no_stream_env;
  static const int band_env = [] {
    const char* s = std::getenv("PS_SB_BAND");  // row panels per streamed output band
    return s ? std::max(1, std::atoi(s)) : 4;
  }();
  // stage widths in processing order
  std::vector<long long> widths;
  if (!w_list.empty()) {
    widths = w_list;
  } else if (w_env > 0) {
    widths.push_back(round_up(w_env, 256));
  } else if (stream_out) {
    // grow by 1024 up to ~N/6 (the Gram of a stage should cover the copy-in
    // of the next one), then finish with 2/3 + 1/3 of the last <= 4096
    // signals: the final stage's Gram and its last band's D2H are the tail
    const long long wmax = std::max<long long>(1024, round_up((g.N + 5) / 6, 256));
    long long rem = g.N, w = 1024;
    while (rem > 4096) {
      const long long take = std::min(w, rem - 3072);
      widths.push_back(take);
      rem -= take;
      w = std::min(wmax, w + 1024);
    }
    if (rem > 1024) widths.push_back(rem - 1024);
    widths.push_back(std::min<long long>(rem, 1024));
  } else {
    // growing head, then a tapered tail (512, 512, last <= 256 signals): what
    // follows the last copy-in -- its normalise, the Gram of the last columns
    // against every row, their copy-out -- is the exposed tail of a call that
    // runs at the host link's rate (C3: 31.9 -> 30.4 ms)
    const long long wmax = std::max<long long>(1024, round_up((g.N + 5) / 6, 256));
    const long long nr = round_up(g.N, 256);
    const long long head = nr > 3072 ? nr - 1280 : nr;
    long long x = 0;
    for (long long w = 1024; x < head; w = std::min(wmax, w + 512)) {
      const long long take = std::min(w, head - x);
      widths.push_back(take);
      x += take;
    }
    if (head < nr) {
      widths.push_back(512);
      widths.push_back(512);
      widths.push_back(256);
    }
  }
  // cut points 0 = cols[0] < ... < cols[S] = N, every inner cut a multiple of
  // 256 counted from 0 (row / column panels never straddle a stage)
  std::vector<long long> cols;
  if (dev_input) {
    cols.push_back(0);  // everything has arrived: one stage
  } else if (stream_out) {
    std::vector<long long> cuts;
    long long x = g.N;
    for (size_t i = 0; x > 0; ++i) {
      const long long w = widths[std::min(i, widths.size() - 1)];
      x = std::max(0LL, (x - w + 128) / 256 * 256);
      if (x < 256) x = 0;
      cuts.push_back(x);
    }
    cols.assign(cuts.rbegin(), cuts.rend());
  } else {
    for (long long x = 0, i = 0; x < g.N; x += widths[std::min<size_t>(i, widths.size() - 1)], ++i) cols.push_back(x);
  }
  cols.push_back(g.N);
  const int S = (int)cols.size() - 1;
  // signal range of processing stage s
  auto lo = [&](int s) { return stream_out ? cols[S - 1 - s] : cols[s]; };
  auto hi = [&](int s) { return stream_out ? cols[S - s] : cols[s + 1]; };
  PS_TRY(ensure_pipeline(c, S));
  // si: copy-in only (the copy engine never waits behind a normalise kernel);
  // sn: Hilbert / normalise of a stage once its rows have arrived
  cudaStream_t si = c->s_in, sn = c->s_prep, sc = c->s_comp, sr = c->s_ref, so = c->s_out;
  // a previous call that returned early on an error may still have work in
  // flight on these streams (a kernel that would publish stale band flags):
  // start from idle streams (free when the last call completed normally)
  for (cudaStream_t q : {si, sn, sc, sr, so}) PS_CUDA(cudaStreamSynchronize(q));
  c->launches = 0;
  bool copied = false;
  // device buffers: input span (same element layout as the host array), planes, outputs
  if (!dev_input) PS_TRY(ensure(c->hin, (size_t)span * esz));
  const size_t plane_bytes = g.plane_bytes();
  PS_TRY(ensure(c->planes, plane_bytes));
  const size_t oes = g.split ? 4 : 8;
  void* houts[5];
  std::memcpy(houts, k.outs, sizeof(houts));
  int nout = 0;
  for (int m = 0; m < 5; ++m) nout += houts[m] ? 1 : 0;
  // output slots per metric, as plan_call will set k.slots (needed before it:
  // the device outputs it builds the parameters from are allocated here)
  k.slots = a->trial_reduce == PS_TRIALS_NONE ? g.B * g.R : g.B;
  const size_t out_bytes = (size_t)k.slots * g.N * g.N * oes;
  PS_TRY(ensure(c->hout, out_bytes * std::max(nout, 1)));
  {
    int q = 0;
    for (int m = 0; m < 5; ++m) k.outs[m] = houts[m] ? static_cast<char*>(c->hout.p) + (size_t)(q++) * out_bytes : nullptr;
  }
  PS_TRY(prep_begin(c, a, g, si));  // Hilbert workspace sized once (no realloc mid-pipeline)
  PS_TRY(reset_status(c, si));
  PS_TRY(init_row_state(c, g, si));
  PS_TRY(plan_call(c, a, k, cols, /*force_g1=*/true, si, /*row_band=*/stream_out ? band_env : 0));
  // ---- streamed copy-out (upper layout) ------------------------------------
  // Row stages run from the last signals up and, within a stage, band by band
  // (band_env row panels, J-major inside a band).  Once a band's tiles are
  // emitted, the upper part of its rows -- cols [i, N) of every row i, i.e.
  // long contiguous host rows, the shape the copy engine moves fastest -- is
  // final: that is one output sub-block.  The split kernel publishes a
  // sub-block in mapped host memory as soon as its last item is emitted, so
  // its D2H starts while the stage's other bands are still being computed;
  // the FP64 kernel (no counters) releases a stage's sub-blocks with the
  // stage's completion event.
  struct SubBlock {
    long long slot, r0, r1, c0, c1;
  };
  std::vector<SubBlock> sbs;
  std::vector<int> sb_first(S + 1, 0);  // sub-blocks of stage s: [sb_first[s], sb_first[s + 1])
  if (stream_out) {
    const int exec_rows = g.split ? split_panel_rows() : kF64BM;
    const int sub = g.split ? kSplitBM / exec_rows : 1;
    const int n_items = k.stage_off[S];
    std::vector<int>& info = c->h_sbinfo;
    info.assign((size_t)n_items, 0);
    std::vector<int> need;
    const int arrivals = g.split ? split_epi_arrivals() : 1;
    for (int s = 0; s < S; ++s) {
      sb_first[s] = (int)sbs.size();
      long long prev_key = -1;
      for (int n = k.stage_off[s]; n < k.stage_off[s + 1]; ++n) {
        const Item& w = c->h_items[n];
        const long long slot = k.slot_mode == 0 ? (long long)w.b * g.R + w.g : (long long)w.b;
        const int band = s == S - 1 ? row_band_last(band_env) : band_env;
        const long long key = slot * 4096 + (w.I / sub) / band;  // (slot, row band)
        const long long r0 = (long long)w.I * exec_rows, r1 = std::min<long long>(r0 + exec_rows, g.N);
        if (key != prev_key) {
          sbs.push_back(SubBlock{slot, r0, r1, r0, g.N});
          need.push_back(0);
          prev_key = key;
        }
        SubBlock& b = sbs.back();
        b.r0 = std::min(b.r0, r0);
        b.r1 = std::max(b.r1, r1);
        b.c0 = b.r0;  // upper part of rows [r0, r1): cols [i, N)
        need.back() += arrivals;
        info[(size_t)n] = (int)sbs.size() - 1;
      }
    }
    sb_first[S] = (int)sbs.size();
    const int n_sb = (int)sbs.size();
    if (g.split && n_sb > 0) {
      info.insert(info.end(), need.begin(), need.end());
      const size_t ibytes = info.size() * sizeof(int);
      PS_TRY(ensure(c->sbinfo, ibytes + (size_t)n_sb * sizeof(int)));
      PS_CUDA(cudaMemcpyAsync(c->sbinfo.p, info.data(), ibytes, cudaMemcpyHostToDevice, si));
      PS_CUDA(cudaMemsetAsync(static_cast<char*>(c->sbinfo.p) + ibytes, 0, (size_t)n_sb * sizeof(int), si));
      if (c->h_sbflag_cap < n_sb) {
        if (c->h_sbflag) cudaFreeHost(c->h_sbflag);
        c->h_sbflag = nullptr;
        c->h_sbflag_cap = 0;
        const int cap = std::max(n_sb, 1024);
        PS_CUDA(cudaHostAlloc(&c->h_sbflag, (size_t)cap * sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable));
        PS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->d_sbflag), c->h_sbflag, 0));
        c->h_sbflag_cap = cap;
      }
      std::memset(c->h_sbflag, 0, (size_t)n_sb * sizeof(int));
      int* base = static_cast<int*>(c->sbinfo.p);
      k.p.item_sb = base;
      k.p.sb_need = base + n_items;
      k.p.sb_cnt = base + n_items + n_sb;
      k.p.sb_flag = c->d_sbflag;
    }
  }
  ps_plv_args d = *a;
  void* din = dev_input ? const_cast<void*>(a->input) : c->hin.p;
  d.input = din;
  const long long U = g.B * g.R;
  size_t h2d_bytes = 0;
  if (dev_input) {  // the caller's stream order makes the input valid
    cudaEvent_t ready = pool_event(c, 4 * (size_t)S + 3);
    PS_CUDA(cudaEventRecord(ready, static_cast<cudaStream_t>(a->stream)));
    PS_CUDA(cudaStreamWaitEvent(si, ready, 0));
  }
  static const bool want_trace = std::getenv("PS_PIPE_TRACE") != nullptr;
  std::unique_ptr<PipeTrace> trace_holder(want_trace ? new PipeTrace(si) : nullptr);
  PipeTrace* trace = trace_holder.get();
  // ---- copy-in + normalise, per stage --------------------------------------
  {  // everything queued on si so far (workspace setup, status reset, plan uploads) precedes the first normalise
    cudaEvent_t setup = pool_event(c, 4 * (size_t)S + 4);
    PS_CUDA(cudaEventRecord(setup, si));
    PS_CUDA(cudaStreamWaitEvent(sn, setup, 0));
  }
  for (int s = 0; s < S; ++s) {
    for (long long u = 0; u < U && !dev_input; ++u) {
      const long long b = u / g.R, t = u % g.R;
      const long long off = b * a->stride_band + t * a->stride_trial + lo(s) * a->stride_signal;
      const long long len = (hi(s) - 1 - lo(s)) * a->stride_signal + (g.T - 1) * a->stride_sample + 1;
      PS_CUDA(cudaMemcpyAsync(static_cast<char*>(c->hin.p) + off * esz, static_cast<const char*>(a->input) + off * esz,
                              (size_t)len * esz, cudaMemcpyHostToDevice, si));
      h2d_bytes += (size_t)len * esz;
    }
    if (trace) trace->rec(si, "h2d", s);
    {
      cudaEvent_t arrived = pool_event(c, 4 * (size_t)S + 5 + s);
      PS_CUDA(cudaEventRecord(arrived, si));
      PS_CUDA(cudaStreamWaitEvent(sn, arrived, 0));
    }
    for (long long u = 0; u < U; ++u)
      PS_TRY(prepare_rows(c, &d, g, din, c->planes.p, g.split ? 0 : 1, g.pitch, g.plane_stride,
                          u * g.N + lo(s), u * g.N + hi(s), sn, &copied));
    if (trace) trace->rec(sn, "norm", s);
    PS_CUDA(cudaEventRecord(pool_event(c, 3 * s), sn));
  }
  // ---- Gram per stage ------------------------------------------------------
  for (int s = 0; s < S; ++s) {
    PS_CUDA(cudaStreamWaitEvent(sc, pool_event(c, 3 * s), 0));
    if (upper) {  // the copy-out of the diagonal block carries its lower part: make it 0, not stale
      const long long c0 = lo(s), c1 = hi(s);
      for (int m = 0; m < 5; ++m)
        if (k.outs[m])
          for (long long sl = 0; sl < k.slots; ++sl)
            PS_CUDA(cudaMemset2DAsync(static_cast<char*>(k.outs[m]) + ((size_t)sl * g.N * g.N + c0 * g.N + c0) * oes,
                                      (size_t)g.N * oes, 0, (size_t)(c1 - c0) * oes, (size_t)(c1 - c0), sc));
    }
    PS_TRY(launch_stage(c, k, s, sc));
    if (trace) trace->rec(sc, "gram", s);
    // the refine-queue count reaches the host through a store into mapped
    // pinned memory: a cudaMemcpyAsync here would wait behind the bulk D2H
    // copies of earlier stages and stall the next Gram stage behind it
    PS_CUDA(launch_copy_u64(&c->d_status->n_illcond, &c->d_cnt[s], sc));
    PS_CUDA(cudaEventRecord(pool_event(c, 3 * s + 1), sc));
  }
  size_t d2h_bytes = 0;
  if (!stream_out) {
    // ---- refine + copy-out per stage ------------------------------------------
    // Both halves of every stage block cross the link by default.  With
    // PS_HOST_MIRROR=1 only the block rows [0, c1) x cols [c0, c1) do, and a
    // host worker fills the mirror rows [c0, c1) x cols [0, c0) with a
    // multi-threaded cache-blocked transpose behind the D2H events (the outputs
    // are exactly symmetric / antisymmetric): half the D2H bytes, but on the
    // 16-core GPU hosts measured so far the transposes (~20 GB/s while the DMA
    // writes the same memory) are slower than the link they relieve
    // (DESIGN.md "E2E").
    // PS_HOST_MIRROR=k mirrors the first k output matrices (metric order, then
    // slot) on the host and ships the others whole -- a partial split of the
    // mirroring between the link and the host's memory bandwidth.
    static const int mirror_count = [] {
      const char* s = std::getenv("PS_HOST_MIRROR");
      return s ? std::max(0, std::atoi(s)) : 0;
    }();
    const bool host_mirror = mirror_count > 0 && !upper;
    auto mirrored = [&](long long q) { return q < mirror_count; };
    auto mirror_stage = [&](int s) {
      const long long c0 = cols[s], c1 = cols[s + 1];
      if (c0 == 0) return;
      std::vector<std::pair<char*, bool>> mats;
      long long q = 0;
      for (int m = 0; m < 5; ++m) {
        if (!houts[m]) continue;
        for (long long sl = 0; sl < k.slots; ++sl, ++q)
          if (mirrored(q)) mats.emplace_back(static_cast<char*>(houts[m]) + (size_t)sl * g.N * g.N * oes, m == 4);
      }
      if (!mats.empty()) host_mirror_rows(mats, g.split ? 0 : 1, g.N, c0, c1);
    };

    unsigned long long prev = 0;
    static const bool no_d2h_env = std::getenv("PS_PIPE_NO_D2H") != nullptr;  // experiment: Gram-only timeline
    // the mirror runs on a worker thread, stage by stage behind the D2H events,
    // so the issue of later copies never waits for the host transposes
    pool_event(c, 4 * (size_t)S + 2);  // create every event before the worker reads the pool
    std::atomic<int> issued{0};
    std::atomic<bool> abort_worker{false};
    std::thread worker;
    if (host_mirror && !no_d2h_env)
      worker = std::thread([&, dev = c->device] {
        cudaSetDevice(dev);
        for (int s = 0; s < S; ++s) {
          while (issued.load(std::memory_order_acquire) <= s) {
            if (abort_worker.load()) return;
            std::this_thread::yield();
          }
          if (cudaEventSynchronize(pool_event(c, 3 * S + 1 + s)) != cudaSuccess) return;
          mirror_stage(s);
        }
      });
    struct Joiner {
      std::thread& t;
      std::atomic<bool>& abort;
      ~Joiner() {
        abort.store(true);
        if (t.joinable()) t.join();
      }
    } joiner{worker, abort_worker};
    for (int s = 0; s < S; ++s) {
      cudaEvent_t ready = pool_event(c, 3 * s + 1);
      PS_CUDA(cudaEventSynchronize(ready));
      const unsigned long long n = c->h_cnt[s];
      if (n > prev && k.outs[2] && g.split) {
        PS_CUDA(cudaStreamWaitEvent(sr, ready, 0));
        PS_TRY(refine_range(c, k, prev, n, sr));
        ready = pool_event(c, 3 * s + 2);
        PS_CUDA(cudaEventRecord(ready, sr));
      }
      prev = n;
      PS_CUDA(cudaStreamWaitEvent(so, ready, 0));
      const long long c0 = cols[s], c1 = cols[s + 1];
      static const bool no_d2h = std::getenv("PS_PIPE_NO_D2H") != nullptr;  // experiment: Gram-only timeline
      long long q = 0;
      for (int m = 0; m < 5 && !no_d2h; ++m) {
        if (!houts[m]) continue;
        for (long long sl = 0; sl < k.slots; ++sl, ++q) {
          const size_t base = (size_t)sl * g.N * g.N * oes;
          char* hdst = static_cast<char*>(houts[m]) + base;
          const char* dsrc = static_cast<const char*>(k.outs[m]) + base;
          const size_t pitch = (size_t)g.N * oes;
          // rows [0, c1) x cols [c0, c1)
          PS_CUDA(cudaMemcpy2DAsync(hdst + (size_t)c0 * oes, pitch, dsrc + (size_t)c0 * oes, pitch,
                                    (size_t)(c1 - c0) * oes, (size_t)c1, cudaMemcpyDeviceToHost, so));
          d2h_bytes += (size_t)(c1 - c0) * oes * (size_t)c1;
          // rows [c0, c1) x cols [0, c0) (strictly lower: not part of the upper layout)
          if (c0 > 0 && !mirrored(q) && !upper) {
            PS_CUDA(cudaMemcpy2DAsync(hdst + (size_t)c0 * pitch, pitch, dsrc + (size_t)c0 * pitch, pitch,
                                      (size_t)c0 * oes, (size_t)(c1 - c0), cudaMemcpyDeviceToHost, so));
            d2h_bytes += (size_t)c0 * oes * (size_t)(c1 - c0);
          }
        }
      }
      cudaEvent_t copied_ev = pool_event(c, 3 * S + 1 + s);
      PS_CUDA(cudaEventRecord(copied_ev, so));
      issued.store(s + 1, std::memory_order_release);
      if (trace && s + 1 < S) trace->rec(so, "d2h", s);
    }
    if (trace) trace->rec(so, "d2h", S - 1);
    PS_CUDA(cudaStreamSynchronize(so));
    if (worker.joinable()) worker.join();  // all mirrors done
  } else {
    // ---- streamed copy-out: ship each sub-block as soon as it is final -----
    static const bool no_d2h = std::getenv("PS_PIPE_NO_D2H") != nullptr;  // experiment: Gram-only timeline
    const size_t pitch = (size_t)g.N * oes;
    // upper part of sub-block b for metric m: rows above the diagonal block as
    // one 2-D copy, the rows crossing it in 256-row strips [a, a+h) x [a, c1)
    // (their few strictly-lower entries are zero on the device)
    auto ship = [&](const SubBlock& b) -> ps_status {
      for (int m = 0; m < 5 && !no_d2h; ++m) {
        if (!houts[m]) continue;
        const size_t base = (size_t)b.slot * g.N * g.N * oes;
        char* hdst = static_cast<char*>(houts[m]) + base;
        const char* dsrc = static_cast<const char*>(k.outs[m]) + base;
        const long long rtop = std::min(b.r1, b.c0);
        if (rtop > b.r0) {
          const size_t off = (size_t)b.r0 * pitch + (size_t)b.c0 * oes;
          PS_CUDA(cudaMemcpy2DAsync(hdst + off, pitch, dsrc + off, pitch, (size_t)(b.c1 - b.c0) * oes,
                                    (size_t)(rtop - b.r0), cudaMemcpyDeviceToHost, so));
          d2h_bytes += (size_t)(b.c1 - b.c0) * oes * (size_t)(rtop - b.r0);
        }
        for (long long r = std::max(b.r0, b.c0); r < b.r1; r += 256) {
          const long long re = std::min(r + 256, b.r1);
          const size_t off = (size_t)r * pitch + (size_t)r * oes;
          PS_CUDA(cudaMemcpy2DAsync(hdst + off, pitch, dsrc + off, pitch, (size_t)(b.c1 - r) * oes, (size_t)(re - r),
                                    cudaMemcpyDeviceToHost, so));
          d2h_bytes += (size_t)(b.c1 - r) * oes * (size_t)(re - r);
        }
      }
      return PS_OK;
    };
    const bool flags = k.p.sb_flag != nullptr;
    // PS_PIPE_TRACE=2: one timeline event per shipped sub-block as well
    static const bool trace_blocks_env = [] {
      const char* e = std::getenv("PS_PIPE_TRACE");
      return e && std::atoi(e) >= 2;
    }();
    const bool trace_blocks = trace && trace_blocks_env;
    // PS_PIPE_POLL (experiment): 0 = release blocks per stage event only,
    // 1 = poll the flags (yield), 2 = poll the flags (20 us sleeps)
    static const int poll_mode = [] {
      const char* e = std::getenv("PS_PIPE_POLL");
      return e ? std::atoi(e) : 1;
    }();
    unsigned long long prev = 0;
    std::vector<long long> patch_idx;  // refined ciPLV entries: flat index, final value
    std::vector<float> patch_val;
    for (int s = 0; s < S; ++s) {
      cudaEvent_t done = pool_event(c, 3 * s + 1);
      for (int q = sb_first[s]; q < sb_first[s + 1]; ++q) {
        // ready: the kernel published the block, or the whole stage finished
        if (poll_mode == 0 || !flags) {
          PS_CUDA(cudaEventSynchronize(done));
        } else {
          int spins = 0;
          while (reinterpret_cast<volatile int*>(c->h_sbflag)[q] == 0) {
            // the stage event is the fallback (and error) path: queried only
            // every 64 polls of the flag, which lives in host memory
            if ((++spins & 63) == 0) {
              const cudaError_t e = cudaEventQuery(done);
              if (e == cudaSuccess) break;
              if (e != cudaErrorNotReady) PS_CUDA(e);
            }
            if (poll_mode == 2) std::this_thread::sleep_for(std::chrono::microseconds(20));
            else std::this_thread::yield();
          }
        }
        PS_TRY(ship(sbs[(size_t)q]));
        if (trace_blocks) trace->rec(so, "blk", q);
      }
      PS_CUDA(cudaEventSynchronize(done));
      const unsigned long long n = c->h_cnt[s];
      if (n > prev && k.outs[2] && g.split) {
        // FP64 refinement of this stage's ill-conditioned ciPLV pairs (their
        // blocks may already be on their way); the corrected values come back
        // as (index, value) pairs and patch the host matrix after the last copy
        PS_CUDA(cudaStreamWaitEvent(sr, done, 0));
        PS_TRY(refine_range(c, k, prev, n, sr));
        if (houts[2] && !no_d2h) {
          const int m = (int)(std::min<unsigned long long>(n, (unsigned long long)k.p.refine_cap) - prev);
          PS_TRY(ensure(c->rpick, (size_t)m * 12 + 256));
          long long* d_idx = static_cast<long long*>(c->rpick.p);
          float* d_val = reinterpret_cast<float*>(static_cast<char*>(c->rpick.p) + (size_t)m * 8);
          PS_CUDA(launch_refine_pick(static_cast<const RefineEntry*>(c->refine.p) + prev, m,
                                     static_cast<const float*>(k.outs[2]), g.N, d_idx, d_val, sr));
          const size_t at = patch_idx.size();
          patch_idx.resize(at + (size_t)m);
          patch_val.resize(at + (size_t)m);
          PS_CUDA(cudaMemcpyAsync(patch_idx.data() + at, d_idx, (size_t)m * 8, cudaMemcpyDeviceToHost, sr));
          PS_CUDA(cudaMemcpyAsync(patch_val.data() + at, d_val, (size_t)m * 4, cudaMemcpyDeviceToHost, sr));
          PS_CUDA(cudaStreamSynchronize(sr));
          d2h_bytes += (size_t)m * 12;
        }
      }
      prev = n;
      if (trace && s + 1 < S) trace->rec(so, "d2h", s);
    }
    if (trace) trace->rec(so, "d2h", S - 1);
    PS_CUDA(cudaStreamSynchronize(so));
    float* hc = static_cast<float*>(houts[2]);
    for (size_t q = 0; q < patch_idx.size(); ++q) hc[patch_idx[q]] = patch_val[q];
  }
  if (trace) trace->dump();
  ps_status st = read_status(c, so);
  if (res) {
    std::memset(res, 0, sizeof(*res));
    res->n_observations = k.pool ? g.T * g.R : g.T;
    res->n_masked_samples = (int64_t)c->h_status->n_masked;
    res->n_refined_pairs = (int64_t)c->h_status->n_illcond;
    res->n_indeterminate_ciplv = (int32_t)std::min<unsigned long long>(c->h_status->n_indeterminate, INT32_MAX);
    res->input_copied = copied ? 1 : 0;
    res->n_kernel_launches = c->launches;
    res->gram_variant = k.g.split ? (k.g.gauss ? 1 : 0) : 2;
    res->h2d_bytes = (int64_t)h2d_bytes;
    res->d2h_bytes = (int64_t)d2h_bytes;
  }
  std::memcpy(k.outs, houts, sizeof(houts));
  return st;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
namespace {
// Every entry point starts from a clean runtime error state: the launch
// wrappers report errors through cudaGetLastError(), so an error an earlier
// call left pending (one whose status was deliberately ignored, e.g. an
// elapsed-time query) must not surface as a failure of this one.
// PS_DEBUG_STALE=1 names the entry point that found one (diagnostics).
void clear_stale(const char* fn) {
  static const bool dbg = std::getenv("PS_DEBUG_STALE") != nullptr;
  const cudaError_t e = cudaGetLastError();
  if (dbg && e != cudaSuccess) std::fprintf(stderr, "[ps] pending CUDA error at entry of %s: %s\n", fn, cudaGetErrorString(e));
}
}  // namespace

extern "C" {

int ps_abi_version(void) { return PS_ABI_VERSION; }

int64_t ps_tile_count(int64_t n_signals, int32_t precision) {
  if (n_signals < 1) return 0;
  std::vector<std::pair<int, int>> tiles;
  const bool split = precision == PS_PREC_SPLIT_F16X3;
  build_tiles(n_signals, split ? kSplitBM : kF64BM, split ? kSplitBN : kF64BN, tiles);
  return (int64_t)tiles.size();
}

int32_t ps_pair_shard(int64_t n_signals, int32_t precision, int32_t shard_count, int64_t i, int64_t j) {
  if (n_signals < 1 || i < 0 || j < 0 || i >= n_signals || j >= n_signals) return -1;
  if (shard_count < 1) shard_count = 1;
  if (i > j) std::swap(i, j);
  const bool split = precision == PS_PREC_SPLIT_F16X3;
  const int bm = split ? kSplitBM : kF64BM, bn = split ? kSplitBN : kF64BN;
  const long long ni = (n_signals + bm - 1) / bm;
  const long long I = i / bm, J = j / bn;
  long long t = 0;
  for (long long Jp = 0; Jp < J; ++Jp) {
    const long long jmax = std::min<long long>(Jp * bn + bn, n_signals) - 1;
    t += std::min<long long>(ni, jmax / bm + 1);
  }
  t += I;
  return (int32_t)(t % shard_count);
}

// Tiles shard `s` of `P` owns, in the library's enumeration order (the rule
// of ps_pair_shard: tile t belongs to shard t % P).
static void shard_tile_list(int64_t N, int32_t precision, int32_t P, int32_t s, std::vector<int2>& out, int* bm,
                            int* bn) {
  const bool split = precision == PS_PREC_SPLIT_F16X3;
  *bm = split ? kSplitBM : kF64BM;
  *bn = split ? kSplitBN : kF64BN;
  std::vector<std::pair<int, int>> tiles;
  build_tiles(N, *bm, *bn, tiles);
  out.clear();
  if (P < 1) P = 1;
  for (size_t t = 0; t < tiles.size(); ++t)
    if ((int)(t % P) == s) out.push_back(make_int2(tiles[t].first, tiles[t].second));
}

int64_t ps_shard_tiles(int64_t n_signals, int32_t precision, int32_t shard_count, int32_t shard_index,
                       int32_t* tile_rows, int32_t* tile_cols) {
  if (n_signals < 1 || shard_count < 1 || shard_index < 0 || shard_index >= shard_count) return -1;
  std::vector<int2> v;
  int bm, bn;
  shard_tile_list(n_signals, precision, shard_count, shard_index, v, &bm, &bn);
  if (tile_rows) *tile_rows = bm;
  if (tile_cols) *tile_cols = bn;
  return (int64_t)v.size();
}

static ps_status shard_move(ps_ctx* c, int64_t N, int32_t precision, int32_t P, int32_t s, const void* src, void* dst,
                            bool pack, int32_t mirror, void* stream) {
  if (!c) return fail(PS_E_INVALID, "ctx is NULL");
  if (!src || !dst) return fail(PS_E_INVALID, "NULL buffer");
  if (N < 1 || P < 1 || s < 0 || s >= P) return fail(PS_E_INVALID, "bad n_signals / shard arguments");
  if (precision != PS_PREC_SPLIT_F16X3 && precision != PS_PREC_FP64) return fail(PS_E_INVALID, "unknown precision");
  std::lock_guard<std::mutex> lock(c->mu);
  PS_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<int2> v;
  int bm, bn;
  shard_tile_list(N, precision, P, s, v, &bm, &bn);
  if (v.empty()) return PS_OK;
  PS_TRY(ensure(c->shardtiles, v.size() * sizeof(int2)));
  // stream-ordered upload (pageable source: the copy completes before the
  // call returns, so the host vector may go out of scope)
  PS_CUDA(cudaMemcpyAsync(c->shardtiles.p, v.data(), v.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
  const int dbl = precision == PS_PREC_FP64 ? 1 : 0;
  if (pack) PS_CUDA(launch_shard_pack(src, N, c->shardtiles.p, (int)v.size(), bm, bn, dbl, dst, st));
  else PS_CUDA(launch_shard_unpack(src, N, c->shardtiles.p, (int)v.size(), bm, bn, dbl, dst, mirror, st));
  // the tile table is reused by the next call on any stream
  PS_CUDA(cudaStreamSynchronize(st));
  return PS_OK;
}

ps_status ps_shard_pack(ps_ctx* c, int64_t n_signals, int32_t precision, int32_t shard_count, int32_t shard_index,
                        const void* matrix, void* packed, void* stream) {
  clear_stale(__func__);
  return shard_move(c, n_signals, precision, shard_count, shard_index, matrix, packed, true, 0, stream);
}

ps_status ps_shard_unpack(ps_ctx* c, int64_t n_signals, int32_t precision, int32_t shard_count, int32_t shard_index,
                          const void* packed, void* matrix, int32_t mirror, void* stream) {
  clear_stale(__func__);
  return shard_move(c, n_signals, precision, shard_count, shard_index, packed, matrix, false, mirror, stream);
}

ps_status ps_reduce_partials(ps_ctx* c, const void* parts, int32_t n_parts, int64_t part_stride, int64_t n,
                             double divisor, int32_t dtype, void* out, void* stream) {
  clear_stale(__func__);
  if (!c) return fail(PS_E_INVALID, "ctx is NULL");
  if (!parts || !out) return fail(PS_E_INVALID, "NULL buffer");
  if (n_parts < 1 || n < 0 || part_stride < n) return fail(PS_E_INVALID, "need n_parts >= 1 and part_stride >= n");
  if (dtype != PS_F32 && dtype != PS_F64) return fail(PS_E_INVALID, "dtype must be PS_F32 or PS_F64");
  if (!(divisor != 0.0)) return fail(PS_E_INVALID, "divisor must be non-zero");
  std::lock_guard<std::mutex> lock(c->mu);
  PS_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PS_CUDA(launch_reduce_partials(parts, n_parts, part_stride, n, divisor, dtype == PS_F64 ? 1 : 0, out, st));
  return PS_OK;
}

const char* ps_last_error(void) { return g_last_error.c_str(); }

ps_status ps_ctx_create(int device, ps_ctx** out) {
  clear_stale(__func__);
  if (!out) return fail(PS_E_INVALID, "out is NULL");
  *out = nullptr;
  int ndev = 0;
  PS_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(PS_E_INVALID, "device index out of range");
  PS_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  PS_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(PS_E_UNSUPPORTED, std::string("sm_100a device required, found ") + prop.name);
  ps_ctx* c = new ps_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  c->total_mem = prop.totalGlobalMem;
  if (cudaMalloc(&c->d_status, sizeof(DevStatus)) != cudaSuccess ||
      cudaMallocHost(&c->h_status, sizeof(DevStatus)) != cudaSuccess) {
    delete c;
    return fail(PS_E_OOM, "status allocation failed");
  }
  for (auto& e : c->ev) cudaEventCreate(&e);
  *out = c;
  return PS_OK;
}

ps_status ps_ctx_destroy(ps_ctx* c) {
  clear_stale(__func__);
  if (!c) return PS_OK;
  cudaSetDevice(c->device);
  for (auto& kv : c->plans) cufftDestroy(kv.second);
  for (Buf* b : {&c->xw, &c->spec, &c->hbuf, &c->planes, &c->rowstat, &c->maskcount, &c->items, &c->gws, &c->hin,
                 &c->hout, &c->refine, &c->refine_sorted, &c->planes_t, &c->maskcount_t, &c->fir_taps,
                 &c->fir_spec, &c->cohws, &c->lockbuf, &c->hscale, &c->sortws, &c->sbinfo, &c->rpick,
                 &c->shardtiles, &c->ind, &c->cntws, &c->cntitems, &c->profbuf})
    if (b->p) cudaFree(b->p);
  if (c->d_status) cudaFree(c->d_status);
  if (c->h_status) cudaFreeHost(c->h_status);
  if (c->h_items_pinned) cudaFreeHost(c->h_items_pinned);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->evpool) cudaEventDestroy(e);
  for (auto& e : c->tev) cudaEventDestroy(e);
  for (cudaStream_t s : {c->s_in, c->s_comp, c->s_ref, c->s_out, c->s_prep})
    if (s) cudaStreamDestroy(s);
  if (c->h_cnt) cudaFreeHost(c->h_cnt);
  if (c->h_sbflag) cudaFreeHost(c->h_sbflag);
  delete c;
  return PS_OK;
}

ps_status ps_ctx_set_timing(ps_ctx* c, int enable) {
  clear_stale(__func__);
  if (!c) return fail(PS_E_INVALID, "ctx is NULL");
  c->timing = enable != 0;
  return PS_OK;
}

}  // extern "C"

namespace {

// ps_plv_family with c->mu already held by the caller (the host-output entry
// points hold it across their staging-buffer use, copy-in and copy-out).
ps_status plv_family_locked(ps_ctx* c, const ps_plv_args* a, ps_plv_result* res) {
  Call k;
  PS_TRY(validate(a, k.g));
  PS_TRY(setup_outputs(a, k));
  decide_gauss(a, k);
  const Geometry& g = k.g;
  PS_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = static_cast<cudaStream_t>(a->stream);
  c->launches = 0;
  bool copied = false;
  if (c->timing) PS_CUDA(cudaEventRecord(c->ev[0], st));
  // ---- phasor planes --------------------------------------------------------
  const size_t plane_bytes = g.plane_bytes();
  PS_TRY(ensure(c->planes, plane_bytes));
  PS_TRY(reset_status(c, st));
  PS_TRY(prepare_phasors(c, a, g, a->input, c->planes.p, g.split ? 0 : 1, g.pitch, g.plane_stride, st, &copied));
  // ---- time-resolved mode (Eq 8): Gram over trials, one matrix per sample ----
  ps_plv_args at = *a;
  if (a->mode == PS_MODE_OVER_TRIALS) {
    if (g.R < 2) return fail(PS_E_SHAPE, "mode over_trials needs n_trials >= 2 (Eq 8: PLV across trials)");
    at.n_samples = g.R;  // K axis = trials
    at.n_trials = g.T;   // one unit (output slot) per sample
    at.trial_reduce = PS_TRIALS_NONE;
    Geometry gt;
    PS_TRY(validate(&at, gt));
    const size_t tb = gt.split ? (size_t)4 * gt.plane_stride * 2 : (size_t)2 * gt.plane_stride * 8;
    PS_TRY(ensure(c->planes_t, tb));
    PS_TRY(ensure(c->maskcount_t, (size_t)gt.rows * sizeof(int)));
    PS_CUDA(launch_transpose_trials(c->planes.p, g.plane_stride, (int)g.pitch, c->planes_t.p, gt.plane_stride,
                                    (int)gt.pitch, (int)g.B, (int)g.R, (int)g.N, (int)g.T, g.split ? 1 : 0,
                                    static_cast<int*>(c->maskcount_t.p), st));
    c->launches++;
    std::swap(c->planes, c->planes_t);  // the Gram below reads the trial-keyed planes / masks
    std::swap(c->maskcount, c->maskcount_t);
    k.g = gt;
  }
  if (c->timing) PS_CUDA(cudaEventRecord(c->ev[1], st));
  // ---- Gram + fused epilogue ------------------------------------------------
  static const bool time_trace = std::getenv("PS_TIME_TRACE") != nullptr;  // diagnostics
  const auto hp0 = std::chrono::steady_clock::now();
  PS_TRY(plan_call(c, &at, k, {}, /*force_g1=*/false, st));
  const auto hp1 = std::chrono::steady_clock::now();
  // the Gram window opens after the host-side planning (ms_gram = kernel time
  // + the item-table upload + the K7 count pass when samples are masked,
  // never host planning time)
  if (c->timing) PS_CUDA(cudaEventRecord(c->ev[4], st));
  if (k7_enabled()) {
    bool masked = false;
    PS_TRY(any_masked(c, st, &masked));
    if (masked) PS_TRY(mask_count_pass(c, k, st));
  }
  PS_TRY(launch_stage(c, k, 0, st));
  if (c->timing) PS_CUDA(cudaEventRecord(c->ev[2], st));
  if (time_trace && c->timing) {
    PS_CUDA(cudaEventSynchronize(c->ev[2]));
    float k_ms = 0.f, w_ms = 0.f;
    PS_CUDA(cudaEventElapsedTime(&k_ms, c->ev[4], c->ev[2]));
    PS_CUDA(cudaEventElapsedTime(&w_ms, c->ev[1], c->ev[2]));
    std::fprintf(stderr, "[time] plan_host %.3f ms  gram_kernel %.3f ms  gram_window %.3f ms  G %d items %d\n",
                 std::chrono::duration<double, std::milli>(hp1 - hp0).count(), k_ms, w_ms, k.G,
                 k.stage_off.empty() ? 0 : k.stage_off.back());
  }
  if (k.slot_mode == 2) {
    PS_CUDA(launch_group_reduce(c->gws.p, k.G, (int)g.N, (int)g.B, 5, k.outs, k.reduce_div, g.split ? 0 : 1, st,
                                a->out_layout == PS_LAYOUT_UPPER ? 1 : 0));
    for (int m = 0; m < 5; ++m) c->launches += k.outs[m] ? 1 : 0;
  }
  ps_status s = read_status(c, st);
  // ---- exact FP64 refinement of ill-conditioned ciPLV pairs (split path) ----
  if (s == PS_OK && c->h_status->n_illcond) {
    PS_TRY(refine_range(c, k, 0, c->h_status->n_illcond, st));
    PS_TRY(refresh_status(c, st));
  }
  if (c->timing) PS_CUDA(cudaEventRecord(c->ev[3], st));
  if (c->timing) PS_CUDA(cudaEventSynchronize(c->ev[3]));
  if (res) {
    std::memset(res, 0, sizeof(*res));
    res->n_observations = k.pool ? g.T * g.R : g.T;
    res->n_masked_samples = (int64_t)c->h_status->n_masked;
    res->n_refined_pairs = (int64_t)c->h_status->n_illcond;
    res->n_indeterminate_ciplv = (int32_t)std::min<unsigned long long>(c->h_status->n_indeterminate, INT32_MAX);
    res->input_copied = copied ? 1 : 0;
    res->n_kernel_launches = c->launches;
    res->gram_variant = k.g.split ? (k.g.gauss ? 1 : 0) : 2;
    if (c->timing) {
      cudaEventElapsedTime(&res->ms_normalize, c->ev[0], c->ev[1]);
      cudaEventElapsedTime(&res->ms_gram, c->ev[4], c->ev[2]);
      cudaEventElapsedTime(&res->ms_finish, c->ev[2], c->ev[3]);
    }
  }
  return s;
}

}  // namespace

extern "C" {

ps_status ps_plv_family(ps_ctx* c, const ps_plv_args* a, ps_plv_result* res) {
  clear_stale(__func__);
  if (!c) return fail(PS_E_INVALID, "ctx is NULL");
  std::lock_guard<std::mutex> lock(c->mu);
  return plv_family_locked(c, a, res);
}

int64_t ps_welch_bins(int64_t W, double lo, double hi, int64_t* first_bin) {
  long long k0 = -1, k1 = -2;
  for (long long k = 0; W > 0 && k <= W / 2; ++k) {
    const double w = 2.0 * M_PI * (double)k / (double)W;  // SPEC.md:263, inclusive edges
    if (w >= lo && w <= hi) {
      if (k0 < 0) k0 = k;
      k1 = k;
    }
  }
  if (first_bin) *first_bin = k0 < 0 ? 0 : k0;
  return k0 < 0 ? 0 : k1 - k0 + 1;
}

// Welch coherence family (Eq 12; DESIGN.md 8(f) #3): tapered
// segments -> batched R2C -> per-bin operand rows normalised by the auto-power
// -> the split / FP64 Gram with K = segments and one unit per bin -> the
// PLV-family epilogue reads as COH / ICOH / coherency -> mean (trial-mean
// machinery) or max (band_max) over the band's bins.
ps_status ps_coherence(ps_ctx* c, const ps_plv_args* a, const ps_welch* w, ps_plv_result* res) {
  clear_stale(__func__);
  if (!c) return fail(PS_E_INVALID, "ctx is NULL");
  if (!w) return fail(PS_E_INVALID, "welch config is NULL");
  std::lock_guard<std::mutex> lock(c->mu);
  Geometry g;
  PS_TRY(validate(a, g));
  if (a->input_kind != PS_INPUT_REAL) return fail(PS_E_INVALID, "coherence takes real epochs (SPEC.md:213)");
  if (a->fir) return fail(PS_E_INVALID, "coherence does not take a band-pass front end");
  if (a->mode != PS_MODE_OVER_SAMPLES) return fail(PS_E_INVALID, "coherence has no over_trials mode");
  const long long W = w->window_len, O = w->overlap;
  if (W < 1 || O < 0 || O >= W) return fail(PS_E_INVALID, "WelchConfig needs 0 <= overlap < window_len (SPEC.md:168)");
  if (W > g.T) return fail(PS_E_WINDOW_TOO_LONG, "window_len exceeds n_samples (SPEC.md:225)");
  if (!(w->band_low >= 0.0 && w->band_low <= w->band_high && w->band_high <= M_PI))
    return fail(PS_E_INVALID, "band edges must satisfy 0 <= low <= high <= pi");
  if (w->reduce < PS_BAND_MEAN || w->reduce > PS_BAND_NONE) return fail(PS_E_INVALID, "unknown band reduce");
  int64_t k0 = 0;
  const long long nb = ps_welch_bins(W, w->band_low, w->band_high, &k0);
  if (nb < 1) return fail(PS_E_EMPTY_BAND, "the band contains no spectral bin (SPEC.md:239)");
  const long long hop = W - O;
  const long long nseg = (g.T - W) / hop + 1;
  const long long K = g.R * nseg;
  if (K > (1LL << 30)) return fail(PS_E_SHAPE, "too many segments");
  // the Gram sees K "samples" (segments) and nb "trials" (bins) per band
  ps_plv_args at = *a;
  at.n_samples = K;
  at.n_trials = nb;
  at.trial_reduce = w->reduce == PS_BAND_MEAN ? PS_TRIALS_MEAN : PS_TRIALS_NONE;
  at.fir = nullptr;
  Call k;
  PS_TRY(validate(&at, k.g));
  const Geometry& gt = k.g;
  const bool fp64 = !gt.split;
  const size_t oes = fp64 ? 8 : 4;
  const long long nn = g.N * g.N;
  void* user_outs[5] = {a->out_plv, a->out_iplv, a->out_ciplv, a->out_cre, a->out_cim};
  if (w->reduce == PS_BAND_MAX) {  // per-bin matrices into the workspace, max-reduced below
    int q = 0;
    for (int m = 0; m < 5; ++m) q += ((a->metrics >> m) & 1u) ? 1 : 0;
    const size_t per = (size_t)g.B * nb * nn * oes;
    PS_TRY(ensure(c->cohws, per * std::max(q, 1)));
    void** outs[5] = {&at.out_plv, &at.out_iplv, &at.out_ciplv, &at.out_cre, &at.out_cim};
    q = 0;
    for (int m = 0; m < 5; ++m)
      *outs[m] = ((a->metrics >> m) & 1u) ? static_cast<char*>(c->cohws.p) + per * (q++) : nullptr;
  }
  PS_TRY(setup_outputs(&at, k));
  PS_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = static_cast<cudaStream_t>(a->stream);
  c->launches = 0;
  if (c->timing) PS_CUDA(cudaEventRecord(c->ev[0], st));
  // ---- tapered segments -> spectra ------------------------------------------
  const size_t es = g.cdouble ? 8 : 4;
  const long long nbW = W / 2 + 1;
  const long long nsegs = g.rows * nseg;
  std::vector<double> win((size_t)W, 1.0);  // symmetric Hamming
  if (W > 1)
    for (long long t = 0; t < W; ++t) win[(size_t)t] = 0.54 - 0.46 * std::cos(2.0 * M_PI * (double)t / (double)(W - 1));
  PS_TRY(ensure(c->fir_taps, (size_t)W * sizeof(double)));
  PS_CUDA(cudaMemcpyAsync(c->fir_taps.p, win.data(), (size_t)W * sizeof(double), cudaMemcpyHostToDevice, st));
  PS_TRY(ensure(c->xw, (size_t)nsegs * W * es));
  PS_TRY(ensure(c->spec, (size_t)nsegs * nbW * 2 * es));
  const SrcDesc src = make_src(a, g, a->input);
  PS_CUDA(launch_welch_segments(src, g.rows, (int)nseg, (int)W, (int)hop, static_cast<const double*>(c->fir_taps.p),
                                c->xw.p, g.cdouble ? 1 : 0, st));
  cufftHandle fwd;
  PS_TRY(get_plan(c, (int)W, nsegs, W, g.cdouble, 0, &fwd));
  PS_CUFFT(cufftSetStream(fwd, st));
  if (g.cdouble)
    PS_CUFFT(cufftExecD2Z(fwd, (cufftDoubleReal*)c->xw.p, (cufftDoubleComplex*)c->spec.p));
  else
    PS_CUFFT(cufftExecR2C(fwd, (cufftReal*)c->xw.p, (cufftComplex*)c->spec.p));
  // ---- per-bin Gram operands (unit = (band, bin), K = R * S segments) ---------
  const size_t plane_bytes = gt.plane_bytes();
  PS_TRY(ensure(c->planes, plane_bytes));
  PS_TRY(ensure(c->maskcount, (size_t)gt.rows * sizeof(int)));
  PS_TRY(reset_status(c, st));
  PS_CUDA(cudaMemsetAsync(c->maskcount.p, 0, (size_t)gt.rows * sizeof(int), st));
  PS_CUDA(launch_coherence_planes(c->spec.p, g.cdouble ? 1 : 0, (int)nbW, g.B, g.R, g.N, (int)nseg, (int)k0, (int)nb,
                                  (int)K, (int)gt.pitch, c->planes.p, gt.plane_stride, gt.split ? 1 : 0, st));
  c->launches += 2;
  if (c->timing) PS_CUDA(cudaEventRecord(c->ev[1], st));
  // ---- Gram + epilogue (COH = "PLV" of the normalised spectra) ----------------
  PS_TRY(plan_call(c, &at, k, {}, /*force_g1=*/false, st));
  PS_TRY(launch_stage(c, k, 0, st));
  if (k.slot_mode == 2) {
    PS_CUDA(launch_group_reduce(c->gws.p, k.G, (int)gt.N, (int)gt.B, 5, k.outs, k.reduce_div, gt.split ? 0 : 1, st,
                                a->out_layout == PS_LAYOUT_UPPER ? 1 : 0));
    for (int m = 0; m < 5; ++m) c->launches += k.outs[m] ? 1 : 0;
  }
  if (c->timing) PS_CUDA(cudaEventRecord(c->ev[2], st));
  ps_status s = read_status(c, st);
  if (s == PS_OK && c->h_status->n_illcond) {
    PS_TRY(refine_range(c, k, 0, c->h_status->n_illcond, st));
    PS_TRY(refresh_status(c, st));
  }
  if (s == PS_OK && w->reduce == PS_BAND_MAX) {
    for (int m = 0; m < 5; ++m)
      if (k.outs[m]) {
        PS_CUDA(launch_band_max(k.outs[m], g.B, nb, nn, user_outs[m], fp64 ? 1 : 0, st,
                                        a->out_layout == PS_LAYOUT_UPPER ? g.N : 0));
        c->launches++;
      }
    PS_CUDA(cudaStreamSynchronize(st));
  }
  if (c->timing) PS_CUDA(cudaEventRecord(c->ev[3], st));
  if (c->timing) PS_CUDA(cudaEventSynchronize(c->ev[3]));
  if (res) {
    std::memset(res, 0, sizeof(*res));
    res->n_observations = K;
    res->n_refined_pairs = (int64_t)c->h_status->n_illcond;
    res->n_indeterminate_ciplv = (int32_t)std::min<unsigned long long>(c->h_status->n_indeterminate, INT32_MAX);
    res->n_kernel_launches = c->launches;
    res->gram_variant = k.g.split ? (k.g.gauss ? 1 : 0) : 2;
    if (c->timing) {
      cudaEventElapsedTime(&res->ms_normalize, c->ev[0], c->ev[1]);
      cudaEventElapsedTime(&res->ms_gram, c->ev[1], c->ev[2]);
      cudaEventElapsedTime(&res->ms_finish, c->ev[2], c->ev[3]);
    }
  }
  return s;
}

ps_status ps_plv_family_staged(ps_ctx* c, const ps_plv_args* a, ps_plv_result* res, int32_t n_stages,
                               const int64_t* stage_cols, void* const* ready_events) {
  clear_stale(__func__);
  if (!c) return fail(PS_E_INVALID, "ctx is NULL");
  std::lock_guard<std::mutex> lock(c->mu);
  Call k;
  PS_TRY(validate(a, k.g));
  PS_TRY(setup_outputs(a, k));
  decide_gauss(a, k);
  const Geometry& g = k.g;
  if (n_stages < 1 || !stage_cols) return fail(PS_E_INVALID, "n_stages must be >= 1 with stage_cols");
  if (a->mode != PS_MODE_OVER_SAMPLES) return fail(PS_E_UNSUPPORTED, "staged input supports mode over_samples only");
  std::vector<long long> cols(stage_cols, stage_cols + n_stages + 1);
  if (cols.front() != 0 || cols.back() != g.N) return fail(PS_E_INVALID, "stage_cols must run from 0 to n_signals");
  for (int s = 0; s < n_stages; ++s) {
    if (cols[s + 1] <= cols[s]) return fail(PS_E_INVALID, "stage_cols must increase");
    if (s > 0 && cols[s] % kSplitBM != 0) return fail(PS_E_INVALID, "interior stage_cols must be multiples of 256");
  }
  PS_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = static_cast<cudaStream_t>(a->stream);
  PS_TRY(ensure_pipeline(c, n_stages));
  c->launches = 0;
  bool copied = false;
  const size_t plane_bytes = g.plane_bytes();
  PS_TRY(ensure(c->planes, plane_bytes));
  PS_TRY(prep_begin(c, a, g, st));  // Hilbert workspace sized once (no realloc mid-stage)
  PS_TRY(reset_status(c, st));
  PS_TRY(init_row_state(c, g, st));
  PS_TRY(plan_call(c, a, k, cols, /*force_g1=*/true, st));
  const long long U = g.B * g.R;
  for (int s = 0; s < n_stages; ++s) {
    if (ready_events && ready_events[s])
      PS_CUDA(cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(ready_events[s]), 0));
    for (long long u = 0; u < U; ++u)
      PS_TRY(prepare_rows(c, a, g, a->input, c->planes.p, g.split ? 0 : 1, g.pitch, g.plane_stride,
                          u * g.N + cols[s], u * g.N + cols[s + 1], st, &copied));
    PS_CUDA(cudaEventRecord(pool_event(c, 3 * s), st));
  }
  // timing: the Gram stages' kernel time only (each stage's start event is
  // recorded after its wait for the input chunk), summed below
  if (c->timing)
    while ((int)c->tev.size() < 2 * n_stages) {
      cudaEvent_t e;
      PS_CUDA(cudaEventCreate(&e));
      c->tev.push_back(e);
    }
  for (int s = 0; s < n_stages; ++s) {
    PS_CUDA(cudaStreamWaitEvent(c->s_comp, pool_event(c, 3 * s), 0));
    if (c->timing) PS_CUDA(cudaEventRecord(c->tev[2 * s], c->s_comp));
    PS_TRY(launch_stage(c, k, s, c->s_comp));
    if (c->timing) PS_CUDA(cudaEventRecord(c->tev[2 * s + 1], c->s_comp));
  }
  cudaEvent_t done = pool_event(c, 3 * n_stages);
  PS_CUDA(cudaEventRecord(done, c->s_comp));
  PS_CUDA(cudaStreamWaitEvent(st, done, 0));
  ps_status s = read_status(c, st);
  if (s == PS_OK && c->h_status->n_illcond) {
    PS_TRY(refine_range(c, k, 0, c->h_status->n_illcond, st));
    PS_TRY(refresh_status(c, st));
  }
  if (res) {
    std::memset(res, 0, sizeof(*res));
    res->n_observations = k.pool ? g.T * g.R : g.T;
    res->n_masked_samples = (int64_t)c->h_status->n_masked;
    res->n_refined_pairs = (int64_t)c->h_status->n_illcond;
    res->n_indeterminate_ciplv = (int32_t)std::min<unsigned long long>(c->h_status->n_indeterminate, INT32_MAX);
    res->input_copied = copied ? 1 : 0;
    res->n_kernel_launches = c->launches;
    res->gram_variant = k.g.split ? (k.g.gauss ? 1 : 0) : 2;
    if (c->timing) {
      PS_CUDA(cudaEventSynchronize(done));
      float tot = 0.f;
      for (int q = 0; q < n_stages; ++q) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c->tev[2 * q], c->tev[2 * q + 1]);
        tot += ms;
      }
      res->ms_gram = tot;
    }
  }
  return s;
}

}  // extern "C"

namespace {

// E2E host path for multi-trial trial-mean calls (B x R units of N rows each,
// e.g. C2 / C4): pipelined over trials instead of signal stages.  The trial
// groups (partial-sum slots of Rg trials) come from the device path's cost
// model; a stage is a run of groups of one band holding ~384 MB of input.
// Stage s+1's units cross the link (copy stream) while stage s's units are
// normalised (prep stream) and stage s-1's Gram items accumulate their groups'
// partial metric sums (compute stream).  The trial-group reduction, the FP64
// refinement and the copy-out of the B small matrices per metric finish the
// call, which then runs at the host link's rate.
ps_status host_unit_pipelined(ps_ctx* c, const ps_plv_args* a, Call& k, long long span, long long esz,
                              ps_plv_result* res, bool dev_input) {
  const Geometry& g = k.g;
  PS_TRY(ensure_pipeline(c, 1));
  cudaStream_t si = c->s_in, sn = c->s_ref, sc = c->s_comp;
  for (cudaStream_t q : {si, sc, sn, c->s_out}) PS_CUDA(cudaStreamSynchronize(q));
  c->launches = 0;
  bool copied = false;
  if (!dev_input) PS_TRY(ensure(c->hin, (size_t)span * esz));
  const size_t plane_bytes = g.plane_bytes();
  PS_TRY(ensure(c->planes, plane_bytes));
  const size_t oes = g.split ? 4 : 8;
  void* houts[5];
  std::memcpy(houts, k.outs, sizeof(houts));
  int nout = 0;
  for (int m = 0; m < 5; ++m) nout += houts[m] ? 1 : 0;
  const size_t out_bytes = (size_t)g.B * g.N * g.N * oes;
  PS_TRY(ensure(c->hout, out_bytes * std::max(nout, 1)));
  {
    int q = 0;
    for (int m = 0; m < 5; ++m) k.outs[m] = houts[m] ? static_cast<char*>(c->hout.p) + (size_t)(q++) * out_bytes : nullptr;
  }
  if (dev_input) {  // the caller's stream order makes the input valid
    cudaEvent_t ready = pool_event(c, 0);
    PS_CUDA(cudaEventRecord(ready, static_cast<cudaStream_t>(a->stream)));
    PS_CUDA(cudaStreamWaitEvent(si, ready, 0));
  }
  PS_TRY(prep_begin(c, a, g, si));
  PS_TRY(reset_status(c, si));
  PS_TRY(init_row_state(c, g, si));
  PS_TRY(plan_call(c, a, k, {}, /*force_g1=*/false, si));
  const int G = k.G, Rg = k.Rg;
  const double unit_bytes = (double)g.N * (double)g.T * (double)esz;
  const int gps = std::max(1, std::min(G, (int)std::lround(384.0 * (1 << 20) / (Rg * unit_bytes))));
  // items run (band, group, tile): stage boundaries where the band or the
  // group run changes
  struct Stage {
    long long b, t0, t1;
  };
  std::vector<Stage> stages;
  {
    std::vector<int> off(1, 0);
    const std::vector<Item>& it = c->h_items;
    for (size_t n = 0; n < it.size(); ++n) {
      const bool start = n == 0 || it[n].b != it[n - 1].b || it[n].g / gps != it[n - 1].g / gps;
      if (!start) continue;
      if (n > 0) off.push_back((int)n);
      const long long t0 = (long long)(it[n].g / gps) * gps * Rg;
      stages.push_back(Stage{it[n].b, t0, std::min<long long>(g.R, t0 + (long long)gps * Rg)});
    }
    off.push_back((int)it.size());
    k.stage_off = off;
  }
  const int S = (int)stages.size();
  PS_TRY(ensure_pipeline(c, S));
  const bool upper = a->out_layout == PS_LAYOUT_UPPER;
  if (upper || k.slot_mode != 2)  // outputs copied whole: the lower triangle must read 0
    PS_CUDA(cudaMemsetAsync(c->hout.p, 0, out_bytes * std::max(nout, 1), si));
  ps_plv_args d = *a;
  void* din = dev_input ? const_cast<void*>(a->input) : c->hin.p;
  d.input = din;
  size_t h2d_bytes = 0;
  static const bool want_trace = std::getenv("PS_PIPE_TRACE") != nullptr;
  std::unique_ptr<PipeTrace> trace_holder(want_trace ? new PipeTrace(si) : nullptr);
  PipeTrace* trace = trace_holder.get();
  for (int s = 0; s < S; ++s) {
    const Stage& sg = stages[(size_t)s];
    for (long long t = sg.t0; t < sg.t1 && !dev_input; ++t) {
      const long long off = sg.b * a->stride_band + t * a->stride_trial;
      const long long len = (g.N - 1) * a->stride_signal + (g.T - 1) * a->stride_sample + 1;
      PS_CUDA(cudaMemcpyAsync(static_cast<char*>(c->hin.p) + off * esz, static_cast<const char*>(a->input) + off * esz,
                              (size_t)len * esz, cudaMemcpyHostToDevice, si));
      h2d_bytes += (size_t)len * esz;
    }
    if (trace) trace->rec(si, "h2d", s);
    PS_CUDA(cudaEventRecord(pool_event(c, 3 * s + 1), si));
    PS_CUDA(cudaStreamWaitEvent(sn, pool_event(c, 3 * s + 1), 0));
    for (long long t = sg.t0; t < sg.t1; ++t) {
      const long long u = sg.b * g.R + t;
      PS_TRY(prepare_rows(c, &d, g, din, c->planes.p, g.split ? 0 : 1, g.pitch, g.plane_stride, u * g.N,
                          (u + 1) * g.N, sn, &copied));
    }
    if (trace) trace->rec(sn, "norm", s);
    PS_CUDA(cudaEventRecord(pool_event(c, 3 * s + 2), sn));
    PS_CUDA(cudaStreamWaitEvent(sc, pool_event(c, 3 * s + 2), 0));
    PS_TRY(launch_stage(c, k, s, sc));
    if (trace) trace->rec(sc, "gram", s);
  }
  if (k.slot_mode == 2) {
    PS_CUDA(launch_group_reduce(c->gws.p, k.G, (int)g.N, (int)g.B, 5, k.outs, k.reduce_div, g.split ? 0 : 1, sc,
                                upper ? 1 : 0));
    for (int m = 0; m < 5; ++m) c->launches += k.outs[m] ? 1 : 0;
  }
  ps_status st = read_status(c, sc);
  if (st == PS_OK && c->h_status->n_illcond) {
    PS_TRY(refine_range(c, k, 0, c->h_status->n_illcond, sc));
    PS_TRY(refresh_status(c, sc));
  }
  size_t d2h_bytes = 0;
  for (int m = 0; m < 5 && st == PS_OK; ++m)
    if (houts[m]) {
      PS_CUDA(cudaMemcpyAsync(houts[m], k.outs[m], out_bytes, cudaMemcpyDeviceToHost, sc));
      d2h_bytes += out_bytes;
    }
  if (trace) trace->rec(sc, "d2h", S - 1);
  PS_CUDA(cudaStreamSynchronize(sc));
  if (trace) trace->dump();
  if (res) {
    std::memset(res, 0, sizeof(*res));
    res->n_observations = g.T;
    res->n_masked_samples = (int64_t)c->h_status->n_masked;
    res->n_refined_pairs = (int64_t)c->h_status->n_illcond;
    res->n_indeterminate_ciplv = (int32_t)std::min<unsigned long long>(c->h_status->n_indeterminate, INT32_MAX);
    res->input_copied = copied ? 1 : 0;
    res->n_kernel_launches = c->launches;
    res->gram_variant = k.g.split ? (k.g.gauss ? 1 : 0) : 2;
    res->h2d_bytes = (int64_t)h2d_bytes;
    res->d2h_bytes = (int64_t)d2h_bytes;
  }
  std::memcpy(k.outs, houts, sizeof(houts));
  return st;
}

// Host-output calls: outputs land in the caller's host arrays.  dev_input:
// the input is device memory (ready in a->stream's order) -- no copy-in.
ps_status host_output_call(ps_ctx* c, const ps_plv_args* a, ps_plv_result* res, bool dev_input) {
  if (!c) return fail(PS_E_INVALID, "ctx is NULL");
  // c->hin / c->hout are per-context staging buffers: the lock covers their
  // sizing, the copy-in, the compute and the copy-out (concurrent callers on
  // one context serialise instead of sharing the buffers)
  std::lock_guard<std::mutex> lock(c->mu);
  Call k;
  PS_TRY(validate(a, k.g));
  PS_TRY(setup_outputs(a, k));
  decide_gauss(a, k);
  const Geometry& g = k.g;
  PS_CUDA(cudaSetDevice(c->device));
  // span of the (possibly strided) host input, in elements
  const long long esz = (a->dtype == PS_F32) ? 4 : (a->dtype == PS_F64 || a->dtype == PS_C64) ? 8 : 16;
  long long span = 1;
  const long long dims[4] = {g.B, g.N, g.T, g.R};
  const long long strides[4] = {a->stride_band, a->stride_signal, a->stride_sample, a->stride_trial};
  for (int q = 0; q < 4; ++q) {
    if (dims[q] > 1 && strides[q] < 0) return fail(PS_E_INVALID, "negative strides are not supported");
    span += (dims[q] - 1) * strides[q];
  }
  // Pipelined (copy-in / compute / copy-out overlapped) when the signal rows
  // of each unit are contiguous spans and there are enough tiles to fill the
  // GPU with one trial group.
  static const bool no_pipe = std::getenv("PS_NO_PIPELINE") != nullptr;
  const long long ntiles = ps_tile_count(g.N, a->precision);
  // sharded calls pipeline on the streamed (upper layout) path only: each
  // shard then owns whole row bands and ships just those rows
  const bool streamed = a->out_layout == PS_LAYOUT_UPPER && std::getenv("PS_PIPE_NO_STREAM") == nullptr;
  const bool pipelinable = !no_pipe && a->mode == PS_MODE_OVER_SAMPLES && (k.shard_count == 1 || streamed) &&
                           a->stride_sample == 1 && a->stride_signal >= g.T &&
                           g.N >= 2048 && ntiles * g.B >= c->num_sms;
  // multi-trial trial means with a large input: pipelined over trial groups
  static const long long unit_min = [] {
    const char* e = std::getenv("PS_UNIT_PIPE_MIN_MB");  // threshold (MB of input)
    return (e ? std::atoll(e) : 512LL) << 20;
  }();
  const bool unit_pipelinable = !no_pipe && a->mode == PS_MODE_OVER_SAMPLES && k.shard_count == 1 &&
                                (a->trial_reduce == PS_TRIALS_MEAN || a->trial_reduce == PS_TRIALS_SUM) && g.R > 1 &&
                                a->stride_sample == 1 &&
                                a->stride_signal >= g.T && span * esz >= unit_min;
  if (unit_pipelinable) return host_unit_pipelined(c, a, k, span, esz, res, dev_input);
  if (pipelinable) return host_pipelined(c, a, k, span, esz, res, dev_input);
  cudaStream_t st = static_cast<cudaStream_t>(a->stream);
  if (!dev_input) {
    PS_TRY(ensure(c->hin, (size_t)span * esz));
    PS_CUDA(cudaMemcpyAsync(c->hin.p, a->input, (size_t)span * esz, cudaMemcpyHostToDevice, st));
  }
  const bool pool = a->trial_reduce == PS_TRIALS_POOL;
  const long long slots = a->mode == PS_MODE_OVER_TRIALS ? g.B * g.T
                          : (a->trial_reduce == PS_TRIALS_NONE && !pool) ? g.B * g.R
                                                                       : g.B;
  const size_t oes = g.split ? 4 : 8;
  const size_t out_bytes = (size_t)slots * g.N * g.N * oes;
  void* houts[5] = {a->out_plv, a->out_iplv, a->out_ciplv, a->out_cre, a->out_cim};
  int nout = 0;
  for (int m = 0; m < 5; ++m)
    if (((a->metrics >> m) & 1u) && houts[m]) ++nout;
  PS_TRY(ensure(c->hout, out_bytes * std::max(nout, 1)));
  ps_plv_args d = *a;
  d.input = dev_input ? a->input : c->hin.p;
  void** douts[5] = {&d.out_plv, &d.out_iplv, &d.out_ciplv, &d.out_cre, &d.out_cim};
  int q = 0;
  for (int m = 0; m < 5; ++m) {
    if (((a->metrics >> m) & 1u) && houts[m]) *douts[m] = static_cast<char*>(c->hout.p) + (size_t)(q++) * out_bytes;
    else *douts[m] = nullptr;
  }
  // the whole-matrix copy-out carries the entries this call does not write --
  // the lower triangle (upper layout) or other shards' tiles (sharded call):
  // they must arrive as 0, never as a previous call's values in the reused
  // staging buffer
  if (a->out_layout == PS_LAYOUT_UPPER || k.shard_count > 1) PS_CUDA(cudaMemsetAsync(c->hout.p, 0, out_bytes * q, st));
  ps_status s = plv_family_locked(c, &d, res);
  if (s != PS_OK) return s;
  q = 0;
  for (int m = 0; m < 5; ++m)
    if (((a->metrics >> m) & 1u) && houts[m])
      PS_CUDA(cudaMemcpyAsync(houts[m], static_cast<char*>(c->hout.p) + (size_t)(q++) * out_bytes, out_bytes,
                              cudaMemcpyDeviceToHost, st));
  PS_CUDA(cudaStreamSynchronize(st));
  if (res) {
    res->h2d_bytes = dev_input ? 0 : (int64_t)span * esz;
    res->d2h_bytes = (int64_t)out_bytes * q;
  }
  return PS_OK;
}

}  // namespace

extern "C" {

ps_status ps_plv_family_host(ps_ctx* c, const ps_plv_args* a, ps_plv_result* res) {
  clear_stale(__func__);
  return host_output_call(c, a, res, /*dev_input=*/false);
}

ps_status ps_plv_family_to_host(ps_ctx* c, const ps_plv_args* a, ps_plv_result* res) {
  clear_stale(__func__);
  return host_output_call(c, a, res, /*dev_input=*/true);
}

ps_status ps_analytic_signal(ps_ctx* c, const ps_plv_args* a0, void* out) {
  clear_stale(__func__);
  if (!c) return fail(PS_E_INVALID, "ctx is NULL");
  if (!out) return fail(PS_E_INVALID, "out is NULL");
  std::lock_guard<std::mutex> lock(c->mu);
  ps_plv_args a = *a0;
  a.input_kind = PS_INPUT_REAL;
  a.precision = PS_PREC_SPLIT_F16X3;  // compute type follows the input dtype
  Geometry g;
  PS_TRY(validate(&a, g));
  PS_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = static_cast<cudaStream_t>(a.stream);
  SrcDesc src = make_src(&a, g, a.input);
  bool copied = false;
  PS_TRY(reset_status(c, st));
  PS_TRY(prep_begin(c, &a, g, st));
  const long long rc = prep_chunk_rows(&a, g);
  const size_t es = g.cdouble ? 8 : 4;
  for (long long row0 = 0; row0 < g.rows; row0 += rc) {
    const long long nr = std::min(rc, g.rows - row0);
    SrcDesc s = src;
    if (a.fir) {
      PS_TRY(bandpass_chunk(c, &a, g, src, row0, nr, true, st, &s));
    } else {
      PS_TRY(hilbert_chunk(c, &a, g, src, row0, nr, st, &copied, &s.h_scale));
      s.hbuf = c->hbuf.p;
      s.h_row0 = row0;
    }
    PS_CUDA(launch_analytic_out(s, row0, nr, static_cast<char*>(out) + (size_t)row0 * g.T * 2 * es, st));
  }
  return read_status(c, st);
}

ps_status ps_filter_two_pass(ps_ctx* c, const ps_plv_args* a0, void* out) {
  clear_stale(__func__);
  if (!c) return fail(PS_E_INVALID, "ctx is NULL");
  if (!out) return fail(PS_E_INVALID, "out is NULL");
  if (!a0 || !a0->fir) return fail(PS_E_INVALID, "args->fir is required");
  std::lock_guard<std::mutex> lock(c->mu);
  ps_plv_args a = *a0;
  a.input_kind = PS_INPUT_REAL;
  a.precision = PS_PREC_SPLIT_F16X3;  // compute type follows the input dtype
  Geometry g;
  PS_TRY(validate(&a, g));
  PS_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = static_cast<cudaStream_t>(a.stream);
  const SrcDesc src = make_src(&a, g, a.input);
  PS_TRY(prep_begin(c, &a, g, st));
  const FirGeom f = fir_geom(&a, g);
  const long long rc = prep_chunk_rows(&a, g);
  const size_t es = g.cdouble ? 8 : 4;
  for (long long row0 = 0; row0 < g.rows; row0 += rc) {
    const long long nr = std::min(rc, g.rows - row0);
    SrcDesc s;
    PS_TRY(bandpass_chunk(c, &a, g, src, row0, nr, false, st, &s));
    PS_CUDA(launch_trim_rows(c->xw.p, nr, f.Lf, f.P, g.T, static_cast<char*>(out) + (size_t)row0 * g.T * es,
                             g.cdouble ? 1 : 0, st));
  }
  PS_CUDA(cudaStreamSynchronize(st));
  return PS_OK;
}

ps_status ps_normalize_phasors(ps_ctx* c, const ps_plv_args* a, void* out, uint8_t* mask_out) {
  clear_stale(__func__);
  if (!c) return fail(PS_E_INVALID, "ctx is NULL");
  if (!out) return fail(PS_E_INVALID, "out is NULL");
  std::lock_guard<std::mutex> lock(c->mu);
  ps_plv_args aa = *a;
  aa.precision = PS_PREC_SPLIT_F16X3;  // compute type follows the input dtype
  Geometry g;
  PS_TRY(validate(&aa, g));
  PS_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = static_cast<cudaStream_t>(aa.stream);
  bool copied = false;
  PS_TRY(reset_status(c, st));
  PS_TRY(prepare_phasors(c, &aa, g, aa.input, out, 2, g.T, 0, st, &copied));
  ps_status s = read_status(c, st);
  if (s != PS_OK) return s;
  if (mask_out) {
    // masked samples are exactly 0+0i; unmasked unit phasors never are
    const size_t n = (size_t)g.rows * g.T;
    PS_CUDA(ps_mask_from_zero(out, g.cdouble ? 1 : 0, n, mask_out, st));
    PS_CUDA(cudaStreamSynchronize(st));
  }
  return PS_OK;
}

}  // extern "C"

