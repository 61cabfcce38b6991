/*
 * truncmul_b200 — C ABI of the B200-native full / low / high integer products.
 *
 * This is the drop-in boundary for the reference's product entry points
 * (arxiv 1703.00640 artifact, /root/reference/proj/core):
 *
 *   products.hpp:25-34   struct Params          -> tmg_params
 *   products.hpp:39-40   required_precision     -> tmg_required_precision
 *   products.hpp:42-45   default_lambda         -> tmg_default_lambda
 *   products.hpp:47-53   validate_params        -> tmg_validate_params
 *   products.hpp:55-62   select_params          -> tmg_select_params
 *   products.hpp:91-93   full_product / low_product / high_product
 *                        -> tmg_full_product / tmg_low_product /
 *                           tmg_high_product  (host limb arrays)
 *                        -> tmg_product_device  (device-resident limbs)
 *   errors.hpp:9-67      exception classes  -> TMG_ERR_* return codes
 *
 * Operands and results are little-endian arrays of 64-bit limbs (the
 * reference's BigInt::to_limbs / from_limbs, bigint.hpp:113-115).  Operands
 * hold ceil(n/64) limbs; results hold tmg_output_limbs(mode, n) limbs:
 *   full: ceil(2n/64)   low: ceil(n/64)   high: ceil((n+1)/64)
 *
 * Every function returns TMG_OK (0) or a TMG_ERR_* code; tmg_last_error()
 * gives the message of the calling thread's last failure.  No function
 * throws across the ABI.  There is no CPU fallback: products run on the GPU
 * and fail with TMG_ERR_CUDA when no device is usable.
 */
#ifndef TRUNCMUL_B200_H_
#define TRUNCMUL_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mode (products.hpp:14) */
enum {
  TMG_MODE_FULL = 0,
  TMG_MODE_LOW = 1,
  TMG_MODE_HIGH = 2,
  TMG_MODE_ORACLE_FALLBACK = 3
};

/* Backend (convolution.hpp:12).  Only the FFT backend is implemented on the
 * GPU; EXACT parameter sets are accepted by the parameter functions and
 * refused by the product functions with TMG_ERR_UNSUPPORTED. */
enum { TMG_BACKEND_EXACT = 0, TMG_BACKEND_FFT = 1 };

/* Parameter selection policy.  REFERENCE reproduces params.cpp exactly;
 * ACCURATE additionally bounds the predicted rounding error of an FP64 FFT
 * below the 0.25 tripwire and ranks lengths by GPU cost. */
enum { TMG_POLICY_REFERENCE = 0, TMG_POLICY_ACCURATE = 1 };

/* Error codes (errors.hpp) */
enum {
  TMG_OK = 0,
  TMG_ERR_INPUT_OUT_OF_RANGE = 1,   /* InputOutOfRange */
  TMG_ERR_NO_VALID_PARAMS = 2,      /* NoValidParams */
  TMG_ERR_UNSUPPORTED_LENGTH = 3,   /* UnsupportedLength */
  TMG_ERR_PRECISION_FAILURE = 4,    /* ConvolutionPrecisionFailure */
  TMG_ERR_PLAN_MISMATCH = 5,        /* PlanMismatch */
  TMG_ERR_UNSUPPORTED = 6,          /* parameter set the GPU path refuses */
  TMG_ERR_CUDA = 7,                 /* CUDA runtime failure / no device */
  TMG_ERR_INTERNAL = 8
};

/* Params (products.hpp:25-34) */
typedef struct tmg_params {
  int64_t n;
  int32_t b;
  int64_t N;
  int64_t lambda;
  int32_t p;
  int32_t mode;
  int32_t backend;
  int32_t signed_split;
} tmg_params;

/* Per-product statistics filled by the product functions. */
typedef struct tmg_stats {
  double max_round_err; /* max distance of a pre-rounding value to an integer */
  double max_abs;       /* max magnitude of a pre-rounding value */
  uint32_t flags;       /* raw device flag word */
  int64_t transform_length;
  int32_t passes;       /* 1 = fused single CTA, 2 or 3 = multi-pass */
  int32_t kernels;      /* kernels launched for the product */
  int32_t attempts;     /* 1, or 2+ after escalation */
  int32_t b;            /* chunk width of the attempt that produced the result */
  int64_t N;            /* chunk count of that attempt */
  double first_round_err; /* residual of the first attempt (tripwire value) */
} tmg_stats;

/* stats.flags bit: the product was recomputed at a lower chunk width after
 * the first attempt refused (see tmg_context_set_escalation). */
#define TMG_STAT_ESCALATED (1u << 24)

typedef struct tmg_context tmg_context;

const char* tmg_last_error(void);
const char* tmg_version(void);

/* ---- parameters (host only; no GPU needed) ---- */
int tmg_required_precision(int32_t mode, int32_t b, int64_t N, int32_t* out);
int tmg_default_lambda(int32_t mode, int32_t backend, int32_t b, int32_t p,
                       int64_t* out);
int tmg_validate_params(const tmg_params* params);
int tmg_select_params(int64_t n, int32_t mode, int32_t backend,
                      int64_t fallback_cutoff, int32_t policy,
                      tmg_params* out);
int64_t tmg_output_limbs(int32_t mode, int64_t n);
/* Predicted standard deviation of the FP64 rounding error (policy model). */
double tmg_predicted_sigma(const tmg_params* params);

/* ---- context ---- */
int tmg_context_create(int device, tmg_context** out);
void tmg_context_destroy(tmg_context* ctx);
/* Optional: run subsequent work on a caller-owned cudaStream_t. */
int tmg_context_set_stream(tmg_context* ctx, void* stream);
int tmg_synchronize(tmg_context* ctx);

/* ---- products on host limb arrays (H2D, kernels, D2H inside) ----
 * params must be an FFT-backend parameter set of the matching mode, or an
 * ORACLE_FALLBACK set (operands below the cutoff: GPU schoolbook product). */
int tmg_full_product(tmg_context* ctx, const tmg_params* params,
                     const uint64_t* u, const uint64_t* v, uint64_t* out,
                     tmg_stats* stats);
int tmg_low_product(tmg_context* ctx, const tmg_params* params,
                    const uint64_t* u, const uint64_t* v, uint64_t* out,
                    tmg_stats* stats);
int tmg_high_product(tmg_context* ctx, const tmg_params* params,
                     const uint64_t* u, const uint64_t* v, uint64_t* out,
                     tmg_stats* stats);

/* Batched: count independent products of the same params; operands and
 * results are packed back to back.  flags_out (optional, count words)
 * receives each product's device flag word. */
int tmg_product_batched(tmg_context* ctx, const tmg_params* params,
                        const uint64_t* u, const uint64_t* v, int64_t count,
                        uint64_t* out, uint32_t* flags_out, tmg_stats* stats);

/* ---- the ring-change maps on their own (maps_f64.hpp: alpha_star_f64,
 * beta_star_f64, gamma_dagger_f64, delta_dagger_f64 on the tables of
 * build_map_tables_f64(N, b, lambda, ..); maps_f64.cpp:245-384) ----
 * Host arrays of doubles.  alpha*: N -> N and beta*: N -> N (low product);
 * gamma-dagger: N + 1 -> N, *aux receives the root channel, and
 * delta-dagger: N and aux -> N + 1 (high product).  lambda <= 8 and
 * N >= 2 lambda + 2; the high-mode maps need N b >= 64 (power-of-two root).
 * The series coefficients are computed on the fly from the closed forms of
 * series.cpp:146-183, so results agree with the table-driven reference to a
 * few ulps of the largest term, not bit for bit. */
int tmg_alpha_star_f64(tmg_context* ctx, int64_t N, int32_t b, int64_t lambda,
                       const double* in, double* out);
int tmg_beta_star_f64(tmg_context* ctx, int64_t N, int32_t b, int64_t lambda,
                      const double* in, double* out);
int tmg_gamma_dagger_f64(tmg_context* ctx, int64_t N, int32_t b, int64_t lambda,
                         const double* in, double* out, double* aux);
int tmg_delta_dagger_f64(tmg_context* ctx, int64_t N, int32_t b, int64_t lambda,
                         const double* in, double aux, double* out);

/* ---- the FP64 cyclic convolution on its own (convolution.hpp:64-67,
 * cyclic_convolve_f64 on an FFT plan of length n: make_plan(n, p, kFft)) ----
 * out[k] = sum_j f[j] g[(k - j) mod n] for host arrays of n doubles; out may
 * not alias f or g.  n must be {2,3,5,7}-smooth (TMG_ERR_UNSUPPORTED_LENGTH
 * with make_plan's message otherwise, convolution.cpp:92-105).  Lengths above
 * 4096 run the products' transform passes and must be multiples of 4 (every
 * length select_params picks is); shorter ones, and other lengths up to
 * 32768, are summed directly.  Three-pass lengths (above 4096 x 2048) whose
 * column part has no factorisation A x B with 4 | A and both at most 2048 --
 * lengths with very few factors of two, e.g. 2^2 3 5^9 -- are refused with
 * TMG_ERR_UNSUPPORTED_LENGTH as well. */
int tmg_cyclic_convolve_f64(tmg_context* ctx, int64_t n, const double* f,
                            const double* g, double* out);

/* ---- the splitters on their own (products.hpp:68-79, split.cpp:147-158) ----
 * split_low_i64: out receives params->N chunks of params->b bits of u
 * (ceil(n/64) host limbs), u = sum_i out[i] 2^{i b}; with signed_split the
 * chunks below the top lie in (-2^{b-1}, 2^{b-1}] and the top one absorbs the
 * carries.  split_high_i64: the N + 1 chunks of u 2^sigma,
 * sigma = (N + 1) b - n (top-aligned; needs (N+1) b >= n + lg N + 2).
 * Only n, b, N and signed_split of params are read, like the reference.
 * TMG_ERR_INPUT_OUT_OF_RANGE with the reference's messages for b > 62, a
 * covering violation, or an operand outside [0, 2^n). */
int tmg_split_low_i64(tmg_context* ctx, const tmg_params* params,
                      const uint64_t* u, int64_t* out);
int tmg_split_high_i64(tmg_context* ctx, const tmg_params* params,
                       const uint64_t* u, int64_t* out);

/* ---- device-resident variants (enqueue only; no host synchronisation) ----
 * d_u, d_v, d_out are device pointers.  Errors detected on the device are
 * reported by the next tmg_check(). */
int tmg_product_device(tmg_context* ctx, const tmg_params* params,
                       const uint64_t* d_u, const uint64_t* d_v,
                       uint64_t* d_out, int64_t count);
int tmg_check(tmg_context* ctx, tmg_stats* stats);

/* Pinned host buffers for the end-to-end path. */
int tmg_host_alloc(size_t bytes, void** out);
void tmg_host_free(void* p);
int tmg_device_alloc(size_t bytes, void** out);
void tmg_device_free(void* p);
int tmg_memcpy_h2d(tmg_context* ctx, void* dst, const void* src, size_t bytes);
int tmg_memcpy_d2h(tmg_context* ctx, void* dst, const void* src, size_t bytes);

/* Escalation (default 0 = off, the reference's behaviour): when the float
 * pipeline of a single host-buffer product refuses (rounding tripwire,
 * overflow, recombination check -- TMG_ERR_PRECISION_FAILURE), recompute it
 * at chunk width b - 1 with a fresh N and lambda, up to max_escalations
 * times.  Structured operands (long runs of equal limbs) concentrate the
 * spectrum and can exceed the random-input error model the parameters are
 * chosen by (paper section 5); escalation turns that refusal into an exact
 * result.  Batched and device-pointer calls never escalate. */
int tmg_context_set_escalation(tmg_context* ctx, int max_escalations);

/* Kernels launched by the last product call (for launch accounting). */
int32_t tmg_last_kernel_count(tmg_context* ctx);

/* Per-kernel CUDA-event timing on the context stream.  When enabled every
 * launch is bracketed by events; tmg_profile_read synchronises, returns up to
 * max_records (name, milliseconds, algorithmic bytes) and clears the log.
 * names receives max_records strings of name_stride bytes each. */
int tmg_profile_enable(tmg_context* ctx, int on);
int tmg_profile_read(tmg_context* ctx, char* names, int name_stride, double* ms,
                     double* bytes, int max_records, int* count);

/* ---- testing and diagnostics ----
 * Alternative code paths a context can select so that tests reach them
 * (none is needed in normal use; every default is the measured-best
 * configuration, and the library reads nothing from the environment).
 * Setting an option synchronises the context and drops its cached plans. */
enum {
  TMG_OPT_GENERIC_COLUMN_PASSES = 1, /* runtime-dispatched column passes, not the compiled shapes */
  TMG_OPT_FORCE_THREE_PASS = 2,      /* three-pass plans for short column lengths (>= 64) */
  TMG_OPT_GENERIC_ROW_PASS = 3,      /* generic row pass instead of the compiled C = 4096 one */
  TMG_OPT_LOOKBACK_CARRY = 4,        /* single-pass decoupled look-back carry (k_carry + k_high_agg);
                                        the default path uses it only beyond 2^32 carry bits */
  TMG_OPT_PATCH_SCAN_MAX = 5,        /* most carry blocks k_carry_patch scans itself (default 4096;
                                        above, the last k_carry_lanes block scans them) */
  TMG_OPT_NO_PDL = 6,                /* launches without programmatic dependent launch */
  TMG_OPT_DEBUG_SYNC = 7,            /* synchronise and check after every launch */
  TMG_OPT_NO_GRAPH = 8,              /* multi-pass batches always enqueued eagerly */
  TMG_OPT_Z_NATURAL = 9,             /* pre-mapped coefficients stored in natural order */
  TMG_OPT_GENERIC_SMALL = 10,        /* runtime-dispatched stages in the fused small-product kernel */
  TMG_OPT_PREMAP_IN_SPLIT = 11       /* the split kernel applies the pre-map and stores 16-byte
                                        coefficients (default: it stores digits and the first
                                        column pass pre-maps, where a compiled shape allows) */,
  TMG_OPT_CARRY_KERNELS = 12         /* 1: single-pass look-back carry (k_carry_lb); 2: carry-ins by
                                        a second kernel, per-limb lanes (k_carry_lanes +
                                        k_carry_patch); 3: the same with the runs kernel
                                        (k_carry_runs + k_carry_patch) at every size; 0 (default):
                                        one kernel while the carry blocks fit one wave, else
                                        k_carry_runs + k_carry_patch */,
  TMG_OPT_MAX_ROW = 13,               /* longest row length C of multi-pass plans (0: 4096) */
  TMG_OPT_SPLIT_AGGREGATES = 14,     /* the split's block carry-ins always from k_zstat's aggregates
                                        (default: a look-back inside k_zgen) */
  TMG_OPT_GENERIC_RUNS = 15,         /* k_carry_runs with the chunk width as a run-time value
                                        (default: a compiled width where one exists) */
  TMG_OPT_SPLIT_KERNEL = 16          /* 1: the block-scan split k_zgen at every size (default: the
                                        split by runs, k_zsplit, for large products) */
};
int tmg_context_set_option(tmg_context* ctx, int32_t option, int64_t value);

/* Copies the last single product's pre-mapped coefficients (which = 0; in
 * natural order under TMG_OPT_Z_NATURAL) or convolution coefficients
 * (which = 1) to host memory; *bytes is the buffer size in, the bytes
 * copied out. */
int tmg_debug_read(tmg_context* ctx, int which, void* host, size_t* bytes);

#ifdef __cplusplus
}
#endif

#endif /* TRUNCMUL_B200_H_ */
