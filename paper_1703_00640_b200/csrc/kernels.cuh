// Kernel argument blocks and declarations.
#pragma once

#include "common.cuh"
#include "digits.cuh"
#include "fft_smem.cuh"
#include "pipeline.cuh"

namespace tmg {

// Transform lengths up to this run as one fused CTA per product.
constexpr int64_t kSmallMaxL = 8192;
constexpr int64_t kSmallSingleMaxL = 4096;  // single products above: multi-pass (plan.cu)
// Batches of products up to this length (that fit one CTA's shared memory)
// run the fused single-CTA kernel, one CTA per product, instead of a
// multi-pass chain per product (plan.small_batch).
constexpr int64_t kSmallBatchMaxL = 12288;
constexpr int kSmallBatchMaxThreads = 768;
constexpr int64_t kSmallBatchMinCount = 8;

struct SmallArgs {
  const uint64_t* u;  // batch of operands, nlimbs words each
  const uint64_t* v;
  uint64_t* out;      // batch of outputs, out_limbs words each
  uint32_t* pflags;   // per-product flag words (may be null)
  int64_t nlimbs;
  int64_t n;
  int64_t out_limbs;
  int64_t L;      // transform length
  int64_t count;  // chunks per operand
  int64_t lead;   // high split shift sigma
  int64_t K;      // recombination coefficients
  int64_t ML;     // limbs scanned
  int32_t shift_s;
  double scale, scale_lo;  // 1 / (4 L) as hi + lo
  SubFft fwd;     // length L
  SubFft inv;     // length L / 2
  MapConsts mc;
  DevStatus* status;
};

size_t small_smem_bytes(int64_t L, int64_t nlimbs);
// opt-in dynamic shared memory per CTA on sm_100 (227 KB)
constexpr size_t kMaxDynSmem = 232448;
size_t mid_smem_bytes(uint32_t C, uint32_t inv_stablen);
size_t col_smem_bytes(uint32_t R, uint32_t c);

__global__ void k_small_product(const __grid_constant__ SmallArgs a);
__global__ void k_small_product_2(const __grid_constant__ SmallArgs a);  // <= 384 threads, 2 CTAs per SM
__global__ void k_small_product_big(const __grid_constant__ SmallArgs a);  // <= 768 threads (batched L <= 12288)
// compile-time schedules for the full product at 2^16 bits (768 threads)
__global__ void k_small_6144(const __grid_constant__ SmallArgs a);
// compile-time schedules for the low / high products at 2^16 bits (384 threads)
__global__ void k_small_5120(const __grid_constant__ SmallArgs a);

// ---------------------------------------------------------------------------
// Multi-pass pipeline.  The complex transform of length L = A * B * C runs as
// column passes over A (and B) and a row pass over C (the "mid" kernel, which
// also forms the spectral product and starts the inverse).

struct ScanState {
  unsigned long long* state;  // per-block look-back words
  unsigned long long* ctr;    // [0] ticket, [1] done
  uint32_t epoch;
};

// Column pass geometry: element (outer, row, col) at
//   outer * os + row * rs + (col / cw) * cs + (col % cw)
struct ColGeom {
  int64_t os, rs, cs;
  uint32_t cw;
  uint32_t ncols;  // columns per outer matrix
};

// Layout of the pre-mapped coefficients z (N entries): element
// j = row * ncols + col sits in the tile of k_f1's CTA that owns col --
// tiles of 2^logc columns x zrows rows, row-major inside the tile -- so the
// first column pass reads its whole tile contiguously.  zrows = ceil(N /
// ncols) (the full product's upper half is zero and not stored).  natural
// keeps z[j] at j (diagnostics).
struct ZTile {
  FastDiv fdcols;  // division by ncols
  uint32_t logc;
  uint32_t zrows;
  uint32_t natural;
  __device__ __forceinline__ uint32_t index(uint32_t j) const {
    if (natural) return j;
    const uint32_t row = fdiv(j, fdcols);
    const uint32_t col = j - row * fdcols.d;
    return ((col >> logc) * zrows + row) * (1u << logc) + (col & ((1u << logc) - 1));
  }
};

// Balanced split + pre-map of both operands (k_zgen.cu).
struct ZgenArgs {
  const uint64_t* u;
  const uint64_t* v;
  int64_t nlimbs;
  int64_t n;
  int32_t b;
  int64_t count;  // chunks per operand (N, or N + 1 for the high split)
  int64_t N;      // transform chunks
  int64_t lead;
  uint32_t* cbits_u;  // carry-in bit per chunk
  uint32_t* cbits_v;
  double2* z;         // pre-mapped coefficients (N entries)
  MapConsts mc;
  DevStatus* status;
  uint32_t* aggs;  // per-block carry transfer functions (k_zstat)
  ZTile zt;        // layout of z as k_f1 reads it
  int32_t early;   // k_zstat: operands not written by in-flight kernels (read before pdl_wait)
  uint32_t* gen;   // look-back generation (advanced by the row pass, k_mid*)
  int32_t bchunks; // chunks per k_zgen block (kZgenThreads * per)
  // k_zgen without k_zstat: each block's carry-in by a decoupled look-back
  // over these words (the default); null: composed from k_zstat's aggs
  unsigned long long* lbstate;
  int32_t zs_rb;   // k_zsplit: rows of z's tiles per block (8 or 1)
};
constexpr int kZgenThreads = 256;
constexpr int kZgenPer = 16;
constexpr int kZgenChunks = kZgenThreads * kZgenPer;
__global__ void k_zstat(ZgenArgs a);
typedef void (*ZgenFn)(ZgenArgs);
ZgenFn zgen_kernel(int b, int lam, int per = 16);
// Digit form for the first column pass's own pre-map (k_f1d_ct): the
// balanced digits of both operands in z's tile order, as short2 (dig = 1,
// b <= 14) or int2 (dig = 2), no pre-map.
ZgenFn zgen_digits_kernel(int b, int dig, int per = 16);
// digit element type of a chunk width for the digit form
inline int zdig_kind(int b) { return b <= 14 ? 1 : 2; }
size_t zgen_smem(int b, int per = 16);
// Split by runs (k_zsplit.cu): digit form, balanced split, compiled chunk
// widths (nullptr otherwise); no carry aggregates, no look-back.
ZgenFn zsplit_kernel(int b, int dig);
size_t zsplit_smem(int b);
int zsplit_chunks();

// F1: forward column DFTs over A of the pre-mapped coefficients.
struct F1Args {
  const double2* z;
  ZTile zt;
  double2* out;    // T[k_a][col], row length ncols
  uint32_t ncols;  // = L / A
  uint32_t logc;   // columns per CTA = 2^logc
  uint32_t stw;    // inter-pass twiddles staged per CTA (f1_tw_bytes reserved)
  SubFft fft;      // length A
  TwGlobal tw;     // omega_L
  MapConsts mc;
  // high product: top-chunk fold (maps_f64.cpp:337-347) and root channel
  const uint64_t* u;
  const uint64_t* v;
  int64_t nlimbs;
  int32_t b;
  int64_t count;
  int64_t lead;
  const uint32_t* cbits_u;
  const uint32_t* cbits_v;
  double* aux;  // [0] theta_u * theta_v
  const void* dig;  // k_f1d_ct: balanced digits in z's tile order (short2 / int2)
};
__global__ void k_f1(F1Args a);
size_t f1_smem_bytes(uint32_t A, uint32_t c);
// staged inter-pass twiddles of the first column pass (0 when nthr % c != 0)
size_t f1_tw_bytes(uint32_t A, uint32_t c, uint32_t nthr);

struct ColArgs {
  double2* data;  // in place
  ColGeom g;
  uint32_t logc;
  SubFft fft;
  TwGlobal tw;       // omega_L
  int32_t inv;       // inverse transform
  // twiddle after the DFT: omega_L^{((outer * to + col * tc) * k) * tmul}
  uint32_t to, tc, tmul;
};
__global__ void k_col(ColArgs a);
// ping-pong column passes (fft_pp)
constexpr int kColPPThreads = 1024;
__global__ void k_f1_pp(F1Args a);
typedef void (*ColFn)(ColArgs);
ColFn col_pp_kernel(bool inv);
size_t colpp_smem_bytes(uint32_t R, uint32_t c);

struct MidArgs {
  double2* data;  // rows of length C at storage index (k_a * B + k_b) * C
  uint32_t A, B, C;
  SubFft fwd;   // length C
  SubFft inv;   // length C / 2
  TwGlobal tw;  // omega_L
  uint32_t L;
  uint32_t* gen;  // look-back generation of the split and the carry (advanced here)
};
__global__ void k_mid(MidArgs a);
// C = 4096 row pass with compile-time schedules, persistent over row pairs.
constexpr int kMidCtThreads = 512;
__global__ void k_mid_4096(MidArgs a);
// compiled row passes of the shorter rows (mid-size products)
__global__ void k_mid_2048(MidArgs a);
__global__ void k_mid_1024(MidArgs a);

struct ILastArgs {
  const double2* data;  // S[k_a][...] with geometry g (outer = 0)
  double2* coef;        // y_m = (w_2m, w_2m+1), m = col + ncols * m_a
  ColGeom g;
  uint32_t logc;
  SubFft fft;  // length A (inverse)
  double scale, scale_lo;  // 1 / (4 L) as hi + lo, applied to the outputs
};
__global__ void k_ilast(ILastArgs a);
__global__ void k_ilast_pp(ILastArgs a);
// Compile-time column passes (k_f1_ct / k_ilast_ct) for the hot lengths.
using F1Fn = void (*)(F1Args);
using ILastFn = void (*)(ILastArgs);
struct ColCtShape {
  uint32_t R;
  int logc, nthr;
  int uses;  // passes served: 1 = F1, 2 = ilast, 4 = middle column passes (k_col_ct)
  int rad[4];
  F1Fn f1;
  ILastFn ilast;
  void (*col)(ColArgs);  // middle column pass (three-pass plans)
  uint32_t radl;  // radix of the last stage (output twiddle table)
};
// First column pass with the pre-map folded in (k_f1d.cu): compiled
// schedules of at least four columns per CTA; fn[f1d_variant(lambda, dig)]
// (nullptr where the pre-map's halo exceeds the tile).
struct F1DShape {
  uint32_t R;
  int logc, nthr;
  int rad[4];
  uint32_t radl;
  F1Fn fn[5];
};
const F1DShape* f1d_for(uint32_t R);
int f1d_variant(int lam, int dig);
// its shared memory: the colct tile, stage and twiddle tables, two buffers of
// digit slabs (zrows x c pairs; two slabs per buffer with a pre-map), barriers
size_t f1d_smem_bytes(uint32_t R, uint32_t c, uint32_t stablen, uint32_t radl, uint32_t zrows, int lam,
                      int dig);
// The compiled shape serving pass `role` (1 = F1, 2 = ilast) for column
// length R, or nullptr (TMG_NO_COLCT disables them); colct_stages(R) is the
// F1 shape's stage count (0 without one) for the parameter policy's cost
// model.
const ColCtShape* colct_for(uint32_t R, int role);
int colct_stages(uint32_t R);
size_t colct_smem_bytes(uint32_t R, uint32_t c, uint32_t stablen, uint32_t radl);

struct CarryArgs {
  const double* w;  // convolution coefficients (L of them)
  uint64_t* out;
  int64_t n;
  int64_t out_limbs;
  int64_t K;
  int64_t ML;
  int32_t shift_s;
  MapConsts mc;
  const double* aux;
  ScanState scan;
  DevStatus* status;
  uint64_t* tbuf;  // high: all limbs of t (ML words)
  // two-kernel carry (k_carry2.cu)
  void* sbuf;       // limb sums s_m, 16 B per limb
  uint32_t* aggs;   // per-block carry transfer functions
  int* cins;        // per-block carry-in (written by the last lanes block)
  uint32_t* ticket; // completion counter of k_carry_lanes (zero between launches)
  FastDiv fb;       // division by b
  uint32_t* hstop;  // high: first limb of t >> s that is not all ones (atomicMin; ~0 before)
  int32_t lanes_cins; // 1: the last k_carry_lanes block writes cins; 0: k_carry_patch scans aggs
  const uint32_t* gen;  // k_carry_lb: look-back generation (advanced by this product's k_zstat)
  // k_carry_runs (k_carry3.cu)
  int64_t wlen;       // doubles of w that may be read (L)
  int64_t blk_limbs;  // limbs per carry block for k_carry_patch (0: 256 x PT)
  int32_t runs_lb;    // 1: single pass, block carry-ins by look-back (a.scan, a.gen); 0: k_carry_patch follows
};
constexpr int kCarryThreads = 256;
constexpr int kCarryPerThread = 2;
__global__ void k_carry(CarryArgs a);
size_t carry_smem(int b);
constexpr int kC2Threads = 256;
typedef void (*CarryLanesFn)(CarryArgs);
CarryLanesFn carry_lanes_kernel(int lam, int pt);
CarryLanesFn carry_patch_kernel(int pt);
// single-pass lanes kernel with a decoupled look-back carry-in (k_carry_lb;
// nullptr for lambda outside {0, 4, 5}); a.scan: look-back words, ctr
// [0] ticket, [1] done, [2] generation
CarryLanesFn carry_lb_kernel(int lam, int pt);
size_t carry2_smem(int b, int lam, int pt, bool hbuf);
// runs kernel (k_carry3.cu): one thread per run of 64 coefficients, b limbs;
// nullptr without an instantiation for (mode, lambda)
constexpr int kRunThreads = 128;
CarryLanesFn carry_runs_kernel(int mode, int lam, int b, bool compiled_b);
size_t carry_runs_smem(int mode, int lam, int run);
int carry_runs_len(int mode, int lam, int b, bool compiled_b);

struct HighRoundArgs {
  const uint64_t* tbuf;
  uint64_t* out;
  int64_t n;
  int64_t out_limbs;
  int64_t ML;   // limbs of t
  int64_t WL;   // limbs of w examined (covers every bit of t >> s)
  int32_t shift_s;
  DevStatus* status;
  uint32_t* ticket;  // [0] completion counter (zero between launches),
                     // [1] first limb of t >> s that is not all ones, i.e. the
                     //     limb that stops the rounding increment (~0 between launches)
};
constexpr int kHighPerThread = 8;  // limbs of w per thread in k_high_agg / k_high_round
__global__ void k_high_agg(HighRoundArgs a);
__global__ void k_status_publish(const DevStatus* src, uint32_t* flag_out, DevStatus* merge);
__global__ void k_high_round(HighRoundArgs a);

// Schoolbook product for operands below the pipeline cutoff (the reference's
// ORACLE_FALLBACK mode, products.hpp:14-15).
struct BaseArgs {
  const uint64_t* u;
  const uint64_t* v;
  uint64_t* prod;  // 2 * nlimbs words
  int64_t nlimbs;
};
__global__ void k_basecase(BaseArgs a);

// The reference's int64 splitters as an entry point of their own
// (k_split_i64.cu; products.hpp:68-79).
void launch_split_i64(const uint64_t* d_limbs, int64_t nlimbs, int64_t n, int b, int64_t count,
                      bool balanced, int64_t lead, int64_t* d_out, uint32_t* d_flags,
                      cudaStream_t st);

// Stand-alone cyclic convolution (k_conv.cu; convolution.hpp:64-67).
void launch_conv_absmax(const double* d_f, const double* d_g, int64_t n, uint64_t* d_mx,
                        int num_sms, cudaStream_t st);
void launch_conv_pack(const double* d_f, const double* d_g, int64_t n, double gscale,
                      double2* d_z, cudaStream_t st);
void launch_conv_direct(const double* d_f, const double* d_g, int64_t n, double* d_out,
                        cudaStream_t st);

// The ring-change maps on their own (k_maps.cu; maps_f64.hpp).
void launch_map_pre(const MapConsts& mc, const double* d_in, double* d_out, double* d_aux,
                    cudaStream_t st);
void launch_map_post(const MapConsts& mc, const double* d_in, double aux, double* d_out,
                     cudaStream_t st);

}  // namespace tmg
