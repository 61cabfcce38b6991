// The reference's machine-word splitters as a stand-alone entry point:
// split_low_i64 / split_high_i64 (products.hpp:68-79, split.cpp:66-158).
//
//   chunk_i = window_i(u 2^lead) + carry_i, rebalanced into
//   (-2^{b-1}, 2^{b-1}] below the top chunk when the split is signed
//   (chunk_store, split.cpp:66-102); the top chunk absorbs its carry and
//   is not rebalanced; lead = 0 for the low split, sigma = (N + 1) b - n
//   for the top-aligned high split (count = N + 1).
//
// A warp owns kSplitPer tiles of 32 consecutive chunks, a lane one chunk of
// each tile (8-byte stores coalesce; a tile's window loads share a few
// limbs through L1), all of a lane's windows loaded before any is used.  The
// sequential carry of chunk_store needs no scan over the operand: chunk j
// sends a carry up exactly when window_j + carry_j > 2^{b-1}, which window_j
// alone decides unless it equals 2^{b-1} (then it passes its own carry-in
// on).  Per tile the warp ballots "my window generates" and "my window
// passes"; a lane's carry-in comes from the nearest lane below it that does
// not pass, and when every lane below passes from the tile's carry-in: the
// tile before it in the warp decides that the same way, and for the warp's
// first tile the warp walks down from the chunk below it, 32 windows per
// trip, through windows equal to 2^{b-1} (one in 2^b for random operands; an
// operand made of such windows only costs every warp a walk to chunk 0:
// 2^24 bits at b = 13 take 359 ms with a one-window walk).  Algorithmic bytes: n / 8
// read, 8 per chunk written.
//
// The products' own split (k_zsplit / k_zgen) stores FFT-ordered digit
// pairs of both operands; this kernel serves callers that want the chunks
// themselves, like the reference's tests (test_products.cpp:52-176).
#include "kernels.cuh"

namespace tmg {

namespace {

constexpr int kSplitThreads = 256;
constexpr int kSplitPer = 8;  // tiles of 32 chunks per warp

__global__ void __launch_bounds__(kSplitThreads)
k_split_i64(const uint64_t* __restrict__ limbs, int64_t nlimbs, int64_t n, int b, int64_t count,
            int balanced, int64_t lead, long long* __restrict__ out, uint32_t* __restrict__ flags) {
  const uint32_t lane = threadIdx.x & 31u;
  const int64_t warp = (int64_t(blockIdx.x) * kSplitThreads + threadIdx.x) >> 5;
  const int64_t base = warp * (32 * kSplitPer);
  if (warp == 0 && lane == 0 && (n & 63)) {
    // operand outside [0, 2^n) (check_operand, split.cpp:13-18)
    if (__ldg(limbs + nlimbs - 1) >> (n & 63)) atomicOr(flags, uint32_t(kFlagInputRange));
  }
  if (base >= count) return;  // warp-uniform
  const uint64_t half = 1ull << (b - 1);
  // chunks past the last read zero windows (they kill, and nothing reads them)
  uint64_t w[kSplitPer];
#pragma unroll
  for (int k = 0; k < kSplitPer; ++k) {
    const int64_t i = base + 32 * k + lane;
    w[k] = i < count ? window_bits(limbs, nlimbs, i * b - lead, b) : 0ull;
  }
  // the warp's carry-in: the chunk below its first, walked down through passing windows
  int cin = 0;
  if (balanced) {
    // the whole warp walks: 32 windows per trip, the highest lane whose
    // window does not pass decides (a window below chunk 0 reads 0: no carry)
    for (int64_t j = base - 1; j >= 0; j -= 32) {
      const int64_t jj = j - lane;
      const uint64_t x = jj >= 0 ? window_bits(limbs, nlimbs, jj * b - lead, b) : 0ull;
      const uint32_t dec = __ballot_sync(0xffffffffu, x != half);
      if (dec) {
        const int first = __ffs(dec) - 1;  // lane 0 holds the chunk nearest to the warp
        cin = int((__ballot_sync(0xffffffffu, x > half) >> first) & 1u);
        break;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kSplitPer; ++k) {
    const int64_t i = base + 32 * k + lane;
    int carry = 0;
    if (balanced) {
      const uint32_t gen = __ballot_sync(0xffffffffu, w[k] > half);
      const uint32_t decide = ~__ballot_sync(0xffffffffu, w[k] == half);  // lanes that do not pass
      const uint32_t below = decide & ((1u << lane) - 1u);
      carry = below ? int((gen >> (31 - __clz(below))) & 1u) : cin;
      if (decide) cin = int((gen >> (31 - __clz(decide))) & 1u);  // into the next tile
    }
    if (i < count) out[i] = split_digit(w[k], carry, b, !balanced || i == count - 1);
  }
}

}  // namespace

// Enqueues the split of one operand (device pointers) on st.  flags: one
// zeroed device word, kFlagInputRange set when u has bits at or above n.
void launch_split_i64(const uint64_t* d_limbs, int64_t nlimbs, int64_t n, int b, int64_t count,
                      bool balanced, int64_t lead, int64_t* d_out, uint32_t* d_flags,
                      cudaStream_t st) {
  constexpr int64_t per_block = int64_t(kSplitThreads) * kSplitPer;
  const int64_t blocks = (count + per_block - 1) / per_block;
  k_split_i64<<<dim3(unsigned(blocks)), dim3(kSplitThreads), 0, st>>>(
      d_limbs, nlimbs, n, b, count, balanced ? 1 : 0, lead, reinterpret_cast<long long*>(d_out),
      d_flags);
}

}  // namespace tmg
