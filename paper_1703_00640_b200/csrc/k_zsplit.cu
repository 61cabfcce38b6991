// Balanced split by runs: the digit form of the split for the large
// products (the first column pass pre-maps, k_f1d.cu).
//
// One thread owns a run of 32 consecutive chunks: 32 b bits, a whole number
// of 32-bit words whatever b is, so with the chunk width a compile-time
// constant every window is one funnel shift at a static offset of the run's
// b + 1 words (taken once from the block's staged operand bits and
// pre-shifted by the block-uniform sub-word offset).  The carry of the
// balanced split (split.cpp:88-95) enters a run from the window below it: a
// window other than 2^{b-1} decides its carry-out whatever comes in (1 above,
// 0 below), so the run reads that one window (and walks further down only
// through windows equal to 2^{b-1}, inside its row segment; below the segment
// one warp per segment has walked for the block) -- no block scan, no
// aggregates, no look-back.  The thread then walks its chunks with
// the carry in a register and stores the digit pairs of both operands
// (short2 for b <= 14, else int2) in 16-byte pieces in z's tile order, plus
// its 32 carry-in bits per operand (one word: the few places that re-derive
// single digits later read them).
//
// Runs that hold the top chunk (not balanced), chunks at or above N (not
// stored) or the end of the chunks take a per-chunk path.
//
// Reference: split.cpp:66-102 (chunk_store).
#include "kernels.cuh"

namespace tmg {

namespace {

constexpr int kZsThreads = 256;
constexpr int kZsRun = 32;
constexpr int kZsChunks = kZsThreads * kZsRun;

// staged words per operand: the block's chunks and, for each of up to 8 row
// segments, the window below, the sub-word offset and the look-ahead
__host__ __device__ constexpr int zs_seg_words(int b) { return ((((kZsChunks / 8 + 1) * b + 31) / 32 + 12) + 3) / 4 * 4; }
__host__ __device__ constexpr int zs_words_alloc(int b) { return 8 * zs_seg_words(b); }

__device__ __forceinline__ uint32_t ld_word(const uint64_t* limbs, int64_t nlimbs, int64_t wi) {
  return (wi >= 0 && wi < 2 * nlimbs) ? __ldg(reinterpret_cast<const uint32_t*>(limbs) + wi) : 0u;
}

// Carry out of chunk j (>= 0, below the top chunk): its window decides it
// unless it equals 2^{b-1}; then the chunk below does.
// The walk stays inside the thread's row segment (chunks >= cs): below it the
// carry into chunk cs is segcin, which one warp per segment has walked for
// the whole block (see the kernel).
__device__ __noinline__ int carry_below(const uint64_t* limbs, int64_t nlimbs, int64_t lead, int b, int64_t j,
                                        int64_t cs, int segcin) {
  const uint64_t half = 1ull << (b - 1);
  for (; j >= cs; --j) {
    const uint64_t w = window_bits(limbs, nlimbs, j * b - lead, b);
    if (w != half) return w > half ? 1 : 0;
  }
  return segcin;
}

template <int DIG>
struct ZsOut;
template <>
struct ZsOut<1> {
  static constexpr int kPer = 4;  // chunks per 16-byte piece
  __device__ __forceinline__ static void put1(void* z, uint32_t i, int32_t du, int32_t dv) {
    static_cast<short2*>(z)[i] = make_short2(short(du), short(dv));
  }
};
template <>
struct ZsOut<2> {
  static constexpr int kPer = 2;
  __device__ __forceinline__ static void put1(void* z, uint32_t i, int32_t du, int32_t dv) {
    static_cast<int2*>(z)[i] = make_int2(du, dv);
  }
};

template <int B, int DIG>
__global__ void __launch_bounds__(kZsThreads) k_zsplit(ZgenArgs a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* su = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* sv = su + zs_words_alloc(B);
  const int tid = threadIdx.x;
  const int64_t count = a.count, N = a.N;
  // Block geometry: rb rows of z's tiles by cb = 8192 / rb columns (a.zs_rb =
  // 8 where the column count allows: the threads of a warp then own runs of
  // adjacent rows, whose 16-byte digit pieces are adjacent in a tile), or
  // 8192 consecutive chunks (rb = 1).  A row segment is cb consecutive chunks.
  const uint32_t rb = uint32_t(a.zs_rb), cb = uint32_t(kZsChunks) / rb;
  const uint32_t ncols = a.zt.fdcols.d;
  const uint32_t nbands = rb > 1 ? ncols / cb : 1u;
  const uint32_t band = blockIdx.x % nbands, rg = blockIdx.x / nbands;
  auto seg_first = [&](uint32_t sgm) -> int64_t {
    return rb > 1 ? int64_t(rg * rb + sgm) * ncols + int64_t(band) * cb : int64_t(blockIdx.x) * kZsChunks;
  };
  // staged bits of a segment: from the window below its first chunk
  const uint32_t SW = uint32_t(zs_words_alloc(B)) / rb;  // words per segment (multiple of 4: rb divides 8)
  auto seg_geom = [&](uint32_t sgm, int64_t& w4, uint32_t& off0, int& n4) {
    const int64_t cs = seg_first(sgm);
    const int64_t ce = min(count, cs + int64_t(cb));
    const int64_t bitlo = (cs - 1) * B - a.lead;
    w4 = (bitlo >> 5) & ~int64_t(3);  // floor, 16-byte aligned
    off0 = uint32_t(bitlo - (w4 << 5));  // < 128
    const int nwd = ce > cs ? int((off0 + uint32_t(ce - cs + 1) * uint32_t(B) + 31u) >> 5) + 2 : 0;
    n4 = (nwd + 3) / 4;
  };
  {
    // every segment's slot is filled whole (a few words more than its
    // windows need), all of a thread's loads in flight at once; 16-byte loads
    // where the four words lie inside the operand, else word by word with
    // zeros outside
    const bool al = ((reinterpret_cast<uintptr_t>(a.u) | reinterpret_cast<uintptr_t>(a.v)) & 15) == 0;
    constexpr uint32_t NS4 = uint32_t(zs_seg_words(B)) / 4;  // 16-byte pieces per segment slot (rb = 8)
    constexpr uint32_t TOT4 = 8 * NS4;                         // per operand
    constexpr int NIT = int((TOT4 + kZsThreads - 1) / kZsThreads);
    int64_t w40;
    uint32_t off0;
    int n40;
    seg_geom(0, w40, off0, n40);
    // (segments start ncols B bits apart: their 16-byte aligned first words follow from their own bit offsets)
    uint4 vu[NIT], vv[NIT];
    bool vec[NIT];
    int64_t wq[NIT];
#pragma unroll
    for (int k = 0; k < NIT; ++k) {
      const uint32_t i = uint32_t(tid) + uint32_t(k) * kZsThreads;
      const uint32_t sgm = rb == 1 ? 0u : i / NS4;
      const uint32_t e = rb == 1 ? i : i - sgm * NS4;
      int64_t w4s = w40;
      if (sgm) {
        const int64_t bitlo = (seg_first(sgm) - 1) * B - a.lead;
        w4s = (bitlo >> 5) & ~int64_t(3);
      }
      wq[k] = w4s + 4 * int64_t(e);
      vec[k] = i < TOT4 && al && wq[k] >= 0 && wq[k] + 4 <= 2 * a.nlimbs;
      if (vec[k]) {
        vu[k] = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(a.u) + wq[k]));
        vv[k] = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(a.v) + wq[k]));
      }
    }
#pragma unroll
    for (int k = 0; k < NIT; ++k) {
      const uint32_t i = uint32_t(tid) + uint32_t(k) * kZsThreads;
      if (i < TOT4) {
        if (!vec[k]) {
          vu[k] = make_uint4(ld_word(a.u, a.nlimbs, wq[k]), ld_word(a.u, a.nlimbs, wq[k] + 1),
                             ld_word(a.u, a.nlimbs, wq[k] + 2), ld_word(a.u, a.nlimbs, wq[k] + 3));
          vv[k] = make_uint4(ld_word(a.v, a.nlimbs, wq[k]), ld_word(a.v, a.nlimbs, wq[k] + 1),
                             ld_word(a.v, a.nlimbs, wq[k] + 2), ld_word(a.v, a.nlimbs, wq[k] + 3));
        }
        reinterpret_cast<uint4*>(su)[i] = vu[k];
        reinterpret_cast<uint4*>(sv)[i] = vv[k];
      }
    }
  }
  // Carry into the first chunk of each row segment, for the runs whose walk
  // through windows equal to 2^{b-1} reaches the segment's start: warp w
  // walks below segment w with 32 windows per trip (the lane nearest to the
  // segment that does not pass decides; windows below chunk 0 read 0: no
  // carry).  One trip for random operands; an operand made of such windows
  // costs the block 8 warp walks to chunk 0 and not one per run.
  __shared__ int s_segcin[2][8];
  if (uint32_t(tid) >> 5 < rb) {
    const uint32_t wp = uint32_t(tid) >> 5, ln = uint32_t(tid) & 31u;
    const int64_t cs = seg_first(wp);
    constexpr uint64_t halfw = 1ull << (B - 1);
#pragma unroll 1
    for (int op = 0; op < 2; ++op) {
      const uint64_t* lp = op ? a.v : a.u;
      int cin = 0;
#pragma unroll 1
      for (int64_t j = cs - 1; j >= 0; j -= 32) {
        const int64_t jj = j - int64_t(ln);
        const uint64_t x = jj >= 0 ? window_bits(lp, a.nlimbs, jj * B - a.lead, B) : 0ull;
        const uint32_t dec = __ballot_sync(0xffffffffu, x != halfw);
        if (dec) {
          cin = int((__ballot_sync(0xffffffffu, x > halfw) >> (__ffs(dec) - 1)) & 1u);
          break;
        }
      }
      if (ln == 0) s_segcin[op][wp] = cin;
    }
  }
  if (blockIdx.x == 0 && tid == 0 && (a.n & 63)) {
    const uint64_t hm = ~0ull << (a.n & 63);
    if ((__ldg(a.u + a.nlimbs - 1) | __ldg(a.v + a.nlimbs - 1)) & hm)
      atomicOr(&a.status->flags, uint32_t(kFlagInputRange));
  }
  __syncthreads();
  // consecutive threads: consecutive rows of the group, then the next run
  const uint32_t lr = uint32_t(tid) % rb, rc = uint32_t(tid) / rb;
  const int64_t j0 = seg_first(lr) + int64_t(rc) * kZsRun;
  if (j0 >= count) return;
  su += lr * SW;
  sv += lr * SW;
  constexpr uint32_t mask = (1u << B) - 1u, half = 1u << (B - 1);
  constexpr int32_t full = int32_t(1) << B;
  // the window below the run and the run's first window, in staged bits
  uint32_t relp;
  {
    int64_t w4;
    uint32_t off0;
    int n4;
    seg_geom(lr, w4, off0, n4);
    relp = off0 + rc * uint32_t(kZsRun * B);
  }
  const uint32_t rel0 = relp + uint32_t(B);
  int cu, cv;
  {
    const uint32_t wi = relp >> 5, sh = relp & 31u;
    const uint32_t pu = __funnelshift_r(su[wi], su[wi + 1], sh) & mask;
    const uint32_t pv = __funnelshift_r(sv[wi], sv[wi + 1], sh) & mask;
    cu = pu > half ? 1 : 0;
    cv = pv > half ? 1 : 0;
    // a window equal to 2^{b-1} passes the carry of the chunk below it on
    if (pu == half) cu = carry_below(a.u, a.nlimbs, a.lead, B, j0 - 2, seg_first(lr), s_segcin[0][lr]);
    if (pv == half) cv = carry_below(a.v, a.nlimbs, a.lead, B, j0 - 2, seg_first(lr), s_segcin[1][lr]);
    if (j0 == 0) cu = cv = 0;
  }
  const ZTile& zt = a.zt;
  if (j0 + kZsRun <= N && j0 + kZsRun <= count - 1) {
    // every chunk of the run is a balanced, stored chunk
    const uint32_t wi0 = rel0 >> 5, dl = rel0 & 31u;
    uint32_t Wu[B], Wv[B];
    {
      uint32_t lu = su[wi0], lv = sv[wi0];
#pragma unroll
      for (int i = 0; i < B; ++i) {
        const uint32_t nu = su[wi0 + i + 1], nv = sv[wi0 + i + 1];
        Wu[i] = __funnelshift_r(lu, nu, dl);
        Wv[i] = __funnelshift_r(lv, nv, dl);
        lu = nu;
        lv = nv;
      }
    }
    // the run lies in one row of z's tiles (the column count is a multiple of 32)
    uint32_t row = 0, col = uint32_t(j0);
    if (!zt.natural) {
      row = fdiv(uint32_t(j0), zt.fdcols);
      col = uint32_t(j0) - row * zt.fdcols.d;
    }
    const uint32_t cm = (1u << zt.logc) - 1;
    uint4* z4 = static_cast<uint4*>(static_cast<void*>(a.z));
    uint32_t bu = 0, bv = 0;
    constexpr int P = ZsOut<DIG>::kPer;
#pragma unroll
    for (int g = 0; g < kZsRun / P; ++g) {
      int32_t du[P], dv[P];
#pragma unroll
      for (int t = 0; t < P; ++t) {
        const int q = g * P + t;
        const int i = (q * B) >> 5, s = (q * B) & 31;
        // (a window that ends inside word i needs no second word; the last one ends the run)
        const int i1 = (s + B <= 32) ? i : i + 1;
        const uint32_t wu = (s + B <= 32 ? (Wu[i] >> s) : __funnelshift_r(Wu[i], Wu[i1], s)) & mask;
        const uint32_t wv = (s + B <= 32 ? (Wv[i] >> s) : __funnelshift_r(Wv[i], Wv[i1], s)) & mask;
        bu |= uint32_t(cu) << q;
        bv |= uint32_t(cv) << q;
        const int32_t xu = int32_t(wu) + cu, xv = int32_t(wv) + cv;
        cu = xu > int32_t(half) ? 1 : 0;
        cv = xv > int32_t(half) ? 1 : 0;
        du[t] = xu - (cu ? full : 0);
        dv[t] = xv - (cv ? full : 0);
      }
      const uint32_t cg = col + uint32_t(g * P);
      const uint32_t idx = zt.natural ? cg : ((((cg >> zt.logc) * zt.zrows + row) << zt.logc) + (cg & cm));
      uint4 o;
      if constexpr (DIG == 1) {
        o.x = (uint32_t(du[0]) & 0xffffu) | (uint32_t(dv[0]) << 16);
        o.y = (uint32_t(du[1]) & 0xffffu) | (uint32_t(dv[1]) << 16);
        o.z = (uint32_t(du[2]) & 0xffffu) | (uint32_t(dv[2]) << 16);
        o.w = (uint32_t(du[3]) & 0xffffu) | (uint32_t(dv[3]) << 16);
        z4[idx >> 2] = o;
      } else {
        o.x = uint32_t(du[0]);
        o.y = uint32_t(dv[0]);
        o.z = uint32_t(du[1]);
        o.w = uint32_t(dv[1]);
        z4[idx >> 1] = o;
      }
    }
    a.cbits_u[j0 >> 5] = bu;
    a.cbits_v[j0 >> 5] = bv;
    return;
  }
  // per-chunk path: the top chunk keeps its carry (not balanced), chunks at
  // or above N are not stored
  uint32_t bu = 0, bv = 0;
  for (int q = 0; q < kZsRun; ++q) {
    const int64_t j = j0 + q;
    if (j >= count) break;
    const uint32_t rel = rel0 + uint32_t(q * B);
    const uint32_t wi = rel >> 5, sh = rel & 31u;
    const uint32_t wu = __funnelshift_r(su[wi], su[wi + 1], sh) & mask;
    const uint32_t wv = __funnelshift_r(sv[wi], sv[wi + 1], sh) & mask;
    const bool top = j == count - 1;
    bu |= uint32_t(cu) << q;
    bv |= uint32_t(cv) << q;
    const int32_t du = int32_t(split_digit(wu, cu, B, top)), dv = int32_t(split_digit(wv, cv, B, top));
    if (j < N) ZsOut<DIG>::put1(a.z, zt.index(uint32_t(j)), du, dv);
    cu = (!top && int32_t(wu) + cu > int32_t(half)) ? 1 : 0;
    cv = (!top && int32_t(wv) + cv > int32_t(half)) ? 1 : 0;
  }
  a.cbits_u[j0 >> 5] = bu;
  a.cbits_v[j0 >> 5] = bv;
}

}  // namespace

ZgenFn zsplit_kernel(int b, int dig) {
  if (dig == 1) {
    switch (b) {
      case 11: return k_zsplit<11, 1>;
      case 12: return k_zsplit<12, 1>;
      case 13: return k_zsplit<13, 1>;
      case 14: return k_zsplit<14, 1>;
      default: return nullptr;
    }
  }
  switch (b) {
    case 17: return k_zsplit<17, 2>;
    case 18: return k_zsplit<18, 2>;
    case 19: return k_zsplit<19, 2>;
    case 20: return k_zsplit<20, 2>;
    default: return nullptr;
  }
}

size_t zsplit_smem(int b) { return 2 * size_t(zs_words_alloc(b)) * 4; }
int zsplit_chunks() { return kZsChunks; }

}  // namespace tmg
