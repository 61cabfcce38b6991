// Balanced split + pre-map as one streaming pass (both operands at once).
//
// A block owns kZgenChunks consecutive chunks.  It stages the operand bits
// under them in shared memory (coalesced; 32-bit words when b <= 32 so each
// b-bit window is one funnel shift), takes every window once into
// registers, derives the chunks' carry statuses, resolves the carry into the
// block from the per-block aggregates of k_zstat (composed in parallel, no
// look-back wait), writes the balanced digits to shared memory (plus the
// first lambda-1 digits of the next block, whose carry it now knows), and
// emits the pre-mapped coefficients z_j = (alpha*U)_j + i (alpha*V)_j (gamma+
// without its top-coefficient fold for the high product; the full product
// stores the digits themselves) for j in [c0 + lambda - 1, c1 + lambda - 1)
// mod N.  The carry-in bit of every chunk is kept for the few places that
// re-derive single digits later (F1's high-product fold and root channel).
//
// Reference: split.cpp:66-102 (chunk_store), maps_f64.cpp:48-136 and
// 317-348 (alpha*, gamma+).
#include "kernels.cuh"

#include <type_traits>

namespace tmg {

namespace {

// Operand bits as a shared-memory array of W-bit words (W = 32 or 64)
// starting at word wbase (words outside the operand read as zero).
template <bool W32>
struct StagedBits {
  using Word = typename std::conditional<W32, uint32_t, uint64_t>::type;
  static constexpr int kW = W32 ? 32 : 64;
  static constexpr int kLog = W32 ? 5 : 6;
  const Word* s;
  // b-bit window at bit offset rel (>= 0) from the first staged word
  __device__ __forceinline__ uint64_t window(uint32_t rel, uint64_t mask) const {
    const uint32_t wi = rel >> kLog, sh = rel & (kW - 1);
    if constexpr (W32) {
      return uint64_t(__funnelshift_r(s[wi], s[wi + 1], sh)) & mask;
    } else {
      const uint64_t lo = s[wi], hi = s[wi + 1];
      return (sh ? ((lo >> sh) | (hi << (64 - sh))) : lo) & mask;
    }
  }
};

// Digit slot of local chunk i: one pad slot per 16, so that the 16
// consecutive digits a thread writes land in distinct banks across a warp.
__device__ __forceinline__ int32_t zpad(int32_t i) { return i + (i >> 4); }

// Exact int32 -> double on the FP64 pipe (2^52 + 2^31 magic), in place of
// the quarter-rate I2F.
__device__ __forceinline__ double i2d_exact(int32_t x) {
  return __hiloint2double(0x43300000, int(uint32_t(x) ^ 0x80000000u)) - 4503601774854144.0;
}

template <bool W32>
__device__ __forceinline__ typename StagedBits<W32>::Word load_word(const uint64_t* limbs,
                                                                    int64_t nlimbs,
                                                                    int64_t wi) {
  if constexpr (W32) {
    return (wi >= 0 && wi < 2 * nlimbs) ? __ldg(reinterpret_cast<const uint32_t*>(limbs) + wi)
                                        : 0u;
  } else {
    return (wi >= 0 && wi < nlimbs) ? __ldg(limbs + wi) : 0ull;
  }
}

// Staged words per operand: the chunks of one block plus the lambda-1 digits
// of the next, the sub-word offset and one word of look-ahead.
__host__ __device__ inline int64_t zgen_words(int b, int kw, int ch) {
  return (int64_t(ch + kMaxLambda) * b + kw - 1) / kw + 3;
}
// staged words reserved per operand: the 16-byte loads of interior blocks
// start up to 3 words early and round up to a multiple of 4
__host__ __device__ inline int64_t zgen_words_alloc(int b, int kw, int ch) {
  return (zgen_words(b, kw, ch) + 8 + 3) / 4 * 4;  // keeps the second operand 16-byte aligned
}

}  // namespace

size_t zgen_smem(int b, int per) {
  const int kw = b <= 32 ? 32 : 64;
  const int ch = kZgenThreads * per;
  return 2 * size_t(zgen_words_alloc(b, kw, ch)) * (kw / 8) + size_t((ch + kMaxLambda) * 17 / 16 + 2) * 8 + 64;
}

// Carry transfer function of each block of a.bchunks chunks for both
// operands' balanced-split chains (split.cpp:88-95).  A chunk whose window
// differs from 2^{b-1} decides its carry-out (1 above, 0 below) whatever
// comes in, so a block's aggregate is fixed by its last such chunk: one
// thread per block searches backwards from the block's end (one window for
// random operands; the whole block only when every window equals 2^{b-1}).
__global__ void __launch_bounds__(256)
k_zstat(ZgenArgs a) {
  // Reads only the operands and writes only its own aggregate array, so it
  // runs under the predecessor's tail and waits for it at the end instead:
  // its completion still implies the predecessor's, which keeps the
  // programmatic-launch chain intact for k_zgen and everything after it.
  // When the operands may be outputs of products still in flight on the
  // stream (a.early = 0, decided by the host), it waits first.
  pdl_trigger();
  if (!a.early) pdl_wait();
  const int64_t blk = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t count = a.count;
  const int64_t bch = a.bchunks;
  const int64_t nblk = (count + bch - 1) / bch;
  if (blk >= nblk) {
    pdl_wait();
    return;
  }
  const int b = a.b;
  const uint64_t half = 1ull << (b - 1);
  const int64_t c0 = blk * bch;
  // statuses exist for chunks below the (unbalanced) top chunk only
  const int64_t c1 = min(count - 1, c0 + bch);
  uint32_t fu = 2, fv = 2;  // propagate (identity)
  if (a.mc.balanced) {
    bool du = false, dv = false;
    for (int64_t j = c1 - 1; j >= c0 && !(du && dv); --j) {
      const int64_t pos = j * b - a.lead;
      if (!du) {
        const uint64_t w = window_bits(a.u, a.nlimbs, pos, b);
        if (w != half) {
          fu = w > half ? 1u : 0u;
          du = true;
        }
      }
      if (!dv) {
        const uint64_t w = window_bits(a.v, a.nlimbs, pos, b);
        if (w != half) {
          fv = w > half ? 1u : 0u;
          dv = true;
        }
      }
    }
  } else {
    fu = fv = 0;
  }
  a.aggs[blk] = fu | (fv << 2);
  pdl_wait();
}

// LAM: the series length lambda (rows of the pre-map), 0 for the full
// product (the digits themselves).  DIG (LAM = 0 only): 0 stores the digits
// as double2 coefficients, 1 as short2 and 2 as int2 (the digit form that
// k_f1d_ct pre-maps itself).
template <int DIG>
struct DigOut;
template <>
struct DigOut<0> {
  __device__ __forceinline__ static void put(void* z, uint32_t i, int2 d) {
    static_cast<double2*>(z)[i] = make_double2(double(d.x), double(d.y));
  }
};
template <>
struct DigOut<1> {
  __device__ __forceinline__ static void put(void* z, uint32_t i, int2 d) {
    static_cast<short2*>(z)[i] = make_short2(short(d.x), short(d.y));
  }
};
template <>
struct DigOut<2> {
  __device__ __forceinline__ static void put(void* z, uint32_t i, int2 d) { static_cast<int2*>(z)[i] = d; }
};

// PER: chunks per thread (16, or 4 / 1 for short products, whose blocks
// then fill more SMs); a block owns kZgenThreads * PER chunks.
template <bool W32, int LAM, int DIG = 0, int PER = 16>
__global__ void __launch_bounds__(kZgenThreads)
k_zgen_t(ZgenArgs a) {
  constexpr int kCh = kZgenThreads * PER;
  pdl_trigger();
  pdl_wait();
  using SB = StagedBits<W32>;
  using Word = typename SB::Word;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t sw[32];
  __shared__ uint32_t s_cin;

  const int tid = threadIdx.x;
  const MapConsts& mc = a.mc;
  const int b = a.b;
  const int64_t N = a.N;
  const int64_t count = a.count;
  constexpr int lam = LAM > 0 ? LAM : 1;
  constexpr int ext = lam - 1;
  const int64_t nwd = zgen_words(b, SB::kW, kCh);
  Word* su = reinterpret_cast<Word*>(smem_raw);
  Word* sv = su + zgen_words_alloc(b, SB::kW, kCh);
  // digits of the block's chunks (and the next lam-1), u and v packed
  int2* dig = reinterpret_cast<int2*>(sv + zgen_words_alloc(b, SB::kW, kCh));

  const uint32_t blk = blockIdx.x;
  const int64_t c0 = int64_t(blk) * kCh;
  const int64_t c1 = min(count, c0 + int64_t(kCh));
  const int64_t bit0 = c0 * b - a.lead;
  int64_t wbase = bit0 >> SB::kLog;  // floor, bit0 may be negative
  uint32_t off0 = uint32_t(bit0 - (wbase << SB::kLog));
  // Interior blocks (block-uniform): every chunk in [c0, c1 + lam - 1] is a
  // full balanced non-top chunk, its bits lie inside both operands, and
  // b <= 30 -- no per-chunk bound or top tests, 32-bit digit arithmetic and
  // 16-byte staging loads.
  bool interior = false;
  if constexpr (W32) {
    const int64_t w4 = wbase & ~int64_t(3);
    interior = mc.balanced && b <= 30 && c1 == c0 + kCh && c1 + ext < count - 1 &&
               w4 >= 0 && w4 + 4 * ((nwd + 6) / 4) <= 2 * a.nlimbs &&
               ((reinterpret_cast<uintptr_t>(a.u) | reinterpret_cast<uintptr_t>(a.v)) & 15) == 0;
    if (interior) {
      off0 += uint32_t(wbase - w4) * 32u;
      wbase = w4;
      const uint4* gu4 = reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(a.u) + wbase);
      const uint4* gv4 = reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(a.v) + wbase);
      uint4* su4 = reinterpret_cast<uint4*>(su);
      uint4* sv4 = reinterpret_cast<uint4*>(sv);
      const int64_t n4 = (nwd + 6) / 4;
      for (int64_t i = tid; i < n4; i += kZgenThreads) {
        su4[i] = __ldg(gu4 + i);
        sv4[i] = __ldg(gv4 + i);
      }
    }
  }
  if (!interior) {
    for (int64_t i = tid; i < nwd; i += kZgenThreads) {
      su[i] = load_word<W32>(a.u, a.nlimbs, wbase + i);
      sv[i] = load_word<W32>(a.v, a.nlimbs, wbase + i);
    }
  }
  __syncthreads();
  const SB Lu{su}, Lv{sv};
  const uint64_t half = 1ull << (b - 1);
  const uint64_t mask = (1ull << b) - 1;

  // this thread's PER windows, taken once
  const uint32_t q0 = uint32_t(tid) * PER;  // chunk offset in the block
  const int64_t t0 = c0 + q0;
  using Win = typename std::conditional<W32, uint32_t, uint64_t>::type;
  Win wu[PER], wv[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const uint32_t rel = off0 + (q0 + q) * uint32_t(b);
    wu[q] = Win(Lu.window(rel, mask));
    wv[q] = Win(Lv.window(rel, mask));
  }
  uint32_t gu = 0, pu = 0, gv = 0, pv = 0;
  if (interior) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      gu |= uint32_t(wu[q] > half) << q;
      pu |= uint32_t(wu[q] == half) << q;
      gv |= uint32_t(wv[q] > half) << q;
      pv |= uint32_t(wv[q] == half) << q;
    }
  } else if (mc.balanced) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int64_t j = t0 + q;
      if (j < c1 && j < count - 1) {
        gu |= uint32_t(wu[q] > half) << q;
        pu |= uint32_t(wu[q] == half) << q;
        gv |= uint32_t(wv[q] > half) << q;
        pv |= uint32_t(wv[q] == half) << q;
      }
    }
  }
  // kill / generate / propagate of this thread's run: its last non-P chunk
  auto kgp_of = [](uint32_t g, uint32_t p) -> uint32_t {
    const uint32_t np = ~p & ((PER >= 32) ? ~0u : ((1u << PER) - 1u));
    if (!np) return 2u;
    const int last = 31 - __clz(np);
    return (g >> last) & 1u;
  };
  uint32_t agg2;
  const uint32_t ex2 = block_scan_kgp(kgp_of(gu, pu) | (kgp_of(gv, pv) << 2), sw, &agg2);
  // carry into the block: by a look-back over the predecessors' published
  // aggregates (one-wave grids, no k_zstat), or the aggregates of the blocks
  // before it (k_zstat) composed in order by the whole block
  if (a.lbstate) {
    if (tid == 0) {
      const unsigned long long ep = (unsigned long long)(*a.gen) << 32;
      volatile unsigned long long* st = a.lbstate;
      if (blk != 0) st[blk] = ep | (1ull << 30) | agg2;
      // G = F_{blk-1} o ... o F_j until it has no propagate field (its value
      // no longer depends on the carries before) or an inclusive word
      uint32_t G = kKgpIdentity, cin = 0u;
      for (int64_t j = int64_t(blk) - 1; j >= 0; --j) {
        unsigned long long w;
        do {
          w = st[j];
        } while ((w >> 32) != (ep >> 32) || ((w >> 30) & 3u) == 0);
        if (((w >> 30) & 3u) == 2) {
          G = kgp_compose(uint32_t(w & 0xFu), G);
          break;
        }
        G = kgp_compose(uint32_t(w & 0xFu), G);
        if (((G >> 1) & 0x5u) == 0) break;  // no propagate field left
      }
      cin = kgp_compose(0u, G);  // both chains start with carry 0
      st[blk] = ep | (2ull << 30) | kgp_compose(cin, agg2);
      s_cin = cin;
    }
  } else {
    uint32_t g = kKgpIdentity;
    const uint32_t Q = (blk + kZgenThreads - 1) / kZgenThreads;
    const uint32_t i0 = uint32_t(tid) * Q, i1 = min(blk, i0 + Q);
    for (uint32_t i = i0; i < i1; ++i) g = kgp_compose(g, __ldg(a.aggs + i));
    uint32_t pre;
    (void)block_scan_kgp(g, sw, &pre);
    if (tid == 0) s_cin = kgp_compose(0u, pre);  // both chains start with carry 0
  }
  __syncthreads();
  const uint32_t cc = kgp_compose(s_cin, ex2);
  int cu = int(cc & 1u), cv = int((cc >> 2) & 1u);

  // digits and carry-in bits
  uint32_t bu = 0, bv = 0;
  if (interior) {
    const int32_t hb = int32_t(half), full = int32_t(1) << b;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      bu |= uint32_t(cu) << q;
      bv |= uint32_t(cv) << q;
      int32_t xu = int32_t(wu[q]) + cu, xv = int32_t(wv[q]) + cv;
      xu -= (xu > hb) ? full : 0;
      xv -= (xv > hb) ? full : 0;
      dig[zpad(q0 + q)] = make_int2(xu, xv);
      if (!((pu >> q) & 1u)) cu = int((gu >> q) & 1u);
      if (!((pv >> q) & 1u)) cv = int((gv >> q) & 1u);
    }
  } else {
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int64_t j = t0 + q;
    if (j < c1) {
      bu |= uint32_t(cu) << q;
      bv |= uint32_t(cv) << q;
      const bool top = j == count - 1 || !mc.balanced;
      dig[zpad(q0 + q)] = make_int2(int32_t(split_digit(wu[q], cu, b, top)),
                              int32_t(split_digit(wv[q], cv, b, top)));
      if (!((pu >> q) & 1u)) cu = int((gu >> q) & 1u);
      if (!((pv >> q) & 1u)) cv = int((gv >> q) & 1u);
    }
  }
  }
  // the next block's first lam-1 digits (carry out of this block known)
  if (t0 < c1 && t0 + PER >= c1) {
    for (int q = 0; q < ext; ++q) {
      const int64_t j = c1 + q;
      if (j >= N) break;
      const uint32_t rel = off0 + uint32_t(j - c0) * uint32_t(b);
      const uint64_t xu = Lu.window(rel, mask), xv = Lv.window(rel, mask);
      const bool top = j == count - 1 || !mc.balanced;
      dig[zpad(j - c0)] = make_int2(int32_t(split_digit(xu, cu, b, top)),
                              int32_t(split_digit(xv, cv, b, top)));
      cu = mc.balanced ? tf_apply(split_tf(xu, b), cu) : 0;
      cv = mc.balanced ? tf_apply(split_tf(xv, b), cv) : 0;
    }
  }
  {
    // 32 / PER consecutive threads fill one 32-bit word of carry bits
    constexpr int G = 32 / PER;
    uint32_t wu32 = bu << ((tid % G) * PER), wv32 = bv << ((tid % G) * PER);
#pragma unroll
    for (int off = 1; off < G; off <<= 1) {
      wu32 |= __shfl_xor_sync(0xffffffffu, wu32, off);
      wv32 |= __shfl_xor_sync(0xffffffffu, wv32, off);
    }
    if ((tid % G) == 0 && t0 < count) {
      a.cbits_u[t0 >> 5] = wu32;
      a.cbits_v[t0 >> 5] = wv32;
    }
  }
  if (blk == 0 && tid == 0 && (a.n & 63)) {
    const uint64_t hm = ~0ull << (a.n & 63);
    if ((__ldg(a.u + a.nlimbs - 1) | __ldg(a.v + a.nlimbs - 1)) & hm)
      atomicOr(&a.status->flags, uint32_t(kFlagInputRange));
  }
  const int64_t ce = min(c1, N);
  const int32_t nloc = int32_t(ce - c0);  // local chunks with a digit in this block
  const int32_t nN = int32_t(N - c0);     // local index of chunk N (wrap start)
  __syncthreads();
  // the wrap of the cyclic pre-map: digits of chunks 0 .. lam-2 (carry 0 in)
  // follow chunk N-1 (they replace chunk N's digit, which the pre-map does
  // not use -- the high product folds it in k_f1)
  if (LAM > 1 && tid == 0 && c1 + ext > N) {
    int cu = 0, cv = 0;
    for (int i = 0; i < ext; ++i) {
      const uint64_t wu = window_bits(a.u, a.nlimbs, int64_t(i) * b - a.lead, b);
      const uint64_t wv = window_bits(a.v, a.nlimbs, int64_t(i) * b - a.lead, b);
      dig[zpad(nN + i)] = make_int2(int32_t(split_digit(wu, cu, b, i == count - 1 || !mc.balanced)),
                              int32_t(split_digit(wv, cv, b, i == count - 1 || !mc.balanced)));
      cu = mc.balanced ? tf_apply(split_tf(wu, b), cu) : 0;
      cv = mc.balanced ? tf_apply(split_tf(wv, b), cv) : 0;
    }
  }
  __syncthreads();

  // outputs
  if constexpr (LAM == 0) {
    const ZTile& zt = a.zt;
    const uint32_t row0 = zt.natural ? 0u : fdiv(uint32_t(c0), zt.fdcols);
    const uint32_t col0 = uint32_t(c0) - row0 * zt.fdcols.d;
    if (!zt.natural && col0 + uint32_t(nloc) <= zt.fdcols.d) {
      // the block's chunks lie in one row of the column tiles: index by column
      const uint32_t cm = (1u << zt.logc) - 1;
      for (int32_t jl = tid; jl < nloc; jl += kZgenThreads) {
        const int2 d = dig[zpad(jl)];
        const uint32_t col = col0 + uint32_t(jl);
        DigOut<DIG>::put(a.z, ((col >> zt.logc) * zt.zrows + row0) * (cm + 1) + (col & cm), d);
      }
    } else {
      for (int32_t jl = tid; jl < nloc; jl += kZgenThreads) {
        const int2 d = dig[zpad(jl)];
        DigOut<DIG>::put(a.z, zt.index(uint32_t(c0 + jl)), d);
      }
    }
  } else {
    const double Nd = double(N);
    constexpr int fam_low = 0, fam_high = 2;
    const bool low = mc.mode == kModeLow;
    double cr[LAM];
#pragma unroll
    for (int r = 0; r < LAM; ++r) cr[r] = mc.cpre[r];
    if (nloc + ext <= nN) {
      // No output of this block wraps (block-uniform).  Row r of output j
      // uses coef_r(j - r) = ((j - r) g_1 ... g_{r-1}) c_r with g_i = j -/+ i N:
      // the exact integer factors are formed once per output and the products
      // run in coef_rt's order (bit-identical); digits convert on the FP64 pipe.
      const double sgN = low ? -Nd : Nd;
      const ZTile& zt = a.zt;
      const uint32_t row0 = zt.natural ? 0u : fdiv(uint32_t(c0), zt.fdcols);
      const uint32_t col0 = uint32_t(c0) - row0 * zt.fdcols.d;
      const bool onerow = !zt.natural && col0 + uint32_t(nloc + ext) <= 2 * zt.fdcols.d;
      const uint32_t cm = (1u << zt.logc) - 1;
      for (int32_t jl = ext + tid; jl < nloc + ext; jl += kZgenThreads) {
        const double jd = double(c0 + jl);
        double g[LAM > 1 ? LAM - 1 : 1];
#pragma unroll
        for (int i = 1; i < LAM - 1; ++i) g[i] = jd + double(i) * sgN;
        double au = 0.0, av = 0.0;
#pragma unroll
        for (int r = LAM - 1; r >= 0; --r) {
          double cf = 1.0;
          if (r > 0) {
            double pp = jd - double(r);
#pragma unroll
            for (int i = 1; i < r; ++i) pp *= g[i];
            cf = pp * cr[r];
          }
          const int2 d = dig[zpad(jl - r)];
          au += i2d_exact(d.x) * cf;
          av += i2d_exact(d.y) * cf;
        }
        if (onerow) {
          // z index without a division: the block spans at most two rows
          uint32_t col = col0 + uint32_t(jl), row = row0;
          if (col >= zt.fdcols.d) {
            col -= zt.fdcols.d;
            ++row;
          }
          a.z[((col >> zt.logc) * zt.zrows + row) * (cm + 1) + (col & cm)] = make_double2(au, av);
        } else {
          a.z[zt.index(uint32_t(c0 + jl))] = make_double2(au, av);
        }
      }
      return;
    }
    for (int32_t jl = ext + tid; jl < nloc + ext; jl += kZgenThreads) {
      double au = 0.0, av = 0.0;
      const double jd = double(c0 + jl);
#pragma unroll
      for (int r = LAM - 1; r >= 0; --r) {
        const int32_t il = jl - r;  // local chunk, in [0, nloc + ext)
        const int2 d = dig[zpad(il)];
        const double kd = jd - double(r) - (il >= nN ? Nd : 0.0);
        double cf;
        if (r == 0) cf = 1.0;
        else cf = low ? coef_rt(fam_low, r, kd, Nd, cr[r]) : coef_rt(fam_high, r, kd, Nd, cr[r]);
        au += double(d.x) * cf;
        av += double(d.y) * cf;
      }
      const int64_t j = c0 + jl;
      a.z[a.zt.index(uint32_t(j >= N ? j - N : j))] = make_double2(au, av);
    }
  }
}

template <bool W32, int PER>
ZgenFn zgen_kernel_l(int lam) {
  switch (lam) {
    case 0: return k_zgen_t<W32, 0, 0, PER>;
    case 1: return k_zgen_t<W32, 1, 0, PER>;
    case 2: return k_zgen_t<W32, 2, 0, PER>;
    case 3: return k_zgen_t<W32, 3, 0, PER>;
    case 4: return k_zgen_t<W32, 4, 0, PER>;
    case 5: return k_zgen_t<W32, 5, 0, PER>;
    case 6: return k_zgen_t<W32, 6, 0, PER>;
    case 7: return k_zgen_t<W32, 7, 0, PER>;
    default: return k_zgen_t<W32, 8, 0, PER>;
  }
}

ZgenFn zgen_kernel(int b, int lam, int per) {
  if (b > 32) return zgen_kernel_l<false, 16>(lam);
  return per == 1 ? zgen_kernel_l<true, 1>(lam) : per == 4 ? zgen_kernel_l<true, 4>(lam) : zgen_kernel_l<true, 16>(lam);
}

ZgenFn zgen_digits_kernel(int b, int dig, int per) {
  if (b > 32) return nullptr;
  if (per == 1) return dig == 1 ? k_zgen_t<true, 0, 1, 1> : k_zgen_t<true, 0, 2, 1>;
  if (per == 4) return dig == 1 ? k_zgen_t<true, 0, 1, 4> : k_zgen_t<true, 0, 2, 4>;
  return dig == 1 ? k_zgen_t<true, 0, 1, 16> : k_zgen_t<true, 0, 2, 16>;
}

}  // namespace tmg
