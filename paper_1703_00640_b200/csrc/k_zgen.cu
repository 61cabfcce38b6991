// Balanced split + pre-map as one streaming pass (both operands at once).
//
// A block owns kZgenChunks consecutive chunks.  It stages the limbs under
// them (coalesced), derives every chunk's carry status, resolves the carry
// into the block with a warp-parallel decoupled look-back over the paired
// (u, v) chains, writes the balanced digits to shared memory (plus the
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

namespace tmg {

namespace {

struct StagedLimbs {
  const uint64_t* s;
  int64_t i0, n;
  __device__ __forceinline__ uint64_t operator()(int64_t i) const {
    const int64_t o = i - i0;
    return (o >= 0 && o < n) ? s[o] : 0ull;
  }
};

__device__ __forceinline__ uint64_t window_at(const StagedLimbs& L, int64_t pos, int b) {
  const int64_t idx = pos >> 6;
  const uint32_t sh = uint32_t(pos & 63);
  const uint64_t lo = L(idx), hi = L(idx + 1);
  const uint64_t w = sh ? ((lo >> sh) | (hi << (64 - sh))) : lo;
  return w & ((1ull << b) - 1);
}

}  // namespace

size_t zgen_smem(int b) {
  const size_t nl = size_t((int64_t(kZgenChunks + kMaxLambda) * b + 63) / 64 + 3);
  return 2 * nl * 8 + size_t(2) * (kZgenChunks + kMaxLambda) * 4 + 64;
}

__global__ void __launch_bounds__(kZgenThreads)
k_zgen(ZgenArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t sw[32];
  __shared__ uint32_t s_blk, s_cin;
  __shared__ int32_t s_wrap[2][kMaxLambda];
  const int tid = threadIdx.x;
  const MapConsts& mc = a.mc;
  const int b = a.b;
  const int64_t N = a.N;
  const int64_t count = a.count;
  const int lam = (mc.mode == kModeFull) ? 1 : mc.lambda;
  const int ext = lam - 1;
  const int64_t nl = (int64_t(kZgenChunks + kMaxLambda) * b + 63) / 64 + 3;
  uint64_t* slu = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* slv = slu + nl;
  int32_t* digu = reinterpret_cast<int32_t*>(slv + nl);
  int32_t* digv = digu + (kZgenChunks + kMaxLambda);

  if (tid == 0) s_blk = uint32_t(atomicAdd(a.scan.ctr, 1ull));
  __syncthreads();
  const uint32_t blk = s_blk;
  const int64_t c0 = int64_t(blk) * kZgenChunks;
  const int64_t c1 = min(count, c0 + kZgenChunks);
  const int64_t pos0 = c0 * b - a.lead;
  const int64_t i0 = pos0 >> 6;
  for (int64_t i = tid; i < nl; i += kZgenThreads) {
    const int64_t g = i0 + i;
    const bool in = g >= 0 && g < a.nlimbs;
    slu[i] = in ? __ldg(a.u + g) : 0ull;
    slv[i] = in ? __ldg(a.v + g) : 0ull;
  }
  // digits of chunks 0 .. lam-2 (the wrap of the cyclic pre-map), carry 0 in
  if (tid == 0 && mc.mode != kModeFull && c1 + ext > N) {
    int cu = 0, cv = 0;
    for (int i = 0; i < ext; ++i) {
      const uint64_t wu = window_bits(a.u, a.nlimbs, int64_t(i) * b - a.lead, b);
      const uint64_t wv = window_bits(a.v, a.nlimbs, int64_t(i) * b - a.lead, b);
      s_wrap[0][i] = int32_t(split_digit(wu, cu, b, i == count - 1 || !mc.balanced));
      s_wrap[1][i] = int32_t(split_digit(wv, cv, b, i == count - 1 || !mc.balanced));
      cu = mc.balanced ? tf_apply(split_tf(wu, b), cu) : 0;
      cv = mc.balanced ? tf_apply(split_tf(wv, b), cv) : 0;
    }
  }
  __syncthreads();
  const StagedLimbs Lu{slu, i0, nl}, Lv{slv, i0, nl};
  const uint64_t half = 1ull << (b - 1);

  // statuses of this thread's kZgenPer chunks
  const int64_t t0 = c0 + int64_t(tid) * kZgenPer;
  uint32_t gu = 0, pu = 0, gv = 0, pv = 0;
#pragma unroll
  for (int q = 0; q < kZgenPer; ++q) {
    const int64_t j = t0 + q;
    if (j < c1 && j < count - 1 && mc.balanced) {
      const uint64_t wu = window_at(Lu, j * b - a.lead, b);
      const uint64_t wv = window_at(Lv, j * b - a.lead, b);
      gu |= uint32_t(wu > half) << q;
      pu |= uint32_t(wu == half) << q;
      gv |= uint32_t(wv > half) << q;
      pv |= uint32_t(wv == half) << q;
    }
  }
  auto agg_of = [](uint32_t g, uint32_t p) -> uint32_t {
    const uint32_t np = ~p & 0xffffu;
    if (!np) return kTfIdentity;
    const int last = 31 - __clz(np);
    return ((g >> last) & 1u) ? tf_const(1) : tf_const(0);
  };
  uint32_t agg2;
  const uint32_t ex2 = block_scan_tf2(tf2_pack(agg_of(gu, pu), agg_of(gv, pv)), sw, &agg2);
  if (tid < 32) {
    const uint32_t cin = lookback_warp2(a.scan.state, blk, agg2, a.scan.epoch, 5u);
    if (tid == 0) s_cin = cin;
  }
  __syncthreads();
  const uint32_t cc = tf2_apply(ex2, s_cin);
  int cu = int(cc & 3u) - 1, cv = int((cc >> 2) & 3u) - 1;

  // digits and carry-in bits
  uint32_t bu = 0, bv = 0;
#pragma unroll
  for (int q = 0; q < kZgenPer; ++q) {
    const int64_t j = t0 + q;
    if (j < c1) {
      bu |= uint32_t(cu) << q;
      bv |= uint32_t(cv) << q;
      const uint64_t wu = window_at(Lu, j * b - a.lead, b);
      const uint64_t wv = window_at(Lv, j * b - a.lead, b);
      digu[j - c0] = int32_t(split_digit(wu, cu, b, j == count - 1 || !mc.balanced));
      digv[j - c0] = int32_t(split_digit(wv, cv, b, j == count - 1 || !mc.balanced));
      if (!((pu >> q) & 1u)) cu = int((gu >> q) & 1u);
      if (!((pv >> q) & 1u)) cv = int((gv >> q) & 1u);
    }
  }
  // the next block's first lam-1 digits (carry out of this block known)
  if (t0 < c1 && t0 + kZgenPer >= c1) {
    for (int q = 0; q < ext; ++q) {
      const int64_t j = c1 + q;
      if (j >= N) break;
      const uint64_t wu = window_at(Lu, j * b - a.lead, b);
      const uint64_t wv = window_at(Lv, j * b - a.lead, b);
      digu[j - c0] = int32_t(split_digit(wu, cu, b, j == count - 1 || !mc.balanced));
      digv[j - c0] = int32_t(split_digit(wv, cv, b, j == count - 1 || !mc.balanced));
      cu = mc.balanced ? tf_apply(split_tf(wu, b), cu) : 0;
      cv = mc.balanced ? tf_apply(split_tf(wv, b), cv) : 0;
    }
  }
  {
    const uint32_t ou = __shfl_xor_sync(0xffffffffu, bu, 1);
    const uint32_t ov = __shfl_xor_sync(0xffffffffu, bv, 1);
    if ((tid & 1) == 0 && t0 < count) {
      a.cbits_u[t0 >> 5] = bu | (ou << 16);
      a.cbits_v[t0 >> 5] = bv | (ov << 16);
    }
  }
  if (blk == 0 && tid == 0 && (a.n & 63)) {
    const uint64_t hm = ~0ull << (a.n & 63);
    if ((__ldg(a.u + a.nlimbs - 1) | __ldg(a.v + a.nlimbs - 1)) & hm)
      atomicOr(&a.status->flags, uint32_t(kFlagInputRange));
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(a.scan.ctr + 1, 1ull) == gridDim.x - 1) {
      a.scan.ctr[0] = 0;
      a.scan.ctr[1] = 0;
    }
  }

  // outputs
  const int64_t ce = min(c1, N);
  if (mc.mode == kModeFull) {
    for (int64_t j = c0 + tid; j < ce; j += kZgenThreads)
      a.z[j] = make_double2(double(digu[j - c0]), double(digv[j - c0]));
    return;
  }
  const double Nd = double(N);
  const int fam = (mc.mode == kModeLow) ? 0 : 2;
  auto Du = [&](int64_t i) -> double {
    return (i < N) ? double(digu[i - c0]) : double(s_wrap[0][i - N]);
  };
  auto Dv = [&](int64_t i) -> double {
    return (i < N) ? double(digv[i - c0]) : double(s_wrap[1][i - N]);
  };
  for (int64_t j = c0 + ext + tid; j < ce + ext; j += kZgenThreads) {
    double au = 0.0, av = 0.0;
    RowLoopDown<kMaxLambda>::run([&](auto rc) {
      constexpr int r = decltype(rc)::value;
      if (r < lam) {
        const int64_t i = j - r;  // chunk, in [c0, c1 + ext)
        int64_t k = i;
        if (k >= N) k -= N;
        const double cf = coef_r<r>(fam, double(k), Nd, mc.cpre[r]);
        au += Du(i) * cf;
        av += Dv(i) * cf;
      }
    });
    a.z[j >= N ? j - N : j] = make_double2(au, av);
  }
}

}  // namespace tmg
