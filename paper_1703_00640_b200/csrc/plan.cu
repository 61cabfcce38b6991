// Host-side plan construction: transform shape, radix schedules, exact
// twiddle tables, map constants (maps_f64.cpp:192-245 of the reference).
#include "plan.hpp"

#include <atomic>

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "../../include/truncmul_b200.h"

namespace tmg {
std::vector<int> mid_ct_radices(uint32_t C);  // k_multipass.cu

#define TMG_CUDA(call)                                                     \
  do {                                                                     \
    cudaError_t e_ = (call);                                               \
    if (e_ != cudaSuccess) {                                               \
      (void)cudaGetLastError(); /* clear a non-sticky error */             \
      throw Error(TMG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    }                                                                      \
  } while (0)

DevBuf::~DevBuf() {
  if (p) cudaFree(p);
}

std::atomic<uint64_t> g_devbuf_generation{0};

void DevBuf::ensure(size_t nbytes) {
  if (nbytes <= bytes) return;
  // a reallocation invalidates every captured graph that used the old buffer
  if (p) g_devbuf_generation.fetch_add(1);
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
  TMG_CUDA(cudaMalloc(&p, nbytes));
  bytes = nbytes;
}

namespace {

// e^{-2 pi i x / R} in long double with octant reduction, rounded once.
void twiddle(uint64_t x, uint64_t R, double* re, double* im) {
  x %= R;
  const unsigned __int128 t = (unsigned __int128)x * 8u;
  const uint64_t o = uint64_t(t / R);
  const uint64_t rem = uint64_t(t - (unsigned __int128)o * R);
  const long double q = 0.785398163397448309615660845819875721L;  // pi/4
  long double c, s;
  if ((o & 1) == 0) {
    long double th = (long double)rem / (long double)R * q;
    long double ct = cosl(th), st = sinl(th);
    switch (o) {
      case 0: c = ct; s = st; break;
      case 2: c = -st; s = ct; break;
      case 4: c = -ct; s = -st; break;
      default: c = st; s = -ct; break;  // 6
    }
  } else {
    long double th = (long double)(R - rem) / (long double)R * q;
    long double ct = cosl(th), st = sinl(th);
    switch (o) {
      case 1: c = st; s = ct; break;
      case 3: c = -ct; s = st; break;
      case 5: c = -st; s = -ct; break;
      default: c = ct; s = -st; break;  // 7
    }
  }
  *re = double(c);
  *im = double(-s);
}

std::vector<double2> host_table(uint64_t L, uint64_t step, uint64_t count) {
  std::vector<double2> t(count);
  for (uint64_t i = 0; i < count; ++i) {
    double re, im;
    twiddle(i * step, L, &re, &im);
    t[i] = make_double2(re, im);
  }
  return t;
}

// maxrad 16 (default) or 8: the largest power-of-two radix used.
std::vector<int> radix_schedule(uint32_t R, int maxrad = 16) {
  std::array<uint32_t, 4> e;
  if (!factor_2357(R, e)) throw Error(TMG_ERR_UNSUPPORTED_LENGTH, "radix_schedule: not 2357-smooth");
  std::vector<int> rad;
  uint32_t e2 = e[0];
  if (maxrad == 8)
    while (e2 >= 3) { rad.push_back(8); e2 -= 3; }
  while (e2 >= 4) { rad.push_back(16); e2 -= 4; }
  if (e2 == 3) rad.push_back(8);
  if (e2 == 2) rad.push_back(4);
  if (e2 == 1) rad.push_back(2);
  for (uint32_t i = 0; i < e[1]; ++i) rad.push_back(3);
  for (uint32_t i = 0; i < e[2]; ++i) rad.push_back(5);
  for (uint32_t i = 0; i < e[3]; ++i) rad.push_back(7);
  if (rad.size() > size_t(kMaxStages))
    throw Error(TMG_ERR_UNSUPPORTED_LENGTH, "radix_schedule: too many stages");
  return rad;
}

uint32_t largest_pow2_divisor(uint64_t x) {
  uint32_t p = 1;
  while (x % (uint64_t(p) * 2) == 0 && p < (1u << 30)) p *= 2;
  return p;
}

// Columns per CTA for a column pass over length R with ncols columns.
uint32_t pick_logc(uint32_t R, uint64_t ncols, size_t smem_cap) {
  const uint32_t p2 = largest_pow2_divisor(ncols);
  uint32_t best = 0;
  for (uint32_t lc = 0; lc <= 6; ++lc) {
    const uint32_t c = 1u << lc;
    if (c > p2) break;
    const uint64_t thr = (uint64_t(R) * c + 15) / 16;
    const size_t smem = size_t(padded_len(R * c)) * 16 + size_t(R) * 16;
    if (thr > 512 || smem > smem_cap) break;
    best = lc;
    if (thr >= 256 && c >= 4) break;
  }
  return best;
}

int threads_for(uint64_t elems) {
  uint64_t t = (elems + 15) / 16;
  t = (t + 31) / 32 * 32;
  if (t < 32) t = 32;
  return int(t);
}

}  // namespace

const double2* TwiddleCache::table(uint32_t R) {
  auto it = tables_.find(R);
  if (it != tables_.end()) return it->second->as<double2>();
  auto h = host_table(R, 1, R);
  auto buf = std::make_unique<DevBuf>();
  buf->ensure(h.size() * sizeof(double2));
  TMG_CUDA(cudaMemcpy(buf->p, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice));
  const double2* p = buf->as<double2>();
  tables_[R] = std::move(buf);
  return p;
}

TwGlobal TwiddleCache::global(uint64_t L) {
  auto it = glob_.find(L);
  if (it == glob_.end()) {
    uint32_t S = 0;
    while ((uint64_t(1) << (2 * S)) < L) ++S;  // 2^S ~ sqrt(L)
    const uint64_t nlo = uint64_t(1) << S;
    const uint64_t nhi = (L + nlo - 1) / nlo;
    auto lo = host_table(L, 1, nlo);
    auto hi = host_table(L, nlo, nhi);
    auto buf = std::make_unique<DevBuf>();
    buf->ensure((nlo + nhi) * sizeof(double2));
    TMG_CUDA(cudaMemcpy(buf->p, lo.data(), nlo * sizeof(double2), cudaMemcpyHostToDevice));
    TMG_CUDA(cudaMemcpy(buf->as<double2>() + nlo, hi.data(), nhi * sizeof(double2),
                        cudaMemcpyHostToDevice));
    glob_S_[L] = S;
    it = glob_.emplace(L, std::move(buf)).first;
  }
  TwGlobal g;
  g.S = glob_S_[L];
  g.lo = it->second->as<double2>();
  g.hi = g.lo + (uint64_t(1) << g.S);
  return g;
}

const double2* TwiddleCache::stage_table(uint32_t R, int maxrad) {
  return stage_table(R, radix_schedule(R, maxrad));
}

const double2* TwiddleCache::stage_table(uint32_t R, const std::vector<int>& rad) {
  std::string key = std::to_string(R);
  for (int r : rad) key += "," + std::to_string(r);
  auto it = stages_.find(key);
  if (it != stages_.end()) return it->second->as<double2>();
  std::vector<double2> h;
  uint32_t Ns = 1;
  for (size_t s = 0; s < rad.size(); ++s) {
    const uint32_t r = uint32_t(rad[s]);
    if (s > 0) {
      for (uint32_t q = 1; q < r; ++q)
        for (uint32_t j = 0; j < Ns; ++j) {
          double re, im;
          twiddle(uint64_t(j) * q, uint64_t(Ns) * r, &re, &im);
          h.push_back(make_double2(re, im));
        }
    }
    Ns *= r;
  }
  if (h.empty()) h.push_back(make_double2(1.0, 0.0));
  auto buf = std::make_unique<DevBuf>();
  buf->ensure(h.size() * sizeof(double2));
  TMG_CUDA(cudaMemcpy(buf->p, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice));
  const double2* p = buf->as<double2>();
  stages_[key] = std::move(buf);
  return p;
}

SubFft make_subfft(uint32_t R, const double2* tw, uint32_t tw_stride, TwiddleCache* cache,
                   int maxrad) {
  return make_subfft_rad(R, radix_schedule(R, maxrad), tw, tw_stride, cache);
}

// Sub-transform with an explicit radix schedule (compile-time column passes:
// composite radices 10 and 12 that the runtime passes do not dispatch).
SubFft make_subfft_rad(uint32_t R, const std::vector<int>& rad, const double2* tw,
                       uint32_t tw_stride, TwiddleCache* cache) {
  SubFft s;
  std::memset(&s, 0, sizeof(s));
  s.R = R;
  s.tw = tw;
  s.twlen = R * tw_stride;
  s.nst = int32_t(rad.size());
  uint32_t Ns = 1, off = 0;
  for (size_t i = 0; i < rad.size(); ++i) {
    s.rad[i] = rad[i];
    s.Ns[i] = Ns;
    s.twstep[i] = R / (Ns * uint32_t(rad[i])) * tw_stride;
    s.fdNs[i] = make_fastdiv(Ns);
    s.toff[i] = off;
    s.qmul[i] = 1;
    if (i > 0) off += Ns * (uint32_t(rad[i]) - 1);
    Ns *= uint32_t(rad[i]);
  }
  s.stablen = off > 0 ? off : 1;
  s.stab = cache ? cache->stage_table(R, rad) : nullptr;
  return s;
}

// Inverse sub-transform whose stage twiddles are read from the forward
// table of another length (same Ns per stage, radix dividing the forward
// radix); returns false when the schedules do not line up.
bool map_stages(SubFft& inv, const SubFft& fwd) {
  // all-or-nothing: a partial mapping would leave stages indexing the
  // forward table's offsets inside the inverse's own table
  SubFft m = inv;
  for (int i = 1; i < m.nst; ++i) {
    bool found = false;
    for (int f = 1; f < fwd.nst; ++f) {
      if (fwd.Ns[f] == m.Ns[i] && fwd.rad[f] % m.rad[i] == 0) {
        m.toff[i] = fwd.toff[f];
        m.qmul[i] = uint32_t(fwd.rad[f] / m.rad[i]);
        found = true;
        break;
      }
    }
    if (!found) return false;
  }
  m.stab = fwd.stab;
  m.stablen = fwd.stablen;
  inv = m;
  return true;
}

MapConsts make_map_consts(const Params& p) {
  MapConsts m;
  std::memset(&m, 0, sizeof(m));
  m.mode = int32_t(p.mode);
  m.b = p.b;
  m.N = p.N;
  m.lambda = int32_t(p.lambda);
  m.balanced = p.signed_split ? 1 : 0;
  m.step = std::ldexp(1.0, -p.b);
  m.scale_out = (p.mode == PMode::kFull) ? 1.0 : std::ldexp(1.0, p.b);
  m.cofactor_scaled = 1.0;
  if (p.mode == PMode::kFull) return m;
  if (p.lambda > kMaxLambda) throw Error(TMG_ERR_UNSUPPORTED, "lambda above the GPU limit of 8");
  // row scales sgn / (r! N^r 2^{rb}) (series.cpp:146-183 closed forms)
  for (int r = 0; r < p.lambda; ++r) {
    long double den = 1.0L;
    for (int i = 1; i <= r; ++i) den *= (long double)i * (long double)p.N;
    den = ldexpl(den, r * p.b);
    const long double v = 1.0L / den;
    const bool odd = (r & 1) != 0;
    if (p.mode == PMode::kLow) {
      m.cpre[r] = double(odd ? -v : v);   // alpha
      m.cpost[r] = double(v);             // beta
    } else {
      m.cpre[r] = double(v);              // gamma
      m.cpost[r] = double(odd ? -v : v);  // delta
    }
  }
  if (p.mode == PMode::kHigh) {
    const int64_t N = p.N;
    const int64_t total_bits = N * int64_t(p.b);
    double inv_root;
    std::vector<double> fold;
    if (total_bits >= 64) {
      inv_root = std::ldexp(1.0, -p.b);
      const int neg = int(std::min<int64_t>(total_bits, 1100));
      m.root_neg_n = std::ldexp(1.0, -neg);
      m.cofactor_scaled = 1.0 - double(N) * m.root_neg_n;
      for (int64_t i = 0; i < N && i * p.b <= 80; ++i)
        fold.push_back(std::ldexp(1.0, int(-i * p.b)));
    } else {
      // real root of B(X) = X^{N+1} - 2^b X^N + 2^b just below 2^b (Newton,
      // maps.cpp:31-63), then the double ladders of maps_f64.cpp:226-238.
      long double top = ldexpl(1.0L, p.b), x = top;
      for (int it = 0; it < 200; ++it) {
        long double xn = powl(x, (long double)N);
        long double val = xn * (x - top) + top;
        long double slope = powl(x, (long double)(N - 1)) * ((N + 1) * x - N * top);
        if (slope == 0) break;
        long double nx = x - val / slope;
        if (nx > top) nx = top;
        if (fabsl(nx - x) <= ldexpl(fabsl(x), -62)) { x = nx; break; }
        x = nx;
      }
      const double root = double(x);
      inv_root = 1.0 / root;
      double ipow = inv_root;
      for (int64_t i = 0; i < N; ++i) {
        fold.push_back(std::ldexp(ipow, p.b));
        ipow *= inv_root;
      }
      double inv_n = 1.0;
      for (int64_t i = 0; i < N; ++i) inv_n *= inv_root;
      m.root_neg_n = inv_n;
      m.cofactor_scaled = 1.0 - double(N) * std::ldexp(inv_n * inv_root, p.b);
      // the kernels use only the leading entries; keep what fits
      if (fold.size() > size_t(kMaxFold)) fold.resize(kMaxFold);
    }
    if (fold.size() > size_t(kMaxFold)) throw Error(TMG_ERR_UNSUPPORTED, "fold row too long");
    m.nfold = int32_t(fold.size());
    for (size_t i = 0; i < fold.size(); ++i) m.fold[i] = fold[i];
    // root-channel ladders (maps_f64.cpp:291-297, 364-370)
    double ip = 1.0;
    int d = 0;
    m.ipow[0] = 1.0;
    for (d = 0; d <= N; ++d) {
      double nxt = ip * inv_root;
      if (d + 1 < kMaxRootTerms) m.ipow[d + 1] = nxt;
      ip = nxt;
      if (ip < 1e-30) break;
    }
    const int D = int(std::min<int64_t>(d, N));
    if (D + 1 > kMaxRootTerms) throw Error(TMG_ERR_UNSUPPORTED, "root ladder too long");
    m.nroot = D + 1;
    m.nhrho = D;
  }
  return m;
}

std::unique_ptr<Plan> build_plan(const Params& p, TwiddleCache& tw, const PlanOptions& opt) {
  auto pl = std::make_unique<Plan>();
  pl->params = p;
  pl->nlimbs = (p.n + 63) / 64;
  pl->out_limbs = output_limbs(p.mode, p.n);
  if (p.mode == PMode::kOracleFallback) {
    pl->kind = 0;
    pl->kernels = 1;
    return pl;
  }
  if (p.backend != Backend::kFft)
    throw Error(TMG_ERR_UNSUPPORTED, "GPU products run the FFT backend only");
  if (p.b > 48) throw Error(TMG_ERR_UNSUPPORTED, "chunk width above 48 bits");
  const int64_t N = p.N;
  const int64_t L = transform_length(p.mode, N);
  pl->L = L;
  pl->mc = make_map_consts(p);
  if (L % 4 != 0) throw Error(TMG_ERR_UNSUPPORTED, "transform length must be divisible by 4");
  if (p.mode != PMode::kFull && N < 2 * p.lambda + pl->mc.nfold + 2)
    throw Error(TMG_ERR_UNSUPPORTED, "transform length too short for the series maps");
  pl->count = (p.mode == PMode::kHigh) ? N + 1 : N;
  pl->lead = (p.mode == PMode::kHigh) ? (N + 1) * int64_t(p.b) - p.n : 0;
  const int b = p.b;
  if (p.mode == PMode::kFull) {
    pl->K = L;
    pl->ML = ((L - 1) * b + 64 + 63) / 64 + 1;
    pl->ML = std::max(pl->ML, pl->out_limbs);
  } else if (p.mode == PMode::kLow) {
    pl->K = N - 1;
    pl->ML = pl->out_limbs;
  } else {
    pl->K = N + 1;
    pl->shift_s = int32_t(2 * b + pl->lead);
    if (pl->shift_s < 1) throw Error(TMG_ERR_UNSUPPORTED, "high product shift out of range");
    pl->ML = (N * b + 64 + 64 + 63) / 64 + 1;
    pl->ML = std::max<int64_t>(pl->ML, pl->out_limbs + (pl->shift_s >> 6) + 2);
  }

  // One CTA computes the whole product up to L = 4096; a single product of
  // 4096 < L <= 8192 runs the multi-pass pipeline over many SMs (2^16 low:
  // 78 us in one CTA), and batches of it the fused kernel (small_batch).
  if (L <= kSmallSingleMaxL) {
    pl->kind = 1;
    const double2* t = tw.table(uint32_t(L));
    pl->fwd = make_subfft(uint32_t(L), t, 1, nullptr);
    pl->inv = make_subfft(uint32_t(L / 2), t, 2, nullptr);
    pl->small_threads = threads_for(uint64_t(L));
    pl->small_smem = small_smem_bytes(L, pl->nlimbs);
    pl->kernels = 1;
    return pl;
  }

  // batches of this length can still run the fused kernel, one CTA per
  // product, when the whole product fits one CTA's shared memory
  if (L <= kSmallBatchMaxL && threads_for(uint64_t(L)) <= kSmallBatchMaxThreads &&
      small_smem_bytes(L, pl->nlimbs) <= kMaxDynSmem) {
    const double2* t = tw.table(uint32_t(L));
    pl->fwd = make_subfft(uint32_t(L), t, 1, nullptr);
    pl->inv = make_subfft(uint32_t(L / 2), t, 2, nullptr);
    pl->small_threads = threads_for(uint64_t(L));
    pl->small_smem = small_smem_bytes(L, pl->nlimbs);
    pl->small_batch = true;
  }

  // multi-pass: C = row length (even, <= 4096), A (and B) column lengths
  const uint64_t UL = uint64_t(L);
  if (UL >= (uint64_t(1) << 32)) throw Error(TMG_ERR_UNSUPPORTED, "transform length above 2^32");
  // the largest even row length whose row pass (two rows plus the stage
  // twiddles, shared between the forward and inverse schedules when they
  // line up) fits in one CTA's shared memory
  uint32_t C = 0;
  // Mid-size products have few 4096-point row pairs (11 at 2^20), and the
  // row pass then costs one pair's latency.  Below 32 pairs the compiled
  // 2048- / 1024-point row passes are taken: among the lengths with at
  // least 20 pairs (else all), the longest whose column length has a
  // compiled column pass, else the longest (else the shortest)
  // (tools/kernel_times.py with TMG_OPT_MAX_ROW: 2^20 low 45.4 -> 39.9 us,
  // full 58.2 -> 40.6, 2^18 low 40.7 -> 37.8).
  if (!opt.max_row && !opt.generic_row && UL <= (uint64_t(1) << 21) &&
      !(UL % 4096 == 0 && UL / 4096 / 2 + 1 >= 32)) {
    uint32_t pick = 0, pick_col = 0, smallest = 0;
    bool any20 = false;
    for (uint32_t c : {4096u, 2048u, 1024u})
      if (UL % c == 0 && UL / c / 2 + 1 >= 20) any20 = true;
    for (uint32_t c : {4096u, 2048u, 1024u}) {
      if (UL % c || (c != 4096 && mid_ct_radices(c).empty())) continue;
      smallest = c;
      if (any20 && UL / c / 2 + 1 < 20) continue;
      if (!pick) pick = c;
      if (!pick_col && UL / c <= 2048 && colct_for(uint32_t(UL / c), 1)) pick_col = c;
    }
    C = pick_col ? pick_col : (any20 ? pick : smallest);
  }
  for (uint32_t c = opt.max_row ? std::min<uint32_t>(4096, opt.max_row) : 4096; C == 0 && c >= 16; --c) {
    if (c % 2 || UL % c) continue;
    SubFft f = make_subfft(c, nullptr, 1, nullptr);
    SubFft i = make_subfft(c / 2, nullptr, 2, nullptr);
    const bool shared = map_stages(i, f);
    if (mid_smem_bytes(c, shared ? 0u : i.stablen) > kMaxDynSmem) continue;
    C = c;
    break;
  }
  if (C == 0) throw Error(TMG_ERR_UNSUPPORTED, "no row length divides L");
  const uint64_t AB = UL / C;
  uint32_t A = 0, B = 1;
  // opt.force_three_pass (testing): split even short column lengths into A x B
  if (AB <= 2048 && !(opt.force_three_pass && AB >= 64)) {
    A = uint32_t(AB);
    pl->kind = 2;
  } else {
    // balanced split: the divisor of AB closest to sqrt(AB), both <= 2048
    const double root = std::sqrt(double(AB));
    double bestd = 1e300;
    for (uint32_t a = 16; a <= 2048; ++a) {
      if (AB % a || AB / a > 2048 || AB / a < 4 || (a % 4)) continue;
      const double d = std::fabs(std::log(double(a) / root));
      if (d < bestd) { bestd = d; A = a; }
    }
    if (A == 0) throw Error(TMG_ERR_UNSUPPORTED, "cannot factor the transform length");
    B = uint32_t(AB / A);
    pl->kind = 3;
  }
  pl->A = A;
  pl->B = B;
  pl->C = C;
  const size_t cap = 200 * 1024;
  pl->twL = tw.global(UL);
  const double2* tA = tw.table(A);
  const double2* tC = tw.table(C);
  pl->fA = make_subfft(A, tA, 1, &tw);
  pl->iA = pl->fA;
  pl->fC = make_subfft(C, tC, 1, &tw);
  pl->iC = make_subfft(C / 2, tC, 2, &tw);
  pl->mid_shared_table = map_stages(pl->iC, pl->fC);
  // compiled row passes of 2048 / 1024 (k_mid_2048 / k_mid_1024): their own
  // forward schedule's stage table; the inverse reads it at every second entry
  pl->mid_ct = false;
  if (!opt.generic_row) {
    const std::vector<int> mr = mid_ct_radices(C);
    if (!mr.empty()) {
      pl->fC = make_subfft_rad(C, mr, tC, 1, &tw);
      pl->mid_ct = true;
    }
  }
  const int col_logc_cap = 6;  // columns per CTA of the column passes: at most 64
  pl->logc_f1 = std::min<uint32_t>(pick_logc(A, UL / A, cap), uint32_t(col_logc_cap));
  pl->thr_f1 = threads_for(uint64_t(A) << pl->logc_f1);
  pl->smem_f1 = f1_smem_bytes(A, 1u << pl->logc_f1) +
                f1_tw_bytes(A, 1u << pl->logc_f1, uint32_t(pl->thr_f1));
  pl->logc_il = std::min<uint32_t>(pick_logc(A, C / 2, cap), uint32_t(col_logc_cap));
  pl->thr_il = threads_for(uint64_t(A) << pl->logc_il);
  pl->smem_il = col_smem_bytes(A, 1u << pl->logc_il);
  if (pl->kind == 3) {
    const double2* tB = tw.table(B);
    pl->fB = make_subfft(B, tB, 1, &tw);
    pl->iB = pl->fB;
    pl->logc_f2 = pick_logc(B, C, cap);
    pl->thr_f2 = threads_for(uint64_t(B) << pl->logc_f2);
    pl->smem_f2 = col_smem_bytes(B, 1u << pl->logc_f2);
    pl->logc_i2 = pick_logc(B, C / 2, cap);
    pl->thr_i2 = threads_for(uint64_t(B) << pl->logc_i2);
    pl->smem_i2 = col_smem_bytes(B, 1u << pl->logc_i2);
  }
  // Ping-pong column passes (k_*_pp): radix <= 8 schedules, two tiles in
  // shared memory, up to 1024 threads.  Used whenever the two tiles of at
  // least one column fit.
  auto pp_logc = [&](uint32_t R, uint64_t ncols) -> int {
    const uint32_t p2 = largest_pow2_divisor(ncols);
    int best = -1;
    for (uint32_t lc = 0; lc <= 6 && (1u << lc) <= p2; ++lc)
      if (colpp_smem_bytes(R, 1u << lc) <= size_t(220) * 1024) best = int(lc);
    return best;
  };
  auto pp_threads = [](uint32_t R, uint32_t lc) {
    uint64_t t = ((uint64_t(R) << lc) / 8 + 31) / 32 * 32;
    return int(std::min<uint64_t>(kColPPThreads, std::max<uint64_t>(128, t)));
  };
  pl->colpp = false;
  {
    const int lf1 = pp_logc(A, UL / A), lil = pp_logc(A, C / 2);
    int lf2 = 0, li2 = 0;
    if (pl->kind == 3) {
      lf2 = pp_logc(B, C);
      li2 = pp_logc(B, C / 2);
    }
    // only when the two tiles hold as many columns as the single-buffer
    // pass (fewer columns mean shorter global segments, which costs more
    // than the extra warps gain: A = 1792 measured 126 -> 166 us)
    if (lf1 >= int(pl->logc_f1) && lil >= int(pl->logc_il) && lf2 >= 0 && li2 >= 0) {
      pl->colpp = true;
      pl->fA = make_subfft(A, tA, 1, &tw, 8);
      pl->iA = pl->fA;
      pl->logc_f1 = uint32_t(std::min(lf1, col_logc_cap));
      pl->thr_f1 = pp_threads(A, pl->logc_f1);
      pl->smem_f1 = colpp_smem_bytes(A, 1u << pl->logc_f1) +
                    f1_tw_bytes(A, 1u << pl->logc_f1, uint32_t(pl->thr_f1));
      pl->logc_il = uint32_t(std::min(lil, col_logc_cap));
      pl->thr_il = pp_threads(A, pl->logc_il);
      pl->smem_il = colpp_smem_bytes(A, 1u << pl->logc_il);
      if (pl->kind == 3) {
        pl->fB = make_subfft(B, tw.table(B), 1, &tw, 8);
        pl->iB = pl->fB;
        pl->logc_f2 = uint32_t(lf2);
        pl->thr_f2 = pp_threads(B, pl->logc_f2);
        pl->smem_f2 = colpp_smem_bytes(B, 1u << pl->logc_f2);
        pl->logc_i2 = uint32_t(li2);
        pl->thr_i2 = pp_threads(B, pl->logc_i2);
        pl->smem_i2 = colpp_smem_bytes(B, 1u << pl->logc_i2);
      }
    }
  }
  // Compile-time column passes where the column length and its radix-16
  // schedule match a compiled shape (two-pass plans only).
  pl->colct = nullptr;
  pl->colct_il = nullptr;
  pl->colct_b = nullptr;
  if ((pl->kind == 2 || pl->kind == 3) && !opt.generic_columns) {
    const ColCtShape* sf1 = colct_for(A, 1);
    const ColCtShape* sil = colct_for(A, 2);
    // three-pass plans also need the middle passes' shape over B
    const ColCtShape* scb = pl->kind == 3 ? colct_for(B, 4) : nullptr;
    bool same = sf1 && sil && (pl->kind == 2 || scb);
    for (int i = 0; same && i < 4; ++i) same = sf1->rad[i] == sil->rad[i];
    if (same && scb) {
      const uint32_t cb = 1u << scb->logc;
      std::vector<int> radb;
      for (int i = 0; i < 4 && scb->rad[i]; ++i) radb.push_back(scb->rad[i]);
      SubFft fb = make_subfft_rad(B, radb, tw.table(B), 1, &tw);
      const size_t sb = colct_smem_bytes(B, cb, fb.stablen, scb->radl);
      if (C % cb == 0 && (C / 2) % cb == 0 && sb <= kMaxDynSmem) {
        pl->colct_b = scb;
        pl->fB = fb;
        pl->iB = fb;
        pl->logc_f2 = pl->logc_i2 = uint32_t(scb->logc);
        pl->thr_f2 = pl->thr_i2 = scb->nthr;
        pl->smem_f2 = pl->smem_i2 = sb;
      } else {
        same = false;
      }
    }
    if (same) {
      std::vector<int> rad;
      for (int i = 0; i < 4 && sf1->rad[i]; ++i) rad.push_back(sf1->rad[i]);
      SubFft f16 = make_subfft_rad(A, rad, tA, 1, &tw);
      const uint32_t cf = 1u << sf1->logc, ci = 1u << sil->logc;
      const size_t sf = colct_smem_bytes(A, cf, f16.stablen, sf1->radl);
      const size_t si = colct_smem_bytes(A, ci, f16.stablen, 0);
      if ((UL / A) % cf == 0 && (C / 2) % ci == 0 && sf <= kMaxDynSmem && si <= kMaxDynSmem) {
        pl->colct = sf1;
        pl->colct_il = sil;
        pl->colpp = false;
        pl->fA = f16;
        pl->iA = f16;
        pl->logc_f1 = uint32_t(sf1->logc);
        pl->logc_il = uint32_t(sil->logc);
        pl->thr_f1 = sf1->nthr;
        pl->thr_il = sil->nthr;
        pl->smem_f1 = sf;
        pl->smem_il = si;
      }
    }
  }
  // The first column pass applies the pre-map itself where a compiled shape
  // with the same schedule and at least lambda - 1 columns per CTA exists:
  // k_zgen then stores digits (4 or 8 bytes per chunk, not a 16-byte
  // coefficient) and k_f1d_ct reads them.
  pl->f1d = nullptr;
  pl->zdig = 0;
  if (pl->colct && !opt.premap_in_zgen && !opt.z_natural && b <= 30) {
    const F1DShape* sd = f1d_for(A);
    bool same = sd != nullptr;
    for (int i = 0; same && i < 4; ++i) same = sd->rad[i] == pl->colct->rad[i];
    const int lam = p.mode == PMode::kFull ? 0 : int(pl->mc.lambda);
    const int dig = zdig_kind(int(b));
    const int var = f1d_variant(lam, dig);
    if (same && var >= 0 && sd->fn[var] && (lam == 0 || p.N == L)) {
      const uint32_t cd = 1u << sd->logc;
      const uint32_t zrows = uint32_t((p.N + (UL / A) - 1) / (UL / A));
      const size_t sf = f1d_smem_bytes(A, cd, pl->fA.stablen, sd->radl, zrows, lam, dig);
      if ((UL / A) % cd == 0 && sf <= kMaxDynSmem) {
        pl->f1d = sd->fn[var];
        pl->zdig = dig;
        pl->logc_f1 = uint32_t(sd->logc);
        pl->thr_f1 = sd->nthr;
        pl->smem_f1 = sf;
      }
    }
  }
  if (pl->colct) {
    pl->f1_stw = false;
  } else {
    // staged F1 twiddles where the thread count is a multiple of the
    // columns per CTA and the extra table still fits
    const uint32_t c1 = 1u << pl->logc_f1;
    const size_t extra = f1_tw_bytes(A, c1, uint32_t(pl->thr_f1));
    pl->f1_stw = extra > 0 && pl->smem_f1 <= kMaxDynSmem;
    if (!pl->f1_stw) pl->smem_f1 -= extra;
  }
  pl->thr_mid = threads_for(uint64_t(2) * C);
  pl->smem_mid = mid_smem_bytes(C, pl->mid_shared_table ? 0u : pl->iC.stablen);
  const int64_t LB = kCarryThreads * kCarryPerThread;
  pl->smem_carry = carry_smem(b);
  (void)LB;
  pl->kernels = ((pl->kind == 2) ? 5 : 7) + (p.mode == PMode::kHigh ? 1 : 0);
  pl->smem_zgen = zgen_smem(b);
  return pl;
}

size_t small_smem_bytes(int64_t L, int64_t nlimbs) {
  // the transform plus kMaxLambda + 1 slots for the shifted digits (k_small.cu)
  return size_t(padded_len(uint32_t(L) + kMaxLambda + 1)) * 16 + size_t(2 * nlimbs) * 8 + 32 * 4 +
         8 * 8 +
         size_t(tw_smem_len(uint32_t(L))) * 16;
}

}  // namespace tmg
