// Context, launch orchestration and the extern "C" boundary
// (include/truncmul_b200.h).  The launch sequence of one product follows the
// reference's pipeline order (products_f64.cpp:106-171):
//   split -> pre-map -> forward transforms -> pointwise -> inverse ->
//   post-map -> round/accumulate -> carry, with the tripwires of
//   products_f64.cpp:16-27 and 137-169 reported through a device status word.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/truncmul_b200.h"
#include "kernels.cuh"
#include <unordered_map>
#include "params.hpp"
#include "plan.hpp"

namespace tmg {

#define TMG_CUDA(call)                                                     \
  do {                                                                     \
    cudaError_t e_ = (call);                                               \
    if (e_ != cudaSuccess) {                                               \
      (void)cudaGetLastError(); /* clear a non-sticky error */             \
      throw Error(TMG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    }                                                                      \
  } while (0)

thread_local std::string g_last_error;

struct ScanSlot {
  DevBuf state;     // look-back words
  DevBuf ctr;       // ticket / done counters
  uint32_t epoch = 0;
  ScanState next(size_t blocks) {
    const size_t need = std::max<size_t>(blocks, 1) * 8;
    if (need > state.bytes) {
      state.ensure(need);
      TMG_CUDA(cudaMemset(state.p, 0, state.bytes));
    }
    if (!ctr.p) {
      ctr.ensure(64);
      TMG_CUDA(cudaMemset(ctr.p, 0, 64));
    }
    ScanState s;
    s.state = state.as<unsigned long long>();
    s.ctr = ctr.as<unsigned long long>();
    s.epoch = ++epoch;
    return s;
  }
};

// Optional per-kernel CUDA-event timing on the launching stream.
struct Profiler {
  bool on = false;
  struct Rec {
    std::string name;
    cudaEvent_t a, b;
    double bytes;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) throw Error(TMG_ERR_CUDA, "cudaEventCreate");
    return e;
  }
};

// Per-product scratch of the multi-pass pipeline: transform buffers, split
// carry bits, aggregates, completion tickets and the product's status word.
// The context owns one for single products; a batch runs its products on up
// to kMaxBatchStreams workspaces, each on its own stream.
struct Workspace {
  DevBuf work_t, work_c, work_z, cbu, cbv, aux, tbuf, aggs, zaggs, ticket, hticket, status;
  DevBuf gen;  // look-back generation of k_zgen / k_carry_lb, advanced by the row pass (zeroed)
  DevBuf zlb;  // k_zgen look-back words (zeroed)
  ScanSlot scan_c;  // look-back state of the single-pass carry (k_carry)
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
  ~Workspace() {
    if (done) cudaEventDestroy(done);
    if (stream) cudaStreamDestroy(stream);
  }
};
constexpr int kMaxBatchStreams = 32;
// k_carry_patch scans the carry aggregates itself up to this many carry blocks
constexpr unsigned kPatchScanMaxBlocks = 4096;
constexpr int64_t kGraphMinBatch = 4;  // batches replayed as graphs from this size

// Alternative code paths a context can select for testing and diagnostics
// (tmg_context_set_option, TMG_OPT_*); every default is the measured-best
// configuration, and nothing is read from the environment.
struct Options {
  PlanOptions plan;             // TMG_OPT_GENERIC_COLUMN_PASSES, TMG_OPT_FORCE_THREE_PASS
  bool generic_row = false;     // TMG_OPT_GENERIC_ROW_PASS
  bool lookback_carry = false;  // TMG_OPT_LOOKBACK_CARRY
  int carry_kernels = 0;        // TMG_OPT_CARRY_KERNELS (0 by size)
  bool generic_runs = false;    // TMG_OPT_GENERIC_RUNS
  bool old_split = false;       // TMG_OPT_SPLIT_KERNEL
  bool zstat_split = false;     // TMG_OPT_SPLIT_AGGREGATES
  long patch_scan_max = long(kPatchScanMaxBlocks);  // TMG_OPT_PATCH_SCAN_MAX
  bool no_pdl = false;          // TMG_OPT_NO_PDL
  bool debug_sync = false;      // TMG_OPT_DEBUG_SYNC
  bool no_graph = false;        // TMG_OPT_NO_GRAPH
  bool z_natural = false;       // TMG_OPT_Z_NATURAL
  bool generic_small = false;   // TMG_OPT_GENERIC_SMALL
};

struct Context {
  int device = 0;
  int num_sms = 148;
  int escalations = 0;  // re-runs at b - 1 after a precision failure
  Options opt;
  Profiler prof;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  TwiddleCache tw;
  // keyed on every Params field, so a cache hit never skips validate_params
  std::map<std::tuple<int64_t, int32_t, int64_t, int64_t, int32_t, int32_t, int32_t, int32_t>,
           std::unique_ptr<Plan>>
      plans;
  DevBuf status, dop_u, dop_v, dop_out, pflags;
  Workspace ws0;                                  // single products (context stream)
  std::vector<std::unique_ptr<Workspace>> wsb;    // batch workspaces (own streams)
  DevStatus* h_status = nullptr;  // pinned
  // Multi-pass batches replayed as CUDA graphs: a batch shape seen once runs
  // eagerly (allocating every workspace buffer), the second time it is
  // captured, afterwards replayed.  Keyed on plan, count and pointers;
  // dropped when any device buffer reallocates.
  struct BatchKey {
    const void* plan;
    int64_t count;
    const void *u, *v, *out, *flags;
    bool operator<(const BatchKey& o) const {
      return std::tie(plan, count, u, v, out, flags) <
             std::tie(o.plan, o.count, o.u, o.v, o.out, o.flags);
    }
  };
  struct BatchGraph {
    cudaGraphExec_t exec = nullptr;
    int kernels = 0;
  };
  std::map<BatchKey, BatchGraph> graphs;
  std::map<BatchKey, int> graph_seen;
  uint64_t graph_gen = 0;
  bool graphs_off = false;
  cudaStream_t cap_stream = nullptr;  // batches are captured here (the context
                                      // stream may be the legacy default one)
  void clear_graphs() {
    for (auto& g : graphs)
      if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
    graphs.clear();
    graph_seen.clear();
  }
  ~Context() {
    clear_graphs();
    if (cap_stream) cudaStreamDestroy(cap_stream);
  }
  int32_t last_kernels = 0;
  int64_t last_L = 0;
  // k_zstat may read its operands before waiting for its predecessor
  // (programmatic launch) only when no kernel still in flight can be writing
  // them: on the host-buffer path, where the library's own H2D copies wrote
  // them after the context's previous work.  Device-pointer products never
  // read early -- another context sharing the stream, or any kernel that
  // triggers its dependents early, may still be producing the operands.
  bool zstat_early = false;
  void drained() {}
  int32_t last_passes = 0;

  // plans of the stand-alone convolution, by length (tmg_cyclic_convolve_f64)
  std::map<int64_t, std::unique_ptr<Plan>> conv_plans;

  Plan& plan_for(const Params& p) {
    auto key = std::make_tuple(p.n, p.b, p.N, p.lambda, int32_t(p.mode), p.p, int32_t(p.backend),
                               int32_t(p.signed_split));
    auto it = plans.find(key);
    if (it != plans.end()) return *it->second;
    validate_params(p);
    auto pl = build_plan(p, tw, opt.plan);
    Plan& ref = *pl;
    plans.emplace(key, std::move(pl));
    return ref;
  }
};

namespace {

// 1 / (4 L) as an unevaluated pair: L = 2^k m with m odd is rarely a power
// of two, and a single rounded constant would scale every coefficient by the
// same relative error.
void spectral_scale(int64_t L, double* hi, double* lo) {
  const long double v = 1.0L / (4.0L * (long double)L);
  *hi = double(v);
  *lo = double(v - (long double)(*hi));
}

// z layout shared by k_zgen (writer) and k_f1 (reader).
ZTile ztile(const Plan& pl, int64_t L, bool natural) {
  ZTile t;
  const uint32_t ncols = uint32_t(L / pl.A);
  t.fdcols = make_fastdiv(ncols);
  t.logc = pl.logc_f1;
  t.zrows = uint32_t((pl.params.N + ncols - 1) / ncols);
  t.natural = natural ? 1u : 0u;
  return t;
}



// Every kernel of a product goes out through launch(): with programmatic
// dependent launch (default; TMG_OPT_NO_PDL turns it off) the next kernel on
// the stream is scheduled while the current one drains and waits in
// pdl_wait() (common.cuh) for its data, which hides the launch gap between
// the pipeline's dependent kernels.
//
// The first column pass goes without PDL (site "f1"): its 150-190 KB CTAs
// scheduled early share SMs with the draining split kernel (measured +7 % on
// the 2^26 full product).  The fully serialized F1 launch also bounds how far
// a product's chain can run ahead: the next product's k_zstat, which writes
// the split aggregates before its grid-dependency wait, cannot start before
// this product's k_zgen (their reader) has completed.
//
// Kernels without griddepcontrol.wait (the fused small-product kernels) go
// out with pdl = false: launched programmatically they could start under a
// predecessor that triggered early and read its unfinished outputs.
template <class Arg>
void launch(const Context& cx, void (*kernel)(Arg), dim3 grid, dim3 block, size_t smem,
            cudaStream_t st, const Arg& arg, const char* site = nullptr, bool pdl = true) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  const bool skip = site && std::strcmp(site, "f1") == 0;
  attr[0].val.programmaticStreamSerializationAllowed = (pdl && !cx.opt.no_pdl && !skip) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TMG_CUDA(cudaLaunchKernelEx(&cfg, kernel, arg));
}

void check_launch(const Context& cx, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    throw Error(TMG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  if (cx.opt.debug_sync) {
    e = cudaDeviceSynchronize();
    fprintf(stderr, "[tmg] %s done: %s\n", what, cudaGetErrorString(e));
    if (e != cudaSuccess)
      throw Error(TMG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

// Opt in to the dynamic shared memory a launch needs.  The 48 KB default
// covers static + dynamic together, so any sizeable request is opted in
// (a kernel with a few KB of static arrays fails at dynamic sizes just
// under 48 KB otherwise).
// The attribute is per function: remember what each kernel has been granted
// (a driver call per launch costs more than the small products' kernels).
template <class K>
void set_smem(K kernel, size_t bytes) {
  if (bytes <= 16 * 1024) return;
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> granted;
  std::lock_guard<std::mutex> lock(mu);
  size_t& g = granted[reinterpret_cast<const void*>(kernel)];
  if (bytes <= g) return;
  TMG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(bytes)));
  g = bytes;
}

struct KTimer {
  Context& cx;
  Profiler::Rec rec;
  bool on;
  KTimer(Context& c, const char* name, double bytes, int mode = -1,
         cudaStream_t st = nullptr)
      : cx(c), on(c.prof.on && (st == nullptr || st == c.stream)) {
    if (on) {
      static const char* kPrefix[] = {"full:", "low:", "high:"};
      rec.name = std::string(mode >= 0 && mode < 3 ? kPrefix[mode] : "") + name;
      rec.bytes = bytes;
      rec.a = cx.prof.get();
      rec.b = cx.prof.get();
      cudaEventRecord(rec.a, st ? st : cx.stream);
    }
  }
  ~KTimer() {
    if (on) {
      cudaEventRecord(rec.b, cx.stream);  // only context-stream launches are timed
      cx.prof.recs.push_back(rec);
    }
  }
};

// Workspace buffers sized for one product of plan pl.
size_t workspace_bytes(const Plan& pl) {
  const int64_t L = pl.L;
  return size_t(L) * 24 + (size_t(pl.params.N) + size_t(L / std::max<uint32_t>(pl.A, 1))) * 16 +
         size_t(pl.ML) * 8;
}

void ensure_workspace(Workspace& w, const Plan& pl) {
  const Params& p = pl.params;
  const int64_t L = pl.L;
  w.work_t.ensure(size_t(L) * 16);
  w.work_c.ensure(size_t(L) * 8 + 64);
  // z: N entries, plus up to one row of F1's tiling slack (ZTile)
  w.work_z.ensure((size_t(p.N) + (pl.kind >= 2 ? size_t(L / pl.A) : 0)) * 16 + 64);
  const int64_t cwords = (pl.count + 31) / 32 + 1;
  w.cbu.ensure(size_t(cwords) * 4);
  w.cbv.ensure(size_t(cwords) * 4);
  w.aux.ensure(64);
}

// The transform passes of one product or convolution: first column pass
// (reading z), the middle column passes of three-pass plans, the row pass
// with the spectral product, and the inverse column passes, which leave the
// convolution coefficients in w.work_c.  Returns the kernels launched.
// out_scale (a power of two) multiplies the coefficients on their way out.
int enqueue_fft_passes(Context& cx, Workspace& w, cudaStream_t st, Plan& pl, const uint64_t* u,
                       const uint64_t* v, bool z_natural, double out_scale = 1.0) {
  const Params& p = pl.params;
  const int64_t L = pl.L;
  int kernels = 0;
  {
    double2* T = w.work_t.as<double2>();
    {
      F1Args a;
      a.z = w.work_z.as<double2>();
      a.zt = ztile(pl, L, z_natural);
      a.out = T;
      a.ncols = uint32_t(L / pl.A);
      a.logc = pl.logc_f1;
      a.stw = pl.f1_stw ? 1u : 0u;
      a.fft = pl.fA;
      a.tw = pl.twL;
      a.mc = pl.mc;
      a.u = u;
      a.v = v;
      a.nlimbs = pl.nlimbs;
      a.b = p.b;
      a.count = pl.count;
      a.lead = pl.lead;
      a.cbits_u = w.cbu.as<uint32_t>();
      a.cbits_v = w.cbv.as<uint32_t>();
      a.aux = w.aux.as<double>();
      a.dig = w.work_z.p;
      auto f1k = pl.f1d ? pl.f1d : pl.colct ? pl.colct->f1 : pl.colpp ? k_f1_pp : k_f1;
      set_smem(f1k, pl.smem_f1);
      {
        // k_f1d_ct reads the digit rows (the pre-map's halo row again, from L2)
        const double zin = pl.f1d ? (pl.zdig == 1 ? 4.0 : 8.0) : 16.0;
        KTimer kt(cx, "k_f1", double(p.N) * zin + double(L) * 16.0, int(p.mode), st);
        // the compile-time pass is persistent (one wave of CTAs)
        const unsigned tiles = a.ncols >> a.logc;
        const unsigned grid =
            pl.colct ? std::min<unsigned>(tiles, unsigned(cx.num_sms * (pl.thr_f1 <= 288 ? 2 : 1)))
                     : tiles;
        launch(cx, f1k, dim3(grid), dim3(pl.thr_f1), pl.smem_f1, st, a, "f1");
      }
      check_launch(cx, "k_f1");
      ++kernels;
    }
    if (pl.kind == 3) {
      ColArgs a;
      a.data = T;
      a.g.os = int64_t(pl.B) * pl.C;
      a.g.rs = pl.C;
      a.g.cs = pl.C;
      a.g.cw = pl.C;
      a.g.ncols = pl.C;
      a.logc = pl.logc_f2;
      a.fft = pl.fB;
      a.tw = pl.twL;
      a.inv = 0;
      a.to = 0;
      a.tc = 1;
      a.tmul = pl.A;
      auto colk = pl.colct_b ? pl.colct_b->col : pl.colpp ? col_pp_kernel(false) : k_col;
      set_smem(colk, pl.smem_f2);
      {
        KTimer kt(cx, "k_col_f2", double(L) * 32.0, int(p.mode), st);
        launch(cx, colk, dim3(dim3(pl.C >> a.logc, pl.A)), dim3(pl.thr_f2), pl.smem_f2, st, a, "col");
      }
      check_launch(cx, "k_col(f2)");
      ++kernels;
    }
    {
      MidArgs a;
      a.data = T;
      a.A = pl.A;
      a.B = pl.B;
      a.C = pl.C;
      a.fwd = pl.fC;
      a.inv = pl.iC;
      a.tw = pl.twL;
      a.L = uint32_t(L);
      a.gen = w.gen.as<uint32_t>();
      const unsigned npairs = (pl.A * pl.B) / 2 + 1;
      if (pl.mid_ct) {
        // compiled shorter rows, persistent over the row pairs
        auto mk = pl.C == 2048 ? k_mid_2048 : k_mid_1024;
        set_smem(mk, pl.smem_mid);
        const unsigned grid = std::min<unsigned>(npairs, unsigned(cx.num_sms));
        KTimer kt(cx, "k_mid", double(L) * 16.0 + double(L) * 8.0, int(p.mode), st);
        launch(cx, mk, dim3(grid), dim3(kMidCtThreads), pl.smem_mid, st, a, "mid");
      } else if (pl.C == 4096 && pl.mid_shared_table && !cx.opt.generic_row) {
        // compile-time schedule, persistent over row pairs
        set_smem(k_mid_4096, pl.smem_mid);
        const unsigned grid = std::min<unsigned>(npairs, unsigned(cx.num_sms));
        KTimer kt(cx, "k_mid", double(L) * 16.0 + double(L) * 8.0, int(p.mode), st);
        launch(cx, k_mid_4096, dim3(grid), dim3(kMidCtThreads), pl.smem_mid, st, a, "mid");
      } else {
        set_smem(k_mid, pl.smem_mid);
        KTimer kt(cx, "k_mid", double(L) * 16.0 + double(L) * 8.0, int(p.mode), st);
        launch(cx, k_mid, dim3(npairs), dim3(pl.thr_mid), pl.smem_mid, st, a, "mid");
      }
      check_launch(cx, "k_mid");
      ++kernels;
    }
    if (pl.kind == 3) {
      ColArgs a;
      a.data = T;
      a.g.os = int64_t(pl.B) * pl.C;
      a.g.rs = pl.C;
      a.g.cs = pl.C;
      a.g.cw = pl.C / 2;
      a.g.ncols = pl.C / 2;
      a.logc = pl.logc_i2;
      a.fft = pl.iB;
      a.tw = pl.twL;
      a.inv = 1;
      a.to = 1;
      a.tc = 0;
      a.tmul = pl.C;
      auto colk = pl.colct_b ? pl.colct_b->col : pl.colpp ? col_pp_kernel(true) : k_col;
      set_smem(colk, pl.smem_i2);
      {
        KTimer kt(cx, "k_col_i2", double(L) * 16.0, int(p.mode), st);
        launch(cx, colk, dim3(dim3((pl.C / 2) >> a.logc, pl.A)), dim3(pl.thr_i2), pl.smem_i2, st, a, "col");
      }
      check_launch(cx, "k_col(i2)");
      ++kernels;
    }
    double2* coef = w.work_c.as<double2>();
    {
      ILastArgs a;
      a.data = T;
      a.coef = coef;
      a.g.os = 0;
      a.g.rs = int64_t(pl.B) * pl.C;
      a.g.cs = pl.C;
      a.g.cw = pl.C / 2;
      a.g.ncols = pl.B * (pl.C / 2);
      a.logc = pl.logc_il;
      a.fft = pl.iA;
      spectral_scale(L, &a.scale, &a.scale_lo);
      a.scale *= out_scale;
      a.scale_lo *= out_scale;
      auto ilk = pl.colct_il ? pl.colct_il->ilast : pl.colpp ? k_ilast_pp : k_ilast;
      set_smem(ilk, pl.smem_il);
      {
        KTimer kt(cx, "k_ilast", double(L) * 16.0, int(p.mode), st);
        // the compiled pass is persistent (it stages its next tile in shared
        // memory behind its last stage); the others take one CTA per tile
        const unsigned tiles = a.g.ncols >> a.logc;
        const unsigned grid = pl.colct_il ? std::min<unsigned>(tiles, unsigned(cx.num_sms * (pl.thr_il <= 288 ? 2 : 1)))
                                          : tiles;
        launch(cx, ilk, dim3(grid), dim3(pl.thr_il), pl.smem_il, st, a, "ilast");
      }
      check_launch(cx, "k_ilast");
      ++kernels;
    }
  }
  return kernels;
}

// One multi-pass product on stream st with workspace w; device flags,
// residuals and the high product's range words go to status.  Returns the
// number of kernels launched.
int enqueue_product(Context& cx, Workspace& w, cudaStream_t st, DevStatus* status, Plan& pl,
                    const uint64_t* u, const uint64_t* v, uint64_t* out) {
  const Params& p = pl.params;
  const int64_t L = pl.L;
  int kernels = 0;
  {
    // balanced split + pre-map (both operands)
    {
      ZgenArgs a;
      a.u = u;
      a.v = v;
      a.nlimbs = pl.nlimbs;
      a.n = p.n;
      a.b = p.b;
      a.count = pl.count;
      a.N = p.N;
      a.lead = pl.lead;
      a.cbits_u = w.cbu.as<uint32_t>();
      a.cbits_v = w.cbv.as<uint32_t>();
      a.z = w.work_z.as<double2>();
      a.mc = pl.mc;
      a.zt = ztile(pl, L, cx.opt.z_natural);
      a.status = status;
      if (!w.gen.p) {
        w.gen.ensure(64);
        TMG_CUDA(cudaMemsetAsync(w.gen.p, 0, 64, st));
      }
      a.gen = w.gen.as<uint32_t>();
      a.lbstate = nullptr;
      a.aggs = nullptr;
      a.early = 0;
      // Split by runs (k_zsplit): every thread finds its carry-in from the
      // window below its run, so there are no aggregates and no look-back.
      // Digit form, balanced split, compiled chunk widths, runs inside one
      // row of z's tiles; TMG_OPT_SPLIT_KERNEL 1 keeps k_zgen.
      ZgenFn zs = nullptr;
      {
        const uint32_t ncols = a.zt.fdcols.d;
        const int minlog = pl.zdig == 1 ? 2 : 1;
        if (pl.f1d && pl.mc.balanced && !cx.opt.zstat_split && !cx.opt.old_split && pl.count < (int64_t(1) << 31) &&
            (a.zt.natural || (ncols % 32 == 0 && int(a.zt.logc) >= minlog)) &&
            pl.count >= int64_t(zsplit_chunks()) * cx.num_sms / 2)
          zs = zsplit_kernel(int(p.b), pl.zdig);
      }
      if (zs) {
        // blocks of 8 rows by 1024 columns of z's tiles (a warp's 16-byte
        // digit pieces then fill whole lines), or of 8192 consecutive chunks
        const uint32_t ncols = a.zt.fdcols.d;
        const int64_t zch = zsplit_chunks();
        a.zs_rb = (!a.zt.natural && ncols % uint32_t(zch / 8) == 0) ? 8 : 1;
        unsigned blocks = unsigned((pl.count + zch - 1) / zch);
        if (a.zs_rb == 8) {
          const int64_t rows = (pl.count + ncols - 1) / ncols;
          blocks = unsigned(((rows + 7) / 8) * (ncols / uint32_t(zch / 8)));
        }
        const size_t zsm = zsplit_smem(int(p.b));
        set_smem(zs, zsm);
        {
          KTimer kt(cx, "k_zsplit", double(2 * pl.nlimbs) * 8.0 + double(p.N) * (pl.zdig == 1 ? 4.0 : 8.0), int(p.mode), st);
          launch(cx, zs, dim3(blocks), dim3(256), zsm, st, a, "zgen");
        }
        check_launch(cx, "k_zsplit");
        ++kernels;
      } else {
      // chunks per thread of the split: 16, or 4 / 1 when the blocks of 16
      // would not fill the GPU twice (mid-size products are latency-bound
      // per block)
      int per = 16;  // (the 64-bit window path, b > 32, has only this one)
      if (p.b <= 32 && (pl.count + 16 * kZgenThreads - 1) / (16 * kZgenThreads) < 2 * cx.num_sms) per = 4;
      if (per == 4 && (pl.count + 4 * kZgenThreads - 1) / (4 * kZgenThreads) < 2 * cx.num_sms) per = 1;
      a.bchunks = per * kZgenThreads;
      const unsigned blocks = unsigned((pl.count + a.bchunks - 1) / a.bchunks);
      w.zaggs.ensure(size_t(blocks) * 4 + 16);
      a.aggs = w.zaggs.as<uint32_t>();
      a.early = cx.zstat_early ? 1 : 0;
      // the split blocks take their carry-ins by a look-back inside k_zgen
      // (no k_zstat launch): a block's aggregate is published early (after
      // its windows), and its predecessor was dispatched before it, so the
      // waits are short (2^26 low 271.4 -> 267.2 us, 2^24 high 104.2 -> 101.1);
      // TMG_OPT_SPLIT_AGGREGATES composes k_zstat's aggregates instead
      const bool zlb = !cx.opt.zstat_split;
      if (zlb) {
        if (w.zlb.bytes < size_t(blocks) * 8) {
          w.zlb.ensure(size_t(blocks) * 8);
          TMG_CUDA(cudaMemsetAsync(w.zlb.p, 0, w.zlb.bytes, st));
        }
        a.lbstate = w.zlb.as<unsigned long long>();
      } else {
        {
          KTimer kt(cx, "k_zstat", double(2 * pl.nlimbs) * 8.0, int(p.mode), st);
          launch(cx, k_zstat, dim3((blocks + 255) / 256), dim3(256), 0, st, a, "zstat");
        }
        check_launch(cx, "k_zstat");
        ++kernels;
      }
      // with k_f1d_ct the split stores digits and the first column pass pre-maps
      ZgenFn zg = pl.f1d ? zgen_digits_kernel(int(p.b), pl.zdig, per)
                         : zgen_kernel(int(p.b), p.mode == PMode::kFull ? 0 : int(pl.mc.lambda), per);
      const double zbytes = pl.f1d ? (pl.zdig == 1 ? 4.0 : 8.0) : 16.0;
      const size_t zsm = zgen_smem(int(p.b), per);
      set_smem(zg, zsm);
      {
        KTimer kt(cx, "k_zgen", double(2 * pl.nlimbs) * 8.0 + double(p.N) * zbytes, int(p.mode), st);
        launch(cx, zg, dim3(blocks), dim3(kZgenThreads), zsm, st, a, "zgen");
      }
      check_launch(cx, "k_zgen");
      ++kernels;
      }
    }
    kernels += enqueue_fft_passes(cx, w, st, pl, u, v, cx.opt.z_natural);
    double2* coef = w.work_c.as<double2>();
    // high: k_carry_lanes and k_carry_patch nominate the limb that stops the
    // rounding increment (else k_high_agg does, after the single-pass k_carry)
    bool high_stop_fused = false;
    if (p.mode == PMode::kHigh && !w.hticket.p) {
      w.hticket.ensure(64);
      TMG_CUDA(cudaMemsetAsync(w.hticket.p, 0, 4, st));
      TMG_CUDA(cudaMemsetAsync(w.hticket.as<uint32_t>() + 1, 0xff, 4, st));
    }
    {
      CarryArgs a;
      a.hstop = (p.mode == PMode::kHigh) ? w.hticket.as<uint32_t>() + 1 : nullptr;
      a.w = reinterpret_cast<const double*>(coef);
      a.out = out;
      a.n = p.n;
      a.out_limbs = pl.out_limbs;
      a.K = pl.K;
      a.ML = pl.ML;
      a.shift_s = pl.shift_s;
      a.mc = pl.mc;
      a.aux = w.aux.as<double>();
      a.wlen = pl.L;
      a.blk_limbs = 0;
      a.runs_lb = 0;
      const int64_t LB = kCarryThreads * kCarryPerThread;
      const unsigned blocks = unsigned((pl.ML + LB - 1) / LB);
      a.scan = w.scan_c.next(blocks);
      a.status = status;
      if (p.mode == PMode::kHigh) {
        w.tbuf.ensure(size_t(pl.ML) * 8 + 64);
        a.tbuf = w.tbuf.as<uint64_t>();
      } else {
        a.tbuf = nullptr;
      }
      const bool old_carry = cx.opt.lookback_carry;
      const int lam = (p.mode == PMode::kFull) ? 0 : int(pl.mc.lambda);
      // limbs per thread: 4 when the block's coefficient window stays small
      // (wide chunks), else 2 (more CTAs per SM for narrow chunks)
      const bool hb = p.mode == PMode::kHigh;
      int pt = carry2_smem(int(p.b), lam, 4, hb) <= size_t(64) * 1024 ? 4 : 2;
      // products whose carry blocks cannot fill the GPU twice over take one
      // limb per thread: twice the blocks, each with half the latency
      // (single-pass kernel, mid-size products)
      // (the single-pass kernel only: its one-wave rule must still hold)
      if (cx.opt.carry_kernels < 2 && carry_lb_kernel(lam, 1) &&
          (pl.ML + int64_t(kC2Threads) * pt - 1) / (int64_t(kC2Threads) * pt) < int64_t(2 * cx.num_sms) &&
          (pl.ML + kC2Threads - 1) / kC2Threads <= int64_t(4 * cx.num_sms))
        pt = 1;
      const size_t smem2 = carry2_smem(int(p.b), lam, pt, hb);
      if (!old_carry && smem2 <= kMaxDynSmem && 64 * pl.ML + 64 < (int64_t(1) << 32)) {
        high_stop_fused = p.mode == PMode::kHigh;
        a.fb = make_fastdiv(uint32_t(p.b));
        const int64_t limbs = int64_t(kC2Threads) * pt;
        const unsigned blocks2 = unsigned((pl.ML + limbs - 1) / limbs);
        w.aggs.ensure(size_t(blocks2) * 8 + 16);
        a.aggs = w.aggs.as<uint32_t>();
        a.cins = reinterpret_cast<int*>(a.aggs + blocks2);
        if (!w.ticket.p) {
          w.ticket.ensure(64);
          TMG_CUDA(cudaMemsetAsync(w.ticket.p, 0, 64, st));
        }
        a.ticket = w.ticket.as<uint32_t>();
        a.sbuf = w.work_t.p;  // the transform buffer is free after k_ilast
        // k_carry_patch composes the block functions itself while that stays
        // cheap (each patch CTA reads the aggregates before it); above, the
        // last lanes block scans them into cins
        // (TMG_OPT_PATCH_SCAN_MAX lowers the limit for testing)
        a.lanes_cins = long(blocks2) > cx.opt.patch_scan_max ? 1 : 0;
        // one kernel while the blocks fit one wave (4 per SM): their look-back
        // waits stay short, and a launch is saved (2^20 low 57.9 -> 55.3 us);
        // beyond, blocks that wait for a predecessor hold their slots, and the
        // second kernel costs less (2^26 low 271.6 against 278.0 us)
        // (the full product, whose runs have no post-map, takes the runs kernel
        // from 1.5 M coefficients: 2^24 full 18.8 -> 14.8 us; the truncated
        // products' runs are too long a chain below a full wave of them)
        const bool full_runs = p.mode == PMode::kFull && pl.K >= 1500000;
        const bool one = pt == 1 || cx.opt.carry_kernels == 1 ||
                         (cx.opt.carry_kernels == 0 && blocks2 <= unsigned(4 * cx.num_sms) && !full_runs);
        CarryLanesFn lbk = one ? carry_lb_kernel(lam, pt) : nullptr;
        if (lbk) {
          // one kernel: the carry-in by decoupled look-back, every limb written once
          a.scan = w.scan_c.next(blocks2);
          a.gen = w.gen.as<uint32_t>();
          set_smem(lbk, smem2);
          {
            KTimer kt(cx, "k_carry_lb", double(pl.K) * 8.0 + double(hb ? pl.ML : pl.out_limbs) * 8.0, int(p.mode),
                      st);
            launch(cx, lbk, dim3(blocks2), dim3(kC2Threads), smem2, st, a, "carry_lb");
          }
          check_launch(cx, "k_carry_lb");
          kernels += 1;
        } else {
        // runs kernel: one thread per run of 64 coefficients (b limbs); the
        // lanes kernel where it has no instantiation
        CarryLanesFn runs = (cx.opt.carry_kernels == 2 || p.b < 8 || pl.L >= (int64_t(1) << 31))
                                ? nullptr
                                : carry_runs_kernel(int(pl.mc.mode), lam, int(p.b), !cx.opt.generic_runs);
        unsigned blocksp = blocks2;
        bool runs_lb = false;
        if (runs) {
          const int runlen = carry_runs_len(int(pl.mc.mode), lam, int(p.b), !cx.opt.generic_runs);
          const int64_t rl = int64_t(kRunThreads) * p.b * runlen / 64;
          blocksp = unsigned((pl.ML + rl - 1) / rl);
          a.blk_limbs = rl;
          a.wlen = pl.L;
          a.lanes_cins = long(blocksp) > cx.opt.patch_scan_max ? 1 : 0;
          w.aggs.ensure(size_t(blocksp) * 8 + 16);
          a.aggs = w.aggs.as<uint32_t>();
          a.cins = reinterpret_cast<int*>(a.aggs + blocksp);
          const size_t smem3 = carry_runs_smem(int(pl.mc.mode), lam, runlen);
          set_smem(runs, smem3);
          // one kernel: the block carry-ins by a decoupled look-back over the
          // published aggregates (TMG_OPT_CARRY_KERNELS 3 keeps k_carry_patch)
          runs_lb = cx.opt.carry_kernels != 3;
          if (runs_lb) {
            a.runs_lb = 1;
            a.scan = w.scan_c.next(blocksp);
            a.gen = w.gen.as<uint32_t>();
          }
          {
            KTimer kt(cx, "k_carry_runs", double(pl.K) * 8.0 + double(hb ? pl.ML : pl.out_limbs) * 8.0, int(p.mode),
                      st);
            launch(cx, runs, dim3(blocksp), dim3(kRunThreads), smem3, st, a, "runs");
          }
          check_launch(cx, "k_carry_runs");
        } else {
          CarryLanesFn lanes = carry_lanes_kernel(lam, pt);
          if (!lanes) throw Error(TMG_ERR_UNSUPPORTED, "carry lanes kernel: no instantiation for this block shape");
          set_smem(lanes, smem2);
          {
            KTimer kt(cx, "k_carry_lanes", double(pl.K) * 8.0 + double(hb ? pl.ML : pl.out_limbs) * 8.0, int(p.mode),
                      st);
            launch(cx, lanes, dim3(blocks2), dim3(kC2Threads), smem2, st, a, "lanes");
          }
          check_launch(cx, "k_carry_lanes");
        }
        if (!runs_lb) {
          // the limbs are written for a zero carry into each block; one warp
          // per block adds its carry-in
          KTimer kt(cx, "k_carry_patch", 0.0, int(p.mode), st);
          launch(cx, carry_patch_kernel(pt), dim3((blocksp + kC2Threads / 32 - 1) / (kC2Threads / 32)), dim3(kC2Threads),
                 0, st, a, "patch");
          check_launch(cx, "k_carry_patch");
        }
        kernels += runs_lb ? 1 : 2;
        }
      } else {
        set_smem(k_carry, pl.smem_carry);
        {
          KTimer kt(cx, "k_carry", double(pl.K) * 8.0 + double(pl.mc.mode == 2 ? pl.ML : pl.out_limbs) * 8.0, int(p.mode), st);
          launch(cx, k_carry, dim3(blocks), dim3(kCarryThreads), pl.smem_carry, st, a, "carry");
        }
        check_launch(cx, "k_carry");
        ++kernels;
      }
    }
    if (p.mode == PMode::kHigh) {
      HighRoundArgs a;
      a.tbuf = w.tbuf.as<uint64_t>();
      a.out = out;
      a.n = p.n;
      a.out_limbs = pl.out_limbs;
      a.ML = pl.ML;
      a.shift_s = pl.shift_s;
      a.WL = pl.ML - (pl.shift_s >> 6);
      const int64_t LB = kCarryThreads * kHighPerThread;
      const unsigned blocks = unsigned((a.WL + LB - 1) / LB);
      a.status = status;
      if (!w.ticket.p) {
        w.ticket.ensure(64);
        TMG_CUDA(cudaMemsetAsync(w.ticket.p, 0, 64, st));
      }
      a.ticket = w.hticket.as<uint32_t>();
      if (!high_stop_fused) {
        KTimer kt(cx, "k_high_agg", double(pl.ML) * 8.0, int(p.mode), st);
        launch(cx, k_high_agg, dim3(blocks), dim3(kCarryThreads), 0, st, a, "hagg");
        check_launch(cx, "k_high_agg");
        ++kernels;
      }
      {
        KTimer kt(cx, "k_high_round", double(pl.ML) * 8.0 + double(pl.out_limbs) * 8.0, int(p.mode), st);
        launch(cx, k_high_round, dim3(blocks), dim3(kCarryThreads), 0, st, a, "hround");
      }
      check_launch(cx, "k_high_round");
      ++kernels;
    }
  }
  return kernels;
}

// Enqueue one batch of products (device pointers) on the context stream.
// own_operands: the library's own H2D copies wrote du and dv (host-buffer
// path), so k_zstat may read them before its grid-dependency wait.
void enqueue(Context& cx, Plan& pl, const uint64_t* du, const uint64_t* dv,
             uint64_t* dout, int64_t count, uint32_t* pflags, bool own_operands) {
  const Params& p = pl.params;
  cudaStream_t st = cx.stream;
  DevStatus* status = cx.status.as<DevStatus>();
  cx.zstat_early = own_operands;
  cx.last_L = pl.L;
  cx.last_passes = pl.kind;
  if (pl.kind == 0)
    throw Error(TMG_ERR_UNSUPPORTED, "fallback products run through the host entry points");
  if (pl.kind == 1 || (pl.small_batch && count >= kSmallBatchMinCount)) {
    SmallArgs a;
    a.u = du;
    a.v = dv;
    a.out = dout;
    a.pflags = pflags;
    a.nlimbs = pl.nlimbs;
    a.n = p.n;
    a.out_limbs = pl.out_limbs;
    a.L = pl.L;
    a.count = pl.count;
    a.lead = pl.lead;
    a.K = pl.K;
    a.ML = pl.ML;
    a.shift_s = pl.shift_s;
    spectral_scale(pl.L, &a.scale, &a.scale_lo);
    a.fwd = pl.fwd;
    a.inv = pl.inv;
    a.mc = pl.mc;
    a.status = status;
    // the 2-CTA variant only pays when two CTAs' shared memory fits an SM
    // (228 KB, 1 KB reserved per CTA); otherwise its spills cost for nothing
    const bool two = pl.small_threads <= 384 && 2 * (pl.small_smem + 1024) <= size_t(228) * 1024;
    auto sk = pl.small_threads > 512 ? k_small_product_big
                                     : two ? k_small_product_2 : k_small_product;
    unsigned threads = unsigned(pl.small_threads);
    // TMG_OPT_GENERIC_SMALL (testing): the runtime-dispatched stages at every length
    const bool small_generic = cx.opt.generic_small;
    // (a 640-thread 8 x 8 x 8 x 10 variant for the low/high L = 5120 was
    // slower than the 2-CTA generic kernel: 1.57 / 2.12 ms against 1.40 /
    // 1.68 ms for 4096 products; the maps prefer two smaller CTAs per SM)
    if (!small_generic && pl.L == 6144 && p.mode == PMode::kFull) {
      sk = k_small_6144;
      threads = 768;
    } else if (!small_generic && pl.L == 5120 && p.mode != PMode::kFull && two) {
      sk = k_small_5120;
      threads = 384;
    }
    set_smem(sk, pl.small_smem);
    {
      KTimer kt(cx, "k_small_product", double(count) * double(2 * pl.nlimbs + pl.out_limbs) * 8.0, int(p.mode));
      launch(cx, sk, dim3(unsigned(count)), dim3(threads), pl.small_smem, st, a, "small", false);
    }
    check_launch(cx, "k_small_product");
    cx.last_kernels = 1;
    return;
  }
  // multi-pass
  if (count == 1) {
    ensure_workspace(cx.ws0, pl);
    cx.last_kernels = enqueue_product(cx, cx.ws0, st, status, pl, du, dv, dout);
    if (pflags) {
      k_status_publish<<<1, 1, 0, st>>>(status, pflags, nullptr);
      check_launch(cx, "k_status_publish");
    }
    return;
  }
  // a batch: products round-robin over up to kMaxBatchStreams workspaces,
  // each on its own stream with its own status word, published per product
  // into pflags and merged into the context status.  Repeated batch shapes
  // replay a captured graph (the launches of a batch of small multi-pass
  // products cost more host time than their kernels run).
  const bool graphable = !cx.opt.no_graph && !cx.graphs_off && !cx.prof.on && !cx.opt.debug_sync &&
                         count >= kGraphMinBatch;
  Context::BatchKey key{&pl, count, du, dv, dout, pflags};
  bool capture = false;
  if (graphable) {
    const uint64_t gen = g_devbuf_generation.load();
    if (gen != cx.graph_gen) {
      cx.clear_graphs();
      cx.graph_gen = gen;
    }
    auto it = cx.graphs.find(key);
    if (it != cx.graphs.end()) {
      TMG_CUDA(cudaGraphLaunch(it->second.exec, st));
      cx.last_kernels = it->second.kernels;
      return;
    }
    capture = cx.graph_seen[key]++ > 0;
  }
  const cudaStream_t user_st = st;
  if (capture) {
    if (!cx.cap_stream) TMG_CUDA(cudaStreamCreateWithFlags(&cx.cap_stream, cudaStreamNonBlocking));
    st = cx.cap_stream;
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      (void)cudaGetLastError();
      cx.graphs_off = true;
      capture = false;
      st = user_st;
    }
  }
  // an error thrown while capturing must not leave the stream in capture mode
  struct CaptureGuard {
    cudaStream_t st;
    bool* active;
    Context* cx;
    ~CaptureGuard() {
      if (*active) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        (void)cudaGetLastError();
        cx->graphs_off = true;
      }
    }
  } guard{st, &capture, &cx};
  const size_t budget = size_t(4) << 30;
  const int64_t by_mem = int64_t(budget / std::max<size_t>(workspace_bytes(pl), 1));
  const int S = int(std::max<int64_t>(
      1, std::min<int64_t>(std::min<int64_t>(count, kMaxBatchStreams), by_mem)));
  while (int(cx.wsb.size()) < S) {
    auto w = std::make_unique<Workspace>();
    TMG_CUDA(cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking));
    TMG_CUDA(cudaEventCreateWithFlags(&w->done, cudaEventDisableTiming));
    w->status.ensure(sizeof(DevStatus));
    cx.wsb.push_back(std::move(w));
  }
  cudaEvent_t start = cx.wsb[0]->done;
  TMG_CUDA(cudaEventRecord(start, st));
  for (int s2 = 0; s2 < S; ++s2) {
    Workspace& w = *cx.wsb[s2];
    ensure_workspace(w, pl);
    TMG_CUDA(cudaStreamWaitEvent(w.stream, start, 0));
  }
  int kernels = 0;
  for (int64_t i = 0; i < count; ++i) {
    Workspace& w = *cx.wsb[i % S];
    DevStatus* ws = w.status.as<DevStatus>();
    TMG_CUDA(cudaMemsetAsync(ws, 0, sizeof(DevStatus), w.stream));
    kernels += enqueue_product(cx, w, w.stream, ws, pl, du + i * pl.nlimbs, dv + i * pl.nlimbs,
                               dout + i * pl.out_limbs);
    k_status_publish<<<1, 1, 0, w.stream>>>(ws, pflags ? pflags + i : nullptr, status);
    check_launch(cx, "k_status_publish");
  }
  for (int s2 = 0; s2 < S; ++s2) {
    Workspace& w = *cx.wsb[s2];
    TMG_CUDA(cudaEventRecord(w.done, w.stream));
    TMG_CUDA(cudaStreamWaitEvent(st, w.done, 0));
  }
  cx.last_kernels = kernels;
  if (capture) {
    capture = false;  // the guard has nothing left to close
    cudaGraph_t g = nullptr;
    cudaGraphExec_t exec = nullptr;
    const cudaError_t e1 = cudaStreamEndCapture(st, &g);
    const cudaError_t e2 = (e1 == cudaSuccess) ? cudaGraphInstantiate(&exec, g, 0) : e1;
    if (g) cudaGraphDestroy(g);
    if (e2 != cudaSuccess) {
      // capture unsupported here: run this batch eagerly, stop capturing
      (void)cudaGetLastError();
      cx.graphs_off = true;
      enqueue(cx, pl, du, dv, dout, count, pflags, own_operands);
      return;
    }
    cx.graphs[key] = Context::BatchGraph{exec, kernels};
    TMG_CUDA(cudaGraphLaunch(exec, user_st));
  }
}

void reset_status(Context& cx) {
  TMG_CUDA(cudaMemsetAsync(cx.status.p, 0, sizeof(DevStatus), cx.stream));
}

// Reads the status word, clears it for the next products on the stream, and
// maps device flags onto the reference's errors.  The clear comes before any
// throw: a refused product must not leave its flags behind for the next
// tmg_check of good products.
int finish(Context& cx, const Plan* pl, tmg_stats* stats) {
  TMG_CUDA(cudaMemcpyAsync(cx.h_status, cx.status.p, sizeof(DevStatus),
                           cudaMemcpyDeviceToHost, cx.stream));
  TMG_CUDA(cudaStreamSynchronize(cx.stream));
  DevStatus s = *cx.h_status;
  reset_status(cx);
  double e, m;
  std::memcpy(&e, &s.max_err_bits, 8);
  std::memcpy(&m, &s.max_abs_bits, 8);
  if (stats) {
    stats->max_round_err = e;
    stats->max_abs = m;
    stats->flags = s.flags;
    stats->transform_length = cx.last_L;
    stats->passes = cx.last_passes;
    stats->kernels = cx.last_kernels;
  }
  uint32_t f = s.flags;
  if (s.high_topbit && s.high_lownz) f |= kFlagHighRange;
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) throw Error(TMG_ERR_CUDA, cudaGetErrorString(ce));
  if (f & kFlagInputRange)
    throw Error(TMG_ERR_INPUT_OUT_OF_RANGE, "split: operand outside [0, 2^n)");
  if (f & kFlagOverflow)
    throw Error(TMG_ERR_PRECISION_FAILURE,
                "float pipeline coefficient overflowed the exact-integer range");
  if (f & kFlagTripwire)
    throw Error(TMG_ERR_PRECISION_FAILURE,
                "float pipeline rounding tripwire: residual above a quarter");
  if (f & kFlagLowNotDivisible)
    throw Error(TMG_ERR_PRECISION_FAILURE,
                "low product recombination is not divisible by the chunk base");
  if (f & kFlagHighRange)
    throw Error(TMG_ERR_PRECISION_FAILURE, "high product left its admissible range");
  if (f & kFlagNegative)
    throw Error(TMG_ERR_PRECISION_FAILURE, "full product recombined negative");
  if (f & kFlagFullOverflow)
    throw Error(TMG_ERR_PRECISION_FAILURE, "full product exceeded 2n bits");
  if (f & kFlagCarryRange)
    throw Error(TMG_ERR_INTERNAL, "carry propagation left its range");
  (void)pl;
  return TMG_OK;
}

Params from_c(const tmg_params* p) {
  Params q;
  q.n = p->n;
  q.b = p->b;
  q.N = p->N;
  q.lambda = p->lambda;
  q.p = p->p;
  q.mode = PMode(p->mode);
  q.backend = Backend(p->backend);
  q.signed_split = p->signed_split != 0;
  return q;
}

void to_c(const Params& q, tmg_params* p) {
  p->n = q.n;
  p->b = q.b;
  p->N = q.N;
  p->lambda = q.lambda;
  p->p = q.p;
  p->mode = int32_t(q.mode);
  p->backend = int32_t(q.backend);
  p->signed_split = q.signed_split ? 1 : 0;
}

void init_context(Context& cx, int device) {
  cx.device = device;
  TMG_CUDA(cudaSetDevice(device));
  TMG_CUDA(cudaDeviceGetAttribute(&cx.num_sms, cudaDevAttrMultiProcessorCount, device));
  TMG_CUDA(cudaStreamCreateWithFlags(&cx.stream, cudaStreamNonBlocking));
  cx.own_stream = true;
  cx.status.ensure(sizeof(DevStatus));
  TMG_CUDA(cudaMemset(cx.status.p, 0, sizeof(DevStatus)));
  TMG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&cx.h_status), sizeof(DevStatus),
                         cudaHostAllocDefault));
}

// One product (or batch) from host limb arrays.
int host_product_once(Context& cx, const Params& p, int32_t want_mode,
                      const uint64_t* u, const uint64_t* v, int64_t count,
                      uint64_t* out, uint32_t* flags_out, tmg_stats* stats) {
  if (int32_t(p.mode) != want_mode && p.mode != PMode::kOracleFallback)
    throw Error(TMG_ERR_INPUT_OUT_OF_RANGE,
                "product: params were built for a different mode");
  PMode eff = p.mode;
  Params q = p;
  if (eff == PMode::kOracleFallback) q.mode = PMode::kOracleFallback;
  Plan& pl = cx.plan_for(q);
  const int64_t nl = pl.nlimbs;
  const int64_t OLr = output_limbs(PMode(want_mode), p.n);
  TMG_CUDA(cudaSetDevice(cx.device));
  cx.dop_u.ensure(size_t(count * nl) * 8 + 8);
  cx.dop_v.ensure(size_t(count * nl) * 8 + 8);
  const int64_t OLk = (pl.kind == 0) ? pl.out_limbs : OLr;
  (void)OLk;
  // the fallback plan computes the full product; truncate afterwards
  const int64_t OLdev = (pl.kind == 0) ? 2 * nl : pl.out_limbs;
  cx.dop_out.ensure(size_t(count * OLdev) * 8 + 8);
  if (flags_out) cx.pflags.ensure(size_t(count) * 4 + 4);
  reset_status(cx);
  TMG_CUDA(cudaMemcpyAsync(cx.dop_u.p, u, size_t(count * nl) * 8, cudaMemcpyHostToDevice, cx.stream));
  TMG_CUDA(cudaMemcpyAsync(cx.dop_v.p, v, size_t(count * nl) * 8, cudaMemcpyHostToDevice, cx.stream));
  if (pl.kind == 0) {
    // exact product on the GPU, truncated on the host side of the copy
    DevBuf prod;
    prod.ensure(size_t(count * 2 * nl) * 8);
    for (int64_t i = 0; i < count; ++i) {
      BaseArgs a{cx.dop_u.as<uint64_t>() + i * nl, cx.dop_v.as<uint64_t>() + i * nl,
                 prod.as<uint64_t>() + i * 2 * nl, nl};
      k_basecase<<<1, 256, size_t(6 * nl) * 8 + 64, cx.stream>>>(a);
      check_launch(cx, "k_basecase");
    }
    std::vector<uint64_t> h(size_t(count * 2 * nl));
    TMG_CUDA(cudaMemcpyAsync(h.data(), prod.p, h.size() * 8, cudaMemcpyDeviceToHost, cx.stream));
    TMG_CUDA(cudaStreamSynchronize(cx.stream));
    cx.drained();
    cx.last_kernels = int32_t(count);
    cx.last_L = 0;
    cx.last_passes = 0;
    for (int64_t i = 0; i < count; ++i) {
      const uint64_t* P = h.data() + i * 2 * nl;
      uint64_t* o = out + i * OLr;
      // input range check (InputOutOfRange, split.cpp:13-20)
      const uint64_t* ui = u + i * nl;
      const uint64_t* vi = v + i * nl;
      if ((p.n & 63) && ((ui[nl - 1] | vi[nl - 1]) >> (p.n & 63)))
        throw Error(TMG_ERR_INPUT_OUT_OF_RANGE, "split: operand outside [0, 2^n)");
      if (want_mode == TMG_MODE_FULL) {
        for (int64_t k = 0; k < OLr; ++k) o[k] = k < 2 * nl ? P[k] : 0;
      } else if (want_mode == TMG_MODE_LOW) {
        for (int64_t k = 0; k < OLr; ++k) o[k] = P[k];
        if (p.n & 63) o[OLr - 1] &= (uint64_t(1) << (p.n & 63)) - 1;
      } else {
        // oracle_high_set(...).front() = floor(uv / 2^n)
        const int64_t q = p.n >> 6;
        const int r = int(p.n & 63);
        for (int64_t k = 0; k < OLr; ++k) {
          uint64_t lo = (q + k < 2 * nl) ? P[q + k] : 0;
          uint64_t hi = (q + k + 1 < 2 * nl) ? P[q + k + 1] : 0;
          o[k] = r ? ((lo >> r) | (hi << (64 - r))) : lo;
        }
        if ((p.n + 1) & 63) o[OLr - 1] &= (uint64_t(1) << ((p.n + 1) & 63)) - 1;
      }
      if (flags_out) flags_out[i] = 0;
    }
    if (stats) {
      std::memset(stats, 0, sizeof(*stats));
      stats->kernels = int32_t(count);
    }
    return TMG_OK;
  }
  enqueue(cx, pl, cx.dop_u.as<uint64_t>(), cx.dop_v.as<uint64_t>(), cx.dop_out.as<uint64_t>(),
          count, flags_out ? cx.pflags.as<uint32_t>() : nullptr, true);
  TMG_CUDA(cudaMemcpyAsync(out, cx.dop_out.p, size_t(count * pl.out_limbs) * 8,
                           cudaMemcpyDeviceToHost, cx.stream));
  if (flags_out)
    TMG_CUDA(cudaMemcpyAsync(flags_out, cx.pflags.p, size_t(count) * 4, cudaMemcpyDeviceToHost,
                             cx.stream));
  return finish(cx, &pl, stats);
}

// One product from host buffers.  With escalation enabled on the context, a
// single product whose float pipeline refused (tripwire / overflow /
// recombination check) -- or, stricter than the reference's "> 1/4" wire,
// whose residual reached a quarter -- is recomputed at chunk width b - 1, up
// to cx.escalations times; the stats then describe the attempt that
// produced the result, with TMG_STAT_ESCALATED set and the first attempt's
// residual kept.
int host_product(Context& cx, const Params& p, int32_t want_mode,
                 const uint64_t* u, const uint64_t* v, int64_t count,
                 uint64_t* out, uint32_t* flags_out, tmg_stats* stats) {
  Params q = p;
  double first_err = -1.0;
  for (int attempt = 0;; ++attempt) {
    tmg_stats st;
    std::memset(&st, 0, sizeof(st));
    const bool can = attempt < cx.escalations && count == 1 &&
                     q.mode != PMode::kOracleFallback && q.backend == Backend::kFft &&
                     q.b > (q.mode == PMode::kFull ? 1 : 4);
    bool refused = false;
    try {
      host_product_once(cx, q, want_mode, u, v, count, out, flags_out, &st);
      refused = can && !(st.max_round_err < 0.25);
    } catch (const Error& e) {
      if (stats) *stats = st;
      if (!(can && e.code() == TMG_ERR_PRECISION_FAILURE)) throw;
      refused = true;
    }
    if (first_err < 0) first_err = st.max_round_err;
    if (refused) {
      q = params_with_chunk(q.n, q.mode, q.b - 1);
      continue;
    }
    st.attempts = attempt + 1;
    st.first_round_err = first_err;
    st.b = q.b;
    st.N = q.N;
    if (attempt > 0) st.flags |= TMG_STAT_ESCALATED;
    if (stats) *stats = st;
    return TMG_OK;
  }
}

// cyclic_convolve_f64 (convolution.hpp:64-67): out = f (*) g, cyclic of length
// n, host arrays.  The length checks and messages follow make_plan
// (convolution.cpp:92-105).  Lengths above 4096 that are multiples of 4 run
// the products' transform passes on a plan of their own (a low-product shape
// with N = L whose z is read as is: no pre-map in the first column pass, and
// the passes end at the convolution coefficients); the others are summed
// directly.
constexpr int64_t kConvDirectMax = 4096;       // direct below the multi-pass plans
constexpr int64_t kConvDirectMaxOdd = 32768;   // direct for lengths the passes do not take
int conv_f64_host(Context& cx, int64_t n, const double* f, const double* g, double* out) {
  if (n < 1) throw Error(TMG_ERR_UNSUPPORTED_LENGTH, "make_plan: length must be positive");
  if (!is_2357_smooth(uint64_t(n)))
    throw Error(TMG_ERR_UNSUPPORTED_LENGTH,
                "make_plan: FFT backend needs a {2,3,5,7}-smooth length, got " + std::to_string(n));
  const bool direct = n <= kConvDirectMax || (n % 4 != 0 && n <= kConvDirectMaxOdd);
  if (!direct && n % 4 != 0)
    throw Error(TMG_ERR_UNSUPPORTED_LENGTH,
                "cyclic_convolve_f64: GPU transform lengths above " +
                    std::to_string(kConvDirectMaxOdd) + " must be multiples of 4, got " +
                    std::to_string(n));
  TMG_CUDA(cudaSetDevice(cx.device));
  cx.dop_u.ensure(size_t(n) * 8 + 16);
  cx.dop_v.ensure(size_t(n) * 8 + 16);
  TMG_CUDA(cudaMemcpyAsync(cx.dop_u.p, f, size_t(n) * 8, cudaMemcpyHostToDevice, cx.stream));
  TMG_CUDA(cudaMemcpyAsync(cx.dop_v.p, g, size_t(n) * 8, cudaMemcpyHostToDevice, cx.stream));
  const double* res = nullptr;
  if (direct) {
    cx.dop_out.ensure(size_t(n) * 8 + 16);
    {
      KTimer kt(cx, "k_conv_direct", double(n) * 24.0);
      launch_conv_direct(cx.dop_u.as<double>(), cx.dop_v.as<double>(), n, cx.dop_out.as<double>(),
                         cx.stream);
    }
    TMG_CUDA(cudaGetLastError());
    cx.last_kernels = 1;
    res = cx.dop_out.as<double>();
  } else {
    auto it = cx.conv_plans.find(n);
    if (it == cx.conv_plans.end()) {
      Params q;
      q.mode = PMode::kLow;
      q.backend = Backend::kFft;
      q.b = 8;
      q.N = n;
      q.n = n * 8;
      q.lambda = 1;  // one series row: the identity map
      q.p = required_precision(PMode::kLow, q.b, q.N);
      q.signed_split = true;
      PlanOptions po;
      po.premap_in_zgen = true;  // the first column pass reads 16-byte z entries as they are
      po.z_natural = true;
      std::unique_ptr<Plan> pl;
      try {
        pl = build_plan(q, cx.tw, po);
      } catch (const Error& e) {
        throw Error(TMG_ERR_UNSUPPORTED_LENGTH,
                    std::string("cyclic_convolve_f64: no GPU plan for length ") +
                        std::to_string(n) + " (" + e.what() + ")");
      }
      if (pl->kind < 2)
        throw Error(TMG_ERR_INTERNAL, "cyclic_convolve_f64: expected a multi-pass plan");
      it = cx.conv_plans.emplace(n, std::move(pl)).first;
    }
    Plan& pl = *it->second;
    Workspace& w = cx.ws0;
    ensure_workspace(w, pl);
    if (!w.gen.p) {
      w.gen.ensure(64);
      TMG_CUDA(cudaMemsetAsync(w.gen.p, 0, 64, cx.stream));
    }
    // g times the power of two that brings max |g| to max |f| (k_conv.cu)
    cx.pflags.ensure(16);
    TMG_CUDA(cudaMemsetAsync(cx.pflags.p, 0, 16, cx.stream));
    {
      KTimer kt(cx, "k_conv_absmax", double(n) * 16.0);
      launch_conv_absmax(cx.dop_u.as<double>(), cx.dop_v.as<double>(), n, cx.pflags.as<uint64_t>(),
                         cx.num_sms, cx.stream);
    }
    TMG_CUDA(cudaGetLastError());
    double mx[2] = {0.0, 0.0};
    TMG_CUDA(cudaMemcpyAsync(mx, cx.pflags.p, 16, cudaMemcpyDeviceToHost, cx.stream));
    TMG_CUDA(cudaStreamSynchronize(cx.stream));
    if (mx[0] == 0.0 || mx[1] == 0.0) {
      // a zero operand: the packed transform would return rounding noise of the other one
      std::memset(out, 0, size_t(n) * 8);
      cx.last_kernels = 1;
      return TMG_OK;
    }
    double gs = 1.0;
    if (std::isfinite(mx[0]) && std::isfinite(mx[1]) && mx[0] > 0.0 && mx[1] > 0.0) {
      int ef = 0, eg = 0;
      std::frexp(mx[0], &ef);
      std::frexp(mx[1], &eg);
      gs = std::ldexp(1.0, std::max(-500, std::min(500, ef - eg)));
    }
    {
      KTimer kt(cx, "k_conv_pack", double(n) * 32.0);
      launch_conv_pack(cx.dop_u.as<double>(), cx.dop_v.as<double>(), n, gs, w.work_z.as<double2>(),
                       cx.stream);
    }
    TMG_CUDA(cudaGetLastError());
    cx.last_kernels =
        2 + enqueue_fft_passes(cx, w, cx.stream, pl, nullptr, nullptr, true, 1.0 / gs);
    cx.last_L = pl.L;
    res = w.work_c.as<double>();
  }
  TMG_CUDA(cudaMemcpyAsync(out, res, size_t(n) * 8, cudaMemcpyDeviceToHost, cx.stream));
  TMG_CUDA(cudaStreamSynchronize(cx.stream));
  return TMG_OK;
}

// alpha* / beta* / gamma-dagger / delta-dagger on host sequences
// (maps_f64.hpp: alpha_star_f64, beta_star_f64, gamma_dagger_f64,
// delta_dagger_f64 on the tables of build_map_tables_f64(N, b, lambda, ..)).
// which: 0 alpha*, 1 beta*, 2 gamma-dagger, 3 delta-dagger.
//   alpha*:        in N         -> out N
//   beta*:         in N         -> out N
//   gamma-dagger:  in N + 1     -> out N, *aux = the root channel
//   delta-dagger:  in N, aux    -> out N + 1
int map_f64_host(Context& cx, int which, int64_t N, int32_t b, int64_t lambda, const double* in,
                 double aux_in, double* out, double* aux_out) {
  if (N < 1 || b < 1 || b > 62 || lambda < 1)
    throw Error(TMG_ERR_INPUT_OUT_OF_RANGE, "maps: N, b and lambda must be positive (b <= 62)");
  const bool high = which >= 2;
  if (N < 2 * lambda + 2)
    throw Error(TMG_ERR_UNSUPPORTED, "maps: N below 2 lambda + 2");
  if (high && N * int64_t(b) < 64)
    throw Error(TMG_ERR_UNSUPPORTED, "maps: the high-mode maps need N b >= 64 on the GPU");
  Params q;
  q.mode = high ? PMode::kHigh : PMode::kLow;
  q.backend = Backend::kFft;
  q.b = b;
  q.N = N;
  q.lambda = lambda;
  q.n = N * int64_t(b);
  q.signed_split = true;
  MapConsts mc = make_map_consts(q);  // lambda above the GPU limit throws here
  mc.scale_out = 1.0;                 // the products fold 2^b in; the maps do not
  const bool pre = (which == 0 || which == 2);
  const int64_t nin = N + (which == 2 ? 1 : 0), nout = N + (which == 3 ? 1 : 0);
  TMG_CUDA(cudaSetDevice(cx.device));
  cx.dop_u.ensure(size_t(nin) * 8 + 16);
  cx.dop_out.ensure(size_t(nout) * 8 + 16);
  cx.pflags.ensure(16);
  TMG_CUDA(cudaMemcpyAsync(cx.dop_u.p, in, size_t(nin) * 8, cudaMemcpyHostToDevice, cx.stream));
  {
    KTimer kt(cx, pre ? "k_map_pre" : "k_map_post", double(nin + nout) * 8.0);
    if (pre)
      launch_map_pre(mc, cx.dop_u.as<double>(), cx.dop_out.as<double>(), cx.pflags.as<double>(),
                     cx.stream);
    else
      launch_map_post(mc, cx.dop_u.as<double>(), aux_in, cx.dop_out.as<double>(), cx.stream);
  }
  TMG_CUDA(cudaGetLastError());
  TMG_CUDA(cudaMemcpyAsync(out, cx.dop_out.p, size_t(nout) * 8, cudaMemcpyDeviceToHost, cx.stream));
  double aux = 0.0;
  if (which == 2)
    TMG_CUDA(cudaMemcpyAsync(&aux, cx.pflags.p, 8, cudaMemcpyDeviceToHost, cx.stream));
  TMG_CUDA(cudaStreamSynchronize(cx.stream));
  if (which == 2 && aux_out) *aux_out = aux;
  cx.last_kernels = 1;
  return TMG_OK;
}

// split_low_i64 / split_high_i64 (products.hpp:68-79): the chunks of one host
// operand as int64 words.  The shape checks and their messages follow
// split.cpp:104-158 (check_low_shape / check_high_shape, check_operand,
// chunk_store's b <= 62).
int split_i64_host(Context& cx, const Params& p, bool high, const uint64_t* u, int64_t* out) {
  if (p.b < 1 || p.N < (high ? 2 : 1))
    throw Error(TMG_ERR_INPUT_OUT_OF_RANGE, "split: chunk width and count must be positive");
  if (!high && p.N * int64_t(p.b) < p.n)
    throw Error(TMG_ERR_INPUT_OUT_OF_RANGE, "split: N b >= n is required");
  if (high && (p.N + 1) * int64_t(p.b) < p.n + lg_ceil(uint64_t(p.N)) + 2)
    throw Error(TMG_ERR_INPUT_OUT_OF_RANGE, "split: (N+1) b >= n + lg N + 2 is required");
  if (p.n < 1) throw Error(TMG_ERR_INPUT_OUT_OF_RANGE, "split: bit length must be positive");
  if (p.b > 62)
    throw Error(TMG_ERR_INPUT_OUT_OF_RANGE, "split: chunk width too large for int64 chunks");
  const int64_t count = high ? p.N + 1 : p.N;
  const int64_t lead = high ? (p.N + 1) * int64_t(p.b) - p.n : 0;
  const int64_t nl = (p.n + 63) / 64;
  TMG_CUDA(cudaSetDevice(cx.device));
  cx.dop_u.ensure(size_t(nl) * 8 + 8);
  cx.dop_out.ensure(size_t(count) * 8 + 8);
  cx.pflags.ensure(8);
  TMG_CUDA(cudaMemsetAsync(cx.pflags.p, 0, 4, cx.stream));
  TMG_CUDA(cudaMemcpyAsync(cx.dop_u.p, u, size_t(nl) * 8, cudaMemcpyHostToDevice, cx.stream));
  {
    KTimer kt(cx, "k_split_i64", double(nl) * 8.0 + double(count) * 8.0);
    launch_split_i64(cx.dop_u.as<uint64_t>(), nl, p.n, p.b, count, p.signed_split, lead,
                     cx.dop_out.as<int64_t>(), cx.pflags.as<uint32_t>(), cx.stream);
  }
  TMG_CUDA(cudaGetLastError());
  uint32_t flags = 0;
  TMG_CUDA(cudaMemcpyAsync(out, cx.dop_out.p, size_t(count) * 8, cudaMemcpyDeviceToHost, cx.stream));
  TMG_CUDA(cudaMemcpyAsync(&flags, cx.pflags.p, 4, cudaMemcpyDeviceToHost, cx.stream));
  TMG_CUDA(cudaStreamSynchronize(cx.stream));
  cx.last_kernels = 1;
  if (flags & kFlagInputRange)
    throw Error(TMG_ERR_INPUT_OUT_OF_RANGE, "split: operand outside [0, 2^n)");
  return TMG_OK;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code();
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return TMG_ERR_INTERNAL;
  }
}

}  // namespace
}  // namespace tmg

using namespace tmg;

struct tmg_context {
  Context cx;
};

extern "C" {

const char* tmg_last_error(void) { return g_last_error.c_str(); }
const char* tmg_version(void) { return "truncmul_b200 0.1 (sm_100a)"; }

int tmg_required_precision(int32_t mode, int32_t b, int64_t N, int32_t* out) {
  return guarded([&] {
    *out = required_precision(PMode(mode), b, N);
    return TMG_OK;
  });
}

int tmg_default_lambda(int32_t mode, int32_t backend, int32_t b, int32_t p, int64_t* out) {
  return guarded([&] {
    *out = default_lambda(PMode(mode), Backend(backend), b, p);
    return TMG_OK;
  });
}

int tmg_validate_params(const tmg_params* params) {
  return guarded([&] {
    validate_params(from_c(params));
    return TMG_OK;
  });
}

int tmg_select_params(int64_t n, int32_t mode, int32_t backend, int64_t fallback_cutoff,
                      int32_t policy, tmg_params* out) {
  return guarded([&] {
    Params q = select_params(n, PMode(mode), Backend(backend), fallback_cutoff, Policy(policy));
    to_c(q, out);
    return TMG_OK;
  });
}

int64_t tmg_output_limbs(int32_t mode, int64_t n) { return output_limbs(PMode(mode), n); }

double tmg_predicted_sigma(const tmg_params* p) {
  if (p->mode == TMG_MODE_ORACLE_FALLBACK) return 0.0;
  return predicted_sigma(PMode(p->mode), p->b, p->N);
}

int tmg_context_create(int device, tmg_context** out) {
  return guarded([&] {
    auto c = std::make_unique<tmg_context>();
    init_context(c->cx, device);
    *out = c.release();
    return TMG_OK;
  });
}

void tmg_context_destroy(tmg_context* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->cx.device);
  if (cudaStreamSynchronize(ctx->cx.stream) == cudaSuccess) ctx->cx.drained();
  if (ctx->cx.own_stream && ctx->cx.stream) cudaStreamDestroy(ctx->cx.stream);
  if (ctx->cx.h_status) cudaFreeHost(ctx->cx.h_status);
  delete ctx;
}

int tmg_context_set_stream(tmg_context* ctx, void* stream) {
  return guarded([&] {
    if (ctx->cx.own_stream && ctx->cx.stream) cudaStreamDestroy(ctx->cx.stream);
    ctx->cx.stream = static_cast<cudaStream_t>(stream);
    ctx->cx.own_stream = false;
    return TMG_OK;
  });
}

int tmg_synchronize(tmg_context* ctx) {
  return guarded([&] {
    TMG_CUDA(cudaStreamSynchronize(ctx->cx.stream));
    ctx->cx.drained();
    return TMG_OK;
  });
}

int tmg_full_product(tmg_context* ctx, const tmg_params* params, const uint64_t* u,
                     const uint64_t* v, uint64_t* out, tmg_stats* stats) {
  return guarded([&] {
    return host_product(ctx->cx, from_c(params), TMG_MODE_FULL, u, v, 1, out, nullptr, stats);
  });
}

int tmg_low_product(tmg_context* ctx, const tmg_params* params, const uint64_t* u,
                    const uint64_t* v, uint64_t* out, tmg_stats* stats) {
  return guarded([&] {
    return host_product(ctx->cx, from_c(params), TMG_MODE_LOW, u, v, 1, out, nullptr, stats);
  });
}

int tmg_high_product(tmg_context* ctx, const tmg_params* params, const uint64_t* u,
                     const uint64_t* v, uint64_t* out, tmg_stats* stats) {
  return guarded([&] {
    return host_product(ctx->cx, from_c(params), TMG_MODE_HIGH, u, v, 1, out, nullptr, stats);
  });
}

int tmg_product_batched(tmg_context* ctx, const tmg_params* params, const uint64_t* u,
                        const uint64_t* v, int64_t count, uint64_t* out, uint32_t* flags_out,
                        tmg_stats* stats) {
  return guarded([&] {
    Params q = from_c(params);
    const int32_t m = q.mode == PMode::kOracleFallback ? TMG_MODE_FULL : int32_t(q.mode);
    return host_product(ctx->cx, q, m, u, v, count, out, flags_out, stats);
  });
}

int tmg_alpha_star_f64(tmg_context* ctx, int64_t N, int32_t b, int64_t lambda, const double* in,
                       double* out) {
  return guarded([&] { return map_f64_host(ctx->cx, 0, N, b, lambda, in, 0.0, out, nullptr); });
}

int tmg_beta_star_f64(tmg_context* ctx, int64_t N, int32_t b, int64_t lambda, const double* in,
                      double* out) {
  return guarded([&] { return map_f64_host(ctx->cx, 1, N, b, lambda, in, 0.0, out, nullptr); });
}

int tmg_gamma_dagger_f64(tmg_context* ctx, int64_t N, int32_t b, int64_t lambda, const double* in,
                         double* out, double* aux) {
  return guarded([&] { return map_f64_host(ctx->cx, 2, N, b, lambda, in, 0.0, out, aux); });
}

int tmg_delta_dagger_f64(tmg_context* ctx, int64_t N, int32_t b, int64_t lambda, const double* in,
                         double aux, double* out) {
  return guarded([&] { return map_f64_host(ctx->cx, 3, N, b, lambda, in, aux, out, nullptr); });
}

int tmg_cyclic_convolve_f64(tmg_context* ctx, int64_t n, const double* f, const double* g,
                            double* out) {
  return guarded([&] { return conv_f64_host(ctx->cx, n, f, g, out); });
}

int tmg_split_low_i64(tmg_context* ctx, const tmg_params* params, const uint64_t* u,
                      int64_t* out) {
  return guarded([&] { return split_i64_host(ctx->cx, from_c(params), false, u, out); });
}

int tmg_split_high_i64(tmg_context* ctx, const tmg_params* params, const uint64_t* u,
                       int64_t* out) {
  return guarded([&] { return split_i64_host(ctx->cx, from_c(params), true, u, out); });
}

int tmg_product_device(tmg_context* ctx, const tmg_params* params, const uint64_t* d_u,
                       const uint64_t* d_v, uint64_t* d_out, int64_t count) {
  return guarded([&] {
    Params q = from_c(params);
    if (q.mode == PMode::kOracleFallback)
      throw Error(TMG_ERR_UNSUPPORTED, "device path needs a pipeline parameter set");
    Plan& pl = ctx->cx.plan_for(q);
    enqueue(ctx->cx, pl, d_u, d_v, d_out, count, nullptr, false);
    return TMG_OK;
  });
}

int tmg_check(tmg_context* ctx, tmg_stats* stats) {
  return guarded([&] { return finish(ctx->cx, nullptr, stats); });
}

int tmg_host_alloc(size_t bytes, void** out) {
  return guarded([&] {
    TMG_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocDefault));
    return TMG_OK;
  });
}
void tmg_host_free(void* p) {
  if (p) cudaFreeHost(p);
}
int tmg_device_alloc(size_t bytes, void** out) {
  return guarded([&] {
    TMG_CUDA(cudaMalloc(out, bytes));
    return TMG_OK;
  });
}
void tmg_device_free(void* p) {
  if (p) cudaFree(p);
}
int tmg_memcpy_h2d(tmg_context* ctx, void* dst, const void* src, size_t bytes) {
  return guarded([&] {
    TMG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->cx.stream));
    return TMG_OK;
  });
}
int tmg_memcpy_d2h(tmg_context* ctx, void* dst, const void* src, size_t bytes) {
  return guarded([&] {
    TMG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->cx.stream));
    return TMG_OK;
  });
}
int32_t tmg_last_kernel_count(tmg_context* ctx) { return ctx->cx.last_kernels; }

int tmg_context_set_escalation(tmg_context* ctx, int max_escalations) {
  return guarded([&] {
    if (max_escalations < 0 || max_escalations > 8)
      throw Error(TMG_ERR_INPUT_OUT_OF_RANGE, "escalation count must be in [0, 8]");
    ctx->cx.escalations = max_escalations;
    return TMG_OK;
  });
}

int tmg_context_set_option(tmg_context* ctx, int32_t option, int64_t value) {
  return guarded([&] {
    Options& o = ctx->cx.opt;
    const bool on = value != 0;
    switch (option) {
      case TMG_OPT_GENERIC_COLUMN_PASSES: o.plan.generic_columns = on; break;
      case TMG_OPT_FORCE_THREE_PASS: o.plan.force_three_pass = on; break;
      case TMG_OPT_GENERIC_ROW_PASS: o.generic_row = o.plan.generic_row = on; break;
      case TMG_OPT_LOOKBACK_CARRY: o.lookback_carry = on; break;
      case TMG_OPT_PATCH_SCAN_MAX:
        if (value < 0) throw Error(TMG_ERR_INPUT_OUT_OF_RANGE, "patch scan limit must be >= 0");
        o.patch_scan_max = long(value);
        break;
      case TMG_OPT_NO_PDL: o.no_pdl = on; break;
      case TMG_OPT_DEBUG_SYNC: o.debug_sync = on; break;
      case TMG_OPT_NO_GRAPH: o.no_graph = on; break;
      case TMG_OPT_Z_NATURAL: o.z_natural = o.plan.z_natural = on; break;
      case TMG_OPT_GENERIC_SMALL: o.generic_small = on; break;
      case TMG_OPT_PREMAP_IN_SPLIT: o.plan.premap_in_zgen = on; break;
      case TMG_OPT_SPLIT_AGGREGATES: o.zstat_split = on; break;
      case TMG_OPT_GENERIC_RUNS: o.generic_runs = on; break;
      case TMG_OPT_SPLIT_KERNEL: o.old_split = on; break;
      case TMG_OPT_MAX_ROW:
        if (value < 0 || value > 4096) throw Error(TMG_ERR_INPUT_OUT_OF_RANGE, "row length cap in [0, 4096]");
        o.plan.max_row = uint32_t(value);
        break;
      case TMG_OPT_CARRY_KERNELS:
        if (value < 0 || value > 4) throw Error(TMG_ERR_INPUT_OUT_OF_RANGE, "carry kernels: 0 to 4");
        o.carry_kernels = int(value);
        break;
      default: throw Error(TMG_ERR_INPUT_OUT_OF_RANGE, "unknown context option");
    }
    // plans and captured batch graphs were built under the old options
    TMG_CUDA(cudaStreamSynchronize(ctx->cx.stream));
    ctx->cx.plans.clear();
    ctx->cx.clear_graphs();
    return TMG_OK;
  });
}

int tmg_debug_read(tmg_context* ctx, int which, void* host, size_t* bytes) {
  return guarded([&] {
    Context& cx = ctx->cx;
    const DevBuf& B = (which == 0) ? cx.ws0.work_z : cx.ws0.work_c;
    if (which != 0 && which != 1) throw Error(TMG_ERR_INPUT_OUT_OF_RANGE, "debug_read: which");
    *bytes = std::min(*bytes, B.bytes);
    TMG_CUDA(cudaMemcpyAsync(host, B.p, *bytes, cudaMemcpyDeviceToHost, cx.stream));
    TMG_CUDA(cudaStreamSynchronize(cx.stream));
    cx.drained();
    return TMG_OK;
  });
}

int tmg_profile_enable(tmg_context* ctx, int on) {
  return guarded([&] {
    ctx->cx.prof.on = on != 0;
    return TMG_OK;
  });
}

int tmg_profile_read(tmg_context* ctx, char* names, int name_stride, double* ms,
                     double* bytes, int max_records, int* count) {
  return guarded([&] {
    Profiler& P = ctx->cx.prof;
    TMG_CUDA(cudaStreamSynchronize(ctx->cx.stream));
    ctx->cx.drained();
    int n = 0;
    for (auto& r : P.recs) {
      if (n < max_records) {
        float t = 0.f;
        TMG_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
        std::strncpy(names + size_t(n) * name_stride, r.name.c_str(), size_t(name_stride - 1));
        names[size_t(n) * name_stride + name_stride - 1] = 0;
        ms[n] = double(t);
        bytes[n] = r.bytes;
        ++n;
      }
      P.pool.push_back(r.a);
      P.pool.push_back(r.b);
    }
    P.recs.clear();
    *count = n;
    return TMG_OK;
  });
}

}  // extern "C"
