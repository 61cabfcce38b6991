// Device plans: transform shape, radix schedules, twiddle tables and the
// map constants of one parameter set.
#pragma once

#include <atomic>
#include <cstdint>
#include <map>
#include <string>
#include <memory>
#include <vector>

#include "kernels.cuh"
#include "params.hpp"

namespace tmg {

// Owned device allocation.
// Bumped whenever a DevBuf reallocates (captured batch graphs key on it).
extern std::atomic<uint64_t> g_devbuf_generation;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf();
  void ensure(size_t nbytes);  // grows, contents not kept
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

// Twiddle tables keyed by length, shared by all plans of a context.
class TwiddleCache {
 public:
  const double2* table(uint32_t R);               // omega_R^x, x < R
  TwGlobal global(uint64_t L);                    // two-level omega_L
  const double2* stage_table(uint32_t R, int maxrad = 16);  // per-stage q-major table
  const double2* stage_table(uint32_t R, const std::vector<int>& rad);
 private:
  std::map<std::string, std::unique_ptr<DevBuf>> stages_;
  std::map<uint64_t, std::unique_ptr<DevBuf>> tables_;
  std::map<uint64_t, std::unique_ptr<DevBuf>> glob_;
  std::map<uint64_t, uint32_t> glob_S_;
};

SubFft make_subfft(uint32_t R, const double2* tw, uint32_t tw_stride, TwiddleCache* cache,
                   int maxrad = 16);
SubFft make_subfft_rad(uint32_t R, const std::vector<int>& rad, const double2* tw,
                       uint32_t tw_stride, TwiddleCache* cache);
MapConsts make_map_consts(const Params& p);

struct Plan {
  Params params;
  int kind = 0;  // 1 fused single CTA, 2 two-pass, 3 three-pass, 0 basecase
  int64_t L = 0;
  uint32_t A = 1, B = 1, C = 1;
  int64_t count = 0;  // chunks per operand
  int64_t lead = 0;
  int64_t K = 0;      // recombination coefficients
  int64_t ML = 0;     // limbs scanned by the carry
  int32_t shift_s = 0;
  int64_t nlimbs = 0;
  int64_t out_limbs = 0;
  MapConsts mc{};
  // fused
  SubFft fwd{}, inv{};
  size_t small_smem = 0;
  int small_threads = 0;
  bool small_batch = false;  // multi-pass plan whose batches run the fused kernel
  // multi-pass
  SubFft fA{}, iA{}, fB{}, iB{}, fC{}, iC{};
  TwGlobal twL{};
  uint32_t logc_f1 = 0, logc_f2 = 0, logc_i2 = 0, logc_il = 0;
  size_t smem_f1 = 0, smem_f2 = 0, smem_i2 = 0, smem_il = 0, smem_mid = 0,
         smem_carry = 0;
  bool f1_stw = false;  // k_f1 stages its inter-pass twiddles per CTA
  const ColCtShape* colct = nullptr;     // compile-time first column pass (k_f1_ct)
  const ColCtShape* colct_il = nullptr;  // compile-time last column pass (k_ilast_ct)
  const ColCtShape* colct_b = nullptr;   // three-pass plans: middle column passes (k_col_ct)
  F1Fn f1d = nullptr;  // first column pass with the pre-map folded in (k_f1d_ct)
  int zdig = 0;        // with f1d: k_zgen stores digits, 1 short2 / 2 int2
  int thr_f1 = 0, thr_f2 = 0, thr_i2 = 0, thr_il = 0, thr_mid = 0;
  size_t smem_zgen = 0;
  bool mid_shared_table = false;
  bool mid_ct = false;  // C = 2048 / 1024 with a compiled row pass (k_mid_2048 / k_mid_1024)
  bool colpp = false;  // column passes use the ping-pong kernels (k_*_pp)
  int kernels = 0;
};

// Plan-shape choices a context can switch for testing (tmg_context_set_option);
// the defaults are the measured-best shapes.
struct PlanOptions {
  bool generic_columns = false;  // runtime-dispatched column passes, not the compiled shapes
  bool generic_row = false;      // the runtime-dispatched row pass k_mid, not the compiled ones
  bool force_three_pass = false; // three-pass plans for short column lengths
  bool premap_in_zgen = false;   // k_zgen pre-maps (double2 z), k_f1_ct reads z; not k_f1d_ct
  bool z_natural = false;        // z in natural order (k_f1d_ct needs the tile order)
  uint32_t max_row = 0;          // longest row length C (0: 4096)
};

std::unique_ptr<Plan> build_plan(const Params& p, TwiddleCache& tw, const PlanOptions& opt);

}  // namespace tmg
