// gpp_lib.cu -- host side of libgpp_b200.so: the C ABI declared in
// include/gpp_b200.h, the device-buffer manager, launch planning, the NCCL
// band-shard combine and the FP64 peak microbenchmark.
#include <cuda_runtime.h>
#include <nccl.h>
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <list>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "gpp_b200.h"
#include "gpp_kernels.cuh"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  const int code = (e == cudaErrorMemoryAllocation) ? GPP_ERR_OOM : GPP_ERR_CUDA;
  return fail(code, std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                        cudaGetErrorString(e) + ")");
}

#define GPP_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);  \
  } while (0)

#define GPP_NCCL(call)                                                              \
  do {                                                                              \
    ncclResult_t _r = (call);                                                       \
    if (_r != ncclSuccess)                                                          \
      return fail(GPP_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(_r)); \
  } while (0)

// Restores the caller's current device on scope exit, so the library never
// leaves torch (or any other caller) on a different device.
struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    err = cudaGetDevice(&prev);
    if (err != cudaSuccess) return;
    if (prev != dev) err = cudaSetDevice(dev);
    ok = (err == cudaSuccess);
  }
  ~DeviceGuard() {
    if (ok && prev >= 0) cudaSetDevice(prev);
  }
};

template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;  // elements
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&ptr, std::max<size_t>(n, 1) * sizeof(T));
    if (e == cudaSuccess) cap = n;
    return e;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

// ----- launch planning ------------------------------------------------------
struct Plan {
  int igp_t = 4;
  int bchunk = gpp::kMaxChunk;
  int n_igblk = 1, n_igptile = 1;
  long long n_items = 1;
  int grid = 1;
  int blocks_per_sm = 1;
  int regs = 0;
};

// One launch of the production kernel: rows [row0, row0 + n_rows) of (igb,
// igp tile) pairs times the band chunks of the window [wb0, wb0 + wnb); the
// first n_items items (item = chunk * n_rows + row - row0).  `tail`: a
// balanced-tail launch (run on the other stream).
struct SaccLaunch {
  int row0, n_rows;
  int64_t wb0, wnb;
  int bchunk;
  long long n_items;
  bool tail = false;
};

struct CanonLaunch : SaccLaunch {
  long long slot0 = 0;
};
struct Canon {
  Plan pl;
  int n_rows = 0;
  std::vector<CanonLaunch> ls;
  long long n_slots = 0;
};

}  // namespace

struct gpp_ctx {
  int device = -1;
  uint64_t launches = 0;  // kernels this context has launched (gpp_launch_count)
  bool initialized = false;
  cudaStream_t stream = nullptr;
  cudaStream_t cstream = nullptr;  // H2D copies of the pipelined evaluate
  cudaStream_t kstream2 = nullptr;  // odd ig slabs: overlaps a slab's tail with the next
  cudaStream_t nstream = nullptr;   // NCCL broadcasts of the column-split upload
  cudaEvent_t ev_we = nullptr;      // wtilde / eps complete (column-split upload)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> slab_ev;
  int num_sms = 0;

  // Problem (local band shard).
  bool have_problem = false;
  int64_t nbands = 0, ngpown = 0, ncouls = 0;
  int nw = 0;
  double wxmax = 0.0;  // max |wx| over the uploaded shard

  DevBuf<double2> wtilde, eps, aqsn, aqsm;
  DevBuf<double> wxb;
  DevBuf<double> partials;
  DevBuf<unsigned long long> cpartials;
  DevBuf<double> out;                  // 4 * nw
  DevBuf<unsigned long long> counts;   // 2
  double* h_out = nullptr;             // pinned staging
  unsigned long long* h_counts = nullptr;
  size_t h_out_cap = 0;
  double* h_wx = nullptr;              // pinned staging for the expanded wx
  size_t h_wx_cap = 0;

  // Pinned staging ring for pageable host inputs (copy_rows): kStageSlots
  // buffers of stage_cap bytes; slot k is free once stage_ev[k] completed.
  static constexpr int kStageSlots = 16;  // capacity; stage_slots() in use
  unsigned char* h_stage[kStageSlots] = {};
  size_t stage_cap = 0;
  cudaEvent_t stage_ev[kStageSlots] = {};
  int stage_next = 0;
  uint64_t staged_bytes = 0;  // bytes that went through the staging ring (gpp_stats)

  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  bool comm_aborted = false;  // an error after comm init aborted the communicator

  // Launch plans of the uploaded problem, keyed by (variant, nw group, count);
  // cleared whenever a problem is (re)loaded.
  std::vector<std::pair<int, std::vector<int64_t>>> plan_cache;
  // Canonical schedules of the production kernel, keyed by (nw group, count).
  std::list<std::pair<int, Canon>> canon_cache;
  DevBuf<double> stage;      // slot finalize: per-block sums
  DevBuf<unsigned> ticket;   // slot finalize: last-block ticket (self-resetting)
  std::mutex mu;             // one caller at a time (the ABI's contexts are shareable)

  // Factored path (gpp_run_factored): needs a band-invariant wx.
  bool wx_band_invariant = false;
};

namespace {

// One caller at a time per context (the reference allows independent runs to
// proceed concurrently: distinct contexts run in parallel, a
// shared one serialises).  Group calls lock every context in address order.
struct CtxLock {
  std::vector<std::mutex*> ms;
  explicit CtxLock(gpp_ctx* c) {
    if (c) ms.push_back(&c->mu);
    for (auto* m : ms) m->lock();
  }
  CtxLock(gpp_ctx* const* cs, int n) {
    for (int i = 0; cs && i < n; ++i)
      if (cs[i]) ms.push_back(&cs[i]->mu);
    std::sort(ms.begin(), ms.end());
    ms.erase(std::unique(ms.begin(), ms.end()), ms.end());
    for (auto* m : ms) m->lock();
  }
  ~CtxLock() {
    for (auto it = ms.rbegin(); it != ms.rend(); ++it) (*it)->unlock();
  }
  CtxLock(const CtxLock&) = delete;
  CtxLock& operator=(const CtxLock&) = delete;
};

int ensure_init(gpp_ctx* c) {
  if (c->initialized) return GPP_OK;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (c->device >= n)
    return fail(GPP_ERR_ARG, "device " + std::to_string(c->device) + " out of range (" +
                                 std::to_string(n) + " devices)");
  DeviceGuard g(c->device);
  if (!g.ok) return cuda_fail(g.err, "cudaSetDevice");
  GPP_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  GPP_CUDA(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
  GPP_CUDA(cudaStreamCreateWithFlags(&c->kstream2, cudaStreamNonBlocking));
  GPP_CUDA(cudaStreamCreateWithFlags(&c->nstream, cudaStreamNonBlocking));
  GPP_CUDA(cudaEventCreateWithFlags(&c->ev_we, cudaEventDisableTiming));
  for (auto& ev : c->ev) GPP_CUDA(cudaEventCreate(&ev));
  GPP_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  GPP_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  GPP_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
  c->initialized = true;
  return GPP_OK;
}

// ----- launch planning ------------------------------------------------------

using KernelFn = void (*)(gpp::Params);
// The production kernel also takes its band window's wx as a by-value table.
using SaccFn = void (*)(gpp::Params, gpp::WxTable);
struct KernelRef {
  KernelFn fn = nullptr;
  SaccFn sacc = nullptr;
  size_t smem = 0;  // dynamic shared memory of the sacc kernels
  const void* ptr() const {
    return fn ? reinterpret_cast<const void*>(fn) : reinterpret_cast<const void*>(sacc);
  }
};

// Launch-shape override for experiments: GPP_TUNE="igp,bps[,bchunk]" forces
// the igp tile (2..4) of the ladder rcp_sq kernels at nw 2/3, caps resident
// CTAs per SM and (optionally) fixes the band chunk.
// Unset (the default) the planner chooses.
struct Tune {
  int igp = 0, bps = 0, bchunk = 0;
};
Tune read_tune() {
  Tune t;
  const char* e = std::getenv("GPP_TUNE");
  if (e) std::sscanf(e, "%d,%d,%d", &t.igp, &t.bps, &t.bchunk);
  return t;
}

// The igp tile actually instantiated for a frequency group: 3 or 4 igp per
// thread below four frequencies (2 only as a GPP_TUNE experiment at nw 2/3),
// 3 at four (the 4x4 state does not fit 128 registers).
int fast_igp(int nw, int igp_t) {
  if (nw >= 4) return 3;
  if (igp_t == 2) return (nw == 2 || nw == 3) ? 2 : 3;
  return igp_t == 4 ? 4 : 3;
}

template <class FP, int NW, bool C>
KernelFn pick_fast(int igp_t) {
  if constexpr (NW < 4) {
    if (igp_t == 4) return gpp::gpp_main_kernel<FP, NW, 4, C>;
  }
  if constexpr (NW == 2 || NW == 3) {
    if (igp_t == 2) return gpp::gpp_main_kernel<FP, NW, 2, C>;
  }
  return gpp::gpp_main_kernel<FP, NW, 3, C>;
}

template <class FP, bool C>
KernelFn pick_fast_nw(int nw, int igp_t) {
  switch (nw) {
    case 1: return pick_fast<FP, 1, C>(igp_t);
    case 2: return pick_fast<FP, 2, C>(igp_t);
    case 3: return pick_fast<FP, 3, C>(igp_t);
    default: return pick_fast<FP, 4, C>(igp_t);
  }
}

template <class P, bool C>
KernelFn pick_plain(int nw) {
  switch (nw) {
    case 1: return gpp::gpp_main_kernel<P, 1, 2, C>;
    case 2: return gpp::gpp_main_kernel<P, 2, 2, C>;
    case 3: return gpp::gpp_main_kernel<P, 3, 2, C>;
    default: return gpp::gpp_main_kernel<P, 4, 2, C>;
  }
}

// Production kernel: igp tile per frequency-group size, the largest tile
// whose S sums fit the 128-register budget without spills (ptxas -v).
// Four-frequency groups keep the one-seed kernel (FastPolicy3): their S sums
// do not fit beside the ach/asx shared-memory slab.
int sacc_cap(int nw) { return nw >= 2 ? gpp::sacc_cap<3>() : gpp::sacc_cap<1>(); }

// The production kernel's igp tile for a frequency group of nw and a problem
// of ngpown igp columns: the tile of least padded cost, ceil(ngpown / T) * T
// columns weighted by the measured per-column time of each instantiation
// relative to the two-igp tile (tools/probe_variants_sweep.py, all 24 sweep
// points at nw 2 and 3): nw 3: T = 3 x 0.984, T = 4 x 0.980 (one CTA per SM);
// nw 2: T = 3 x 0.985, T = 4 x 0.945.  One frequency keeps T = 3 (two CTAs
// per SM; one CTA per SM measured 4 % slower).  The rule picks the fastest
// measured tile at every sweep point.
int sacc_igp(int nw, int64_t ngpown) {
  if (nw <= 1) return 3;
  const double w3 = nw >= 3 ? 0.984 : 0.985, w4 = nw >= 3 ? 0.980 : 0.945;
  const double c2 = static_cast<double>((ngpown + 1) / 2 * 2);
  const double c3 = w3 * static_cast<double>((ngpown + 2) / 3 * 3);
  const double c4 = w4 * static_cast<double>((ngpown + 3) / 4 * 4);
  if (c4 <= c3 && c4 < c2) return 4;
  if (c3 < c2) return 3;
  return 2;
}

// Resident CTAs per SM of the production kernel for (nw, igp tile), as its
// launch bounds declare (the occupancy API confirms it at plan time).
int sacc_blocks_per_sm(int nw, int igp_t) { return (nw >= 2 && igp_t >= 3) ? 1 : 2; }

template <int NW, int IGP_T, bool C>
KernelRef sacc_ref() {
  KernelRef k;
  k.sacc = gpp::gpp_sacc_kernel<NW, IGP_T, C>;
  k.smem = gpp::sacc_smem_bytes<NW, IGP_T>();
  return k;
}

template <bool C>
KernelRef pick_sacc(int nw, int igp_t) {
  switch (nw) {
    case 1: return sacc_ref<1, 3, C>();
    case 2:
      return igp_t == 4 ? sacc_ref<2, 4, C>() : igp_t == 3 ? sacc_ref<2, 3, C>() : sacc_ref<2, 2, C>();
    case 3:
      return igp_t == 4 ? sacc_ref<3, 4, C>() : igp_t == 3 ? sacc_ref<3, 3, C>() : sacc_ref<3, 2, C>();
    default: {
      KernelRef k;
      k.fn = gpp::gpp_main_kernel<gpp::FastPolicy, 4, 3, C>;
      return k;
    }
  }
}

template <bool C>
KernelRef pick_kernel_c(int variant, int nw, int igp_t) {
  KernelRef k;
  switch (variant) {
    case GPP_VARIANT_DIV: k.fn = pick_plain<gpp::PlainPolicy<0>, C>(nw); break;
    case GPP_VARIANT_RCP: k.fn = pick_plain<gpp::PlainPolicy<1>, C>(nw); break;
    case GPP_KERNEL_SQ_SPLIT: k.fn = pick_fast_nw<gpp::FastPolicyT<0, 2>, C>(nw, igp_t); break;
    case GPP_KERNEL_IW_HOIST: k.fn = pick_fast_nw<gpp::FastPolicyT<1, 3>, C>(nw, igp_t); break;
    case GPP_KERNEL_ONE_SEED: k.fn = pick_fast_nw<gpp::FastPolicy, C>(nw, igp_t); break;
    default: k = pick_sacc<C>(nw, igp_t); break;
  }
  return k;
}

// count: whether the kernel also produces the near/far branch counts (the
// reference's branch_stats, kernel.py:130-137).  The uncounted kernel is the
// evaluate_variant path; the counted one costs two predicated integer adds
// per instance.
KernelRef pick_kernel(int variant, int nw, int igp_t, bool count) {
  return count ? pick_kernel_c<true>(variant, nw, igp_t) : pick_kernel_c<false>(variant, nw, igp_t);
}

using FinalizeFn = void (*)(const double*, const unsigned long long*, int, int, int, int, int,
                            int, double*, unsigned long long*);
FinalizeFn pick_finalize(int nw) {
  switch (nw) {
    case 1: return gpp::gpp_finalize_kernel<1>;
    case 2: return gpp::gpp_finalize_kernel<2>;
    case 3: return gpp::gpp_finalize_kernel<3>;
    default: return gpp::gpp_finalize_kernel<4>;
  }
}

// igp tile for the fast kernel: 3 or 4 igp per thread.  Padded igp columns
// cost full work, and the 4-wide tile runs ~5 % slower per instance under the
// 128-register budget (tools/sweep.py, profiles/r01_sweep.jsonl), so pick the
// smaller padded cost with that weight.
int choose_igp_tile(int64_t ngpown) {
  const double cost3 = static_cast<double>((ngpown + 2) / 3 * 3);
  const double cost4 = 1.05 * static_cast<double>((ngpown + 3) / 4 * 4);
  return cost4 < cost3 ? 4 : 3;
}

// Band chunk: minimise the modelled makespan of the static round-robin,
//   ceil(items / resident CTAs) * (chunk + kItemOverheadBands),
// where an item's fixed cost (state load, staging, barrier, epilogue) was
// measured at ~4 bands' worth of work (tools/probe_shard.py: step time of
// 1/N band shards).  Long chunks amortise that cost; short ones balance
// small shards (and small ig slabs) across the 148 SMs.
// Modelled cost, in band-steps of one CTA slot, of the balanced tail of a
// partial last wave (split_tail): R rows of an nb_last-band chunk cut into
// sub-chunks; 0 in *bc_out when no cut beats one more wave of whole items.
constexpr double kItemOverheadBands = 4.0;  // measured fixed cost of an item, in bands

double tail_cost(long long R, int64_t nb_last, long long slots, int* bc_out) {
  double best = static_cast<double>(nb_last) + kItemOverheadBands;
  *bc_out = 0;
  for (int64_t k = 2; k <= nb_last; ++k) {
    const int64_t bc = (nb_last + k - 1) / k, subs = (nb_last + bc - 1) / bc;
    const long long waves = (R * subs + slots - 1) / slots;
    const double cost = static_cast<double>(waves) * (static_cast<double>(bc) + kItemOverheadBands);
    if (cost < best - 0.5) {
      best = cost;
      *bc_out = static_cast<int>(bc);
    }
  }
  return best;
}

bool balanced_tail_enabled();

// Band chunk: minimise the modelled makespan of the static round-robin,
//   full waves x (chunk + kItemOverheadBands) + the last wave,
// where the last (partial) wave costs one more whole item, or -- for the
// production kernel, which balances it (split_tail) -- its tail_cost.  Long
// chunks amortise the per-item cost (state, staging, barrier, epilogue);
// short ones balance small shards (and small ig slabs) across the SMs.
int choose_bchunk(long long n_igblk, long long n_igptile, int64_t nbands, long long slots,
                  int max_chunk, bool balanced) {
  const long long n_rows = n_igblk * n_igptile;
  int bchunk = 8;
  double best = -1.0;
  for (int bc = 8; bc <= max_chunk; bc *= 2) {
    const int eff = static_cast<int>(std::min<int64_t>(bc, nbands));
    const long long n_chunks = (nbands + eff - 1) / eff;
    const long long items = n_rows * n_chunks;
    const long long full = items / slots, R = items % slots;
    double cost = static_cast<double>((items + slots - 1) / slots) * (eff + kItemOverheadBands);
    if (balanced && full >= 1 && R > 0 && R <= n_rows) {
      int bc2 = 0;
      const int64_t nb_last = nbands - (n_chunks - 1) * eff;
      cost = static_cast<double>(full) * (eff + kItemOverheadBands) + tail_cost(R, nb_last, slots, &bc2);
    }
    if (best < 0.0 || cost < best) {
      best = cost;
      bchunk = eff;
    }
    if (eff >= nbands) break;
  }
  return bchunk;
}

int make_plan_uncached(gpp_ctx* c, int variant, int nw_group, bool count, Plan* pl) {
  // The plain (as-written) variants keep two igp per thread and the fast
  // kernel drops to 3 at four frequencies: both choices avoid spills under
  // the 128-register budget of __launch_bounds__(256, 2).
  const Tune tune = read_tune();
  if (variant == GPP_VARIANT_DIV || variant == GPP_VARIANT_RCP)
    pl->igp_t = 2;  // the only instantiation of the plain kernels
  else if (variant == GPP_VARIANT_RCP_SQ)
    pl->igp_t = sacc_igp(nw_group, c->ngpown);
  else
    pl->igp_t = fast_igp(nw_group, tune.igp >= 2 && tune.igp <= 4 ? tune.igp
                                                                  : choose_igp_tile(c->ngpown));
  pl->n_igblk = static_cast<int>((c->ncouls + gpp::kThreads - 1) / gpp::kThreads);
  pl->n_igptile = static_cast<int>((c->ngpown + pl->igp_t - 1) / pl->igp_t);
  const KernelRef fn = pick_kernel(variant, nw_group, pl->igp_t, count);
  int bps = 0;
  // Dynamic shared memory above the 48 KB default needs an opt-in (per device:
  // plans are made per context, with its device current).
  if (fn.smem > 0)
    GPP_CUDA(cudaFuncSetAttribute(fn.ptr(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(fn.smem)));
  GPP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn.ptr(), gpp::kThreads, fn.smem));
  cudaFuncAttributes attr;
  GPP_CUDA(cudaFuncGetAttributes(&attr, fn.ptr()));
  pl->regs = attr.numRegs;
  pl->blocks_per_sm = std::max(bps, 1);
  if (tune.bps > 0) pl->blocks_per_sm = std::min(pl->blocks_per_sm, tune.bps);
  const long long slots = static_cast<long long>(pl->blocks_per_sm) * c->num_sms;
  const int max_chunk = fn.sacc ? sacc_cap(nw_group) : gpp::kMaxChunk;
  const int bchunk = tune.bchunk > 0 ? static_cast<int>(std::min<int64_t>(
                                           std::min(tune.bchunk, max_chunk), c->nbands))
                                     : choose_bchunk(pl->n_igblk, pl->n_igptile, c->nbands,
                                                     slots, max_chunk,
                                                     fn.sacc && balanced_tail_enabled());
  pl->bchunk = bchunk;
  pl->n_items = static_cast<long long>(pl->n_igblk) * pl->n_igptile *
                ((c->nbands + bchunk - 1) / bchunk);
  pl->grid = static_cast<int>(std::min<long long>(slots, pl->n_items));
  return GPP_OK;
}

// make_plan_uncached, memoised per context: the occupancy / attribute queries
// cost host time that would otherwise dominate small problems.
int make_plan(gpp_ctx* c, int variant, int nw_group, bool count, Plan* pl) {
  const int key = (variant * 16 + nw_group) * 2 + (count ? 1 : 0);
  for (const auto& e : c->plan_cache) {
    if (e.first == key) {
      const std::vector<int64_t>& v = e.second;
      pl->igp_t = static_cast<int>(v[0]);
      pl->bchunk = static_cast<int>(v[1]);
      pl->n_igblk = static_cast<int>(v[2]);
      pl->n_igptile = static_cast<int>(v[3]);
      pl->n_items = v[4];
      pl->grid = static_cast<int>(v[5]);
      pl->blocks_per_sm = static_cast<int>(v[6]);
      pl->regs = static_cast<int>(v[7]);
      return GPP_OK;
    }
  }
  int rc = make_plan_uncached(c, variant, nw_group, count, pl);
  if (rc) return rc;
  c->plan_cache.emplace_back(key, std::vector<int64_t>{pl->igp_t, pl->bchunk, pl->n_igblk,
                                                       pl->n_igptile, pl->n_items, pl->grid,
                                                       pl->blocks_per_sm, pl->regs});
  return GPP_OK;
}

// Frequency groups of one evaluation (one launch sequence each).  The
// production kernel takes at most three frequencies per launch (its S sums
// for four do not fit the register budget), so for nw >= 4 it runs
// ceil(nw / 3) balanced groups -- e.g. 2 + 2 at nw 4 -- which the register-
// file model rates at 46-49 reads per instance against 56 for the four-wide
// one-seed kernel.  The other kernels take groups of four.
int max_group(int variant) { return variant == GPP_VARIANT_RCP_SQ ? 3 : gpp::kMaxNwGroup; }

int nw_groups(int nw, int gmax, std::vector<std::pair<int, int>>* groups) {
  groups->clear();
  const int n = (nw + gmax - 1) / gmax;
  for (int k = 0, iw0 = 0; k < n; ++k) {
    const int sz = nw / n + (k < nw % n ? 1 : 0);
    groups->emplace_back(iw0, sz);
    iw0 += sz;
  }
  return GPP_OK;
}


// Balanced tail: the static round-robin leaves the last wave's R items (the
// last R rows of the last band chunk) on R of the `slots` resident CTAs while
// the others idle.  If that wave is partial, run the whole waves as one launch
// and those R rows' last chunk as a second launch cut into finer band chunks,
// when the modelled makespan (waves x (chunk + per-item overhead)) drops.
// GPP_BALANCED_TAIL=0 keeps one launch per window: ncu captures of a whole
// evaluation in one launch (tools/profile_run.py, tools/ladder.py).
bool balanced_tail_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GPP_BALANCED_TAIL");
    return !(e && e[0] == '0');
  }();
  return on;
}

void split_tail(std::vector<SaccLaunch>& ls, long long slots) {
  if (!balanced_tail_enabled()) return;
  const SaccLaunch L = ls[0];
  const long long R = L.n_items % slots, full = L.n_items / slots;
  if (full < 1 || R == 0 || R > L.n_rows) return;
  const int64_t n_chunks = (L.wnb + L.bchunk - 1) / L.bchunk;
  const int64_t last_b0 = (n_chunks - 1) * L.bchunk, nb_last = L.wnb - last_b0;
  int best_bc = 0;
  tail_cost(R, nb_last, slots, &best_bc);
  if (best_bc == 0) return;
  ls[0].n_items = full * slots;
  const int64_t subs = (nb_last + best_bc - 1) / best_bc;
  ls.push_back({L.n_rows - static_cast<int>(R), static_cast<int>(R), L.wb0 + last_b0, nb_last,
                best_bc, R * subs, true});
}

// Launches of one band window [wb0, wb0 + wnb) over all n_rows rows: whole
// items plus, for the production kernel, the balanced tail.  Pure host logic.
std::vector<SaccLaunch> window_launches(int n_rows, int64_t wb0, int64_t wnb, int bchunk,
                                        long long slots, bool sacc) {
  const long long n_chunks = (wnb + bchunk - 1) / bchunk;
  std::vector<SaccLaunch> launches{{0, n_rows, wb0, wnb, bchunk,
                                    static_cast<long long>(n_rows) * n_chunks, false}};
  if (sacc) split_tail(launches, slots);
  return launches;
}

// ----- the canonical schedule of the production kernel -----------------------
// The whole-problem plan of one frequency group (band windows, each with its
// whole-wave launch and balanced tail) numbers every item once: the item
// (chunk, row) of canonical launch L owns slot L.slot0 + chunk * L.n_rows +
// row - L.row0.  Every schedule that evaluates the problem -- the resident
// run, the ig-slab pipelined evaluate_host, any grid size -- runs exactly
// these items (the same band ranges per row) and writes each item's per-warp
// partial to its slot; the finalize sums the slots in order.  So the result
// is bitwise the same for every schedule, while each schedule
// keeps its own launch boundaries and grid.

std::vector<CanonLaunch> canon_launches(int n_igblk, int n_igptile, int64_t nbands, int nwg,
                                        int plan_bchunk, long long slots, long long* n_slots) {
  const int64_t win = gpp::kWxParam / nwg;
  const int n_rows = n_igblk * n_igptile;
  std::vector<CanonLaunch> all;
  long long slot = 0;
  for (int64_t wb0 = 0; wb0 < nbands; wb0 += win) {
    const int64_t wnb = std::min<int64_t>(win, nbands - wb0);
    // A window shorter than the whole band range re-plans its band chunk.
    const int bchunk = wnb == nbands ? plan_bchunk
                                     : choose_bchunk(n_igblk, n_igptile, wnb, slots, sacc_cap(nwg),
                                                     balanced_tail_enabled());
    for (const SaccLaunch& L : window_launches(n_rows, wb0, wnb, bchunk, slots, true)) {
      CanonLaunch C;
      static_cast<SaccLaunch&>(C) = L;
      C.slot0 = slot;
      slot += L.n_items;
      all.push_back(C);
    }
  }
  *n_slots = slot;
  return all;
}

int make_canon(gpp_ctx* c, int nwg, bool count, const Canon** out) {
  const int key = nwg * 2 + (count ? 1 : 0);
  for (const auto& e : c->canon_cache)
    if (e.first == key) {
      *out = &e.second;
      return GPP_OK;
    }
  Canon cn;
  int rc = make_plan(c, GPP_VARIANT_RCP_SQ, nwg, count, &cn.pl);
  if (rc) return rc;
  cn.n_rows = cn.pl.n_igblk * cn.pl.n_igptile;
  const long long slots = static_cast<long long>(cn.pl.blocks_per_sm) * c->num_sms;
  cn.ls = canon_launches(cn.pl.n_igblk, cn.pl.n_igptile, c->nbands, nwg, cn.pl.bchunk, slots,
                         &cn.n_slots);
  c->canon_cache.emplace_back(key, std::move(cn));
  *out = &c->canon_cache.back().second;
  return GPP_OK;
}

// The items of canonical launch L whose rows lie in [r0, r1), as one launch
// (rows [rr0, rr1), the same chunks; of the last chunk only the rows L runs).
bool sub_launch(const CanonLaunch& L, int r0, int r1, SaccLaunch* out) {
  const int rr0 = std::max(r0, L.row0), rr1 = std::min(r1, L.row0 + L.n_rows);
  if (rr0 >= rr1) return false;
  const long long n_chunks = (L.wnb + L.bchunk - 1) / L.bchunk;
  const long long before_last = (n_chunks - 1) * static_cast<long long>(L.n_rows);
  const long long lim = L.row0 + (L.n_items - before_last);  // rows run in the last chunk
  const int n = rr1 - rr0;
  const long long in_last = std::min<long long>(std::max<long long>(lim - rr0, 0), n);
  *out = {rr0, n, L.wb0, L.wnb, L.bchunk, (n_chunks - 1) * n + in_last, L.tail};
  return out->n_items > 0;
}

// ----- one evaluation, enqueued in pieces ------------------------------------
// eval_begin -> eval_rows(ig blocks [blk0, blk1), after `ready`) ... ->
// eval_end.  The production kernel runs each piece's canonical items as it
// is enqueued (pieces alternate between the two compute streams, the tail
// launches take the other one); the other kernels run the whole problem in
// eval_end (after every piece's `ready` event), so their partial rows -- and
// bits -- do not depend on the pieces either.
struct EvalRun {
  int variant = 0;
  bool count = false, sacc = false;
  std::vector<std::pair<int, int>> groups;
  std::vector<const Canon*> canon;   // per group (production kernel)
  std::vector<size_t> part_off;      // per group: first double of its slots in c->partials
  cudaEvent_t* ev_main = nullptr;
  int piece = 0;
  std::vector<cudaEvent_t> pending;  // other kernels: waits deferred to eval_end
};

constexpr int kSlotsPerFinalizeBlock = 32;

int eval_begin(gpp_ctx* c, int variant, bool count, cudaEvent_t* ev_main, EvalRun* r) {
  r->variant = variant;
  r->count = count;
  r->ev_main = ev_main;
  nw_groups(c->nw, max_group(variant), &r->groups);
  r->sacc = variant == GPP_VARIANT_RCP_SQ;
  if (r->sacc) {
    long long max_slots = 0;
    size_t doubles = 0;
    for (const auto& g : r->groups) {
      const Canon* cn = nullptr;
      int rc = make_canon(c, g.second, count, &cn);
      if (rc) return rc;
      if (cn->n_slots >= (1ll << 31)) return fail(GPP_ERR_ARG, "too many work items");
      r->canon.push_back(cn);
      r->part_off.push_back(doubles);
      max_slots = std::max(max_slots, cn->n_slots);
      doubles += static_cast<size_t>(cn->n_slots) * (gpp::kThreads / 32) * 4 * g.second;
    }
    GPP_CUDA(c->partials.ensure(doubles));
    GPP_CUDA(c->cpartials.ensure(2 * r->groups.size()));
    const size_t g_max = static_cast<size_t>((max_slots + kSlotsPerFinalizeBlock - 1) /
                                             kSlotsPerFinalizeBlock);
    GPP_CUDA(c->stage.ensure(g_max * 4 * gpp::kMaxNwGroup));
    if (!c->ticket.ptr) {
      GPP_CUDA(c->ticket.ensure(1));
      GPP_CUDA(cudaMemsetAsync(c->ticket.ptr, 0, sizeof(unsigned), c->stream));
    }
    if (count)
      GPP_CUDA(cudaMemsetAsync(c->cpartials.ptr, 0,
                               2 * r->groups.size() * sizeof(unsigned long long), c->stream));
  }
  if (ev_main) GPP_CUDA(cudaEventRecord(ev_main[0], c->stream));
  if (r->sacc) {
    GPP_CUDA(cudaEventRecord(c->ev_fork, c->stream));
    GPP_CUDA(cudaStreamWaitEvent(c->kstream2, c->ev_fork, 0));
  }
  return GPP_OK;
}

int launch_sacc(gpp_ctx* c, const EvalRun& r, size_t gi, const SaccLaunch& L, const CanonLaunch& C,
                cudaStream_t s) {
  const int iw0 = r.groups[gi].first, nwg = r.groups[gi].second;
  const Canon& cn = *r.canon[gi];
  const KernelRef fn = pick_kernel(GPP_VARIANT_RCP_SQ, nwg, cn.pl.igp_t, r.count);
  gpp::Params p{};
  p.wtilde = c->wtilde.ptr;
  p.eps = c->eps.ptr;
  p.aqsn = c->aqsn.ptr;
  p.aqsm = c->aqsm.ptr;
  p.wxb = c->wxb.ptr;
  p.ncouls = static_cast<int>(c->ncouls);
  p.ngpown = static_cast<int>(c->ngpown);
  p.nbands = static_cast<int>(L.wnb);
  p.band0 = static_cast<int>(L.wb0);
  p.nw_total = c->nw;
  p.iw0 = iw0;
  p.igblk0 = 0;
  p.n_igblk = cn.pl.n_igblk;
  p.n_igptile = cn.pl.n_igptile;
  p.row0 = L.row0;
  p.n_rows = L.n_rows;
  gpp::fastdiv_init(static_cast<unsigned>(p.n_igptile), &p.igpt_mul, &p.igpt_shift);
  gpp::fastdiv_init(static_cast<unsigned>(p.n_rows), &p.rows_mul, &p.rows_shift);
  p.bchunk = L.bchunk;
  p.n_items = L.n_items;
  p.wxmax = c->wxmax;
  p.slot_base = C.slot0 - C.row0;
  p.slot_stride = C.n_rows;
  p.partials = c->partials.ptr + r.part_off[gi];
  p.cpartials = c->cpartials.ptr + 2 * gi;
  const long long slots = static_cast<long long>(cn.pl.blocks_per_sm) * c->num_sms;
  const int grid = static_cast<int>(std::min<long long>(slots, p.n_items));
  gpp::WxTable t;
  for (int64_t b = 0; b < L.wnb; ++b)
    for (int iw = 0; iw < nwg; ++iw) t.w[b * nwg + iw] = c->h_wx[(L.wb0 + b) * c->nw + iw0 + iw];
  fn.sacc<<<grid, gpp::kThreads, fn.smem, s>>>(p, t);
  ++c->launches;
  GPP_CUDA(cudaGetLastError());
  return GPP_OK;
}

int eval_rows(gpp_ctx* c, EvalRun* r, int blk0, int blk1, cudaEvent_t ready) {
  if (!r->sacc) {
    if (ready) r->pending.push_back(ready);
    return GPP_OK;
  }
  if (blk1 <= blk0) return GPP_OK;
  cudaStream_t ks = (r->piece & 1) ? c->kstream2 : c->stream;
  cudaStream_t other = ks == c->stream ? c->kstream2 : c->stream;
  ++r->piece;
  bool waited_ks = false, waited_other = false;
  for (size_t gi = 0; gi < r->groups.size(); ++gi) {
    const Canon& cn = *r->canon[gi];
    const int r0 = blk0 * cn.pl.n_igptile, r1 = blk1 * cn.pl.n_igptile;
    for (const CanonLaunch& C : cn.ls) {
      SaccLaunch L;
      if (!sub_launch(C, r0, r1, &L)) continue;
      cudaStream_t s = L.tail ? other : ks;
      bool& waited = L.tail ? waited_other : waited_ks;
      if (ready && !waited) {
        GPP_CUDA(cudaStreamWaitEvent(s, ready, 0));
        waited = true;
      }
      int rc = launch_sacc(c, *r, gi, L, C, s);
      if (rc) return rc;
    }
  }
  return GPP_OK;
}

// The as-written and ladder kernels: the whole problem per frequency group,
// one partial row per CTA, the single-block finalize.
int run_plain_group(gpp_ctx* c, const EvalRun& r, size_t gi, bool first) {
  const int iw0 = r.groups[gi].first, nwg = r.groups[gi].second;
  Plan pl;
  int rc = make_plan(c, r.variant, nwg, r.count, &pl);
  if (rc) return rc;
  const KernelRef fn = pick_kernel(r.variant, nwg, pl.igp_t, r.count);
  GPP_CUDA(c->partials.ensure(static_cast<size_t>(pl.grid) * 4 * gpp::kMaxNwGroup));
  GPP_CUDA(c->cpartials.ensure(static_cast<size_t>(pl.grid) * 2));
  gpp::Params p{};
  p.wtilde = c->wtilde.ptr;
  p.eps = c->eps.ptr;
  p.aqsn = c->aqsn.ptr;
  p.aqsm = c->aqsm.ptr;
  p.wxb = c->wxb.ptr;
  p.ncouls = static_cast<int>(c->ncouls);
  p.ngpown = static_cast<int>(c->ngpown);
  p.nbands = static_cast<int>(c->nbands);
  p.band0 = 0;
  p.nw_total = c->nw;
  p.iw0 = iw0;
  p.igblk0 = 0;
  p.n_igblk = pl.n_igblk;
  p.n_igptile = pl.n_igptile;
  p.row0 = 0;
  p.n_rows = pl.n_igblk * pl.n_igptile;
  p.bchunk = pl.bchunk;
  p.n_items = pl.n_items;
  p.wxmax = c->wxmax;
  p.partials = c->partials.ptr;
  p.cpartials = c->cpartials.ptr;
  fn.fn<<<pl.grid, gpp::kThreads, 0, c->stream>>>(p);
  ++c->launches;
  GPP_CUDA(cudaGetLastError());
  if (r.ev_main && gi + 1 == r.groups.size()) GPP_CUDA(cudaEventRecord(r.ev_main[1], c->stream));
  pick_finalize(nwg)<<<1, 256, 0, c->stream>>>(c->partials.ptr, c->cpartials.ptr, pl.grid, c->nw,
                                                iw0, r.variant >= GPP_VARIANT_RCP_SQ, first ? 1 : 0,
                                                r.count ? 1 : 0, c->out.ptr, c->counts.ptr);
  ++c->launches;
  GPP_CUDA(cudaGetLastError());
  return GPP_OK;
}

using SlotFinalizeFn = void (*)(const double*, long long, int, double*, unsigned*,
                                const unsigned long long*, int, int, int, int, int, double*,
                                unsigned long long*);
SlotFinalizeFn pick_slot_finalize(int nw) {
  switch (nw) {
    case 1: return gpp::gpp_slot_finalize_kernel<1>;
    case 2: return gpp::gpp_slot_finalize_kernel<2>;
    default: return gpp::gpp_slot_finalize_kernel<3>;
  }
}

int eval_end(gpp_ctx* c, EvalRun* r) {
  if (!r->sacc) {
    for (cudaEvent_t e : r->pending) GPP_CUDA(cudaStreamWaitEvent(c->stream, e, 0));
    for (size_t gi = 0; gi < r->groups.size(); ++gi) {
      int rc = run_plain_group(c, *r, gi, gi == 0);
      if (rc) return rc;
    }
    return GPP_OK;
  }
  GPP_CUDA(cudaEventRecord(c->ev_join, c->kstream2));
  GPP_CUDA(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  if (r->ev_main) GPP_CUDA(cudaEventRecord(r->ev_main[1], c->stream));
  for (size_t gi = 0; gi < r->groups.size(); ++gi) {
    const int iw0 = r->groups[gi].first, nwg = r->groups[gi].second;
    const long long n_slots = r->canon[gi]->n_slots;
    const int grid = static_cast<int>((n_slots + kSlotsPerFinalizeBlock - 1) / kSlotsPerFinalizeBlock);
    const double* part = c->partials.ptr + r->part_off[gi];
    pick_slot_finalize(nwg)<<<grid, 256, 0, c->stream>>>(
        part, n_slots, kSlotsPerFinalizeBlock, c->stage.ptr, c->ticket.ptr,
        c->cpartials.ptr + 2 * gi, 1, c->nw, iw0, gi == 0 ? 1 : 0, r->count ? 1 : 0, c->out.ptr,
        c->counts.ptr);
    ++c->launches;
    GPP_CUDA(cudaGetLastError());
  }
  return GPP_OK;
}

int allreduce_out(gpp_ctx* c) {
  if (!(c->comm && c->nranks > 1)) return GPP_OK;
  GPP_NCCL(ncclGroupStart());
  GPP_NCCL(ncclAllReduce(c->out.ptr, c->out.ptr, 4 * c->nw, ncclDouble, ncclSum, c->comm,
                         c->stream));
  GPP_NCCL(ncclAllReduce(c->counts.ptr, c->counts.ptr, 2, ncclUint64, ncclSum, c->comm,
                         c->stream));
  GPP_NCCL(ncclGroupEnd());
  return GPP_OK;
}

// Enqueue one full evaluation of the resident problem on c->stream.  If
// ev_main is non-null, the main kernels are bracketed by ev_main[0..1].
int enqueue_eval(gpp_ctx* c, int variant, bool count, cudaEvent_t* ev_main, bool allreduce) {
  if (c->nbands == 0) {  // empty shard: zeros, then the collective
    if (ev_main) GPP_CUDA(cudaEventRecord(ev_main[0], c->stream));
    GPP_CUDA(cudaMemsetAsync(c->out.ptr, 0, 4 * sizeof(double) * c->nw, c->stream));
    GPP_CUDA(cudaMemsetAsync(c->counts.ptr, 0, 2 * sizeof(unsigned long long), c->stream));
    if (ev_main) GPP_CUDA(cudaEventRecord(ev_main[1], c->stream));
    return allreduce ? allreduce_out(c) : GPP_OK;
  }
  EvalRun r;
  int rc = eval_begin(c, variant, count, ev_main, &r);
  if (rc) return rc;
  const int n_blk = static_cast<int>((c->ncouls + gpp::kThreads - 1) / gpp::kThreads);
  rc = eval_rows(c, &r, 0, n_blk, nullptr);
  if (rc) return rc;
  rc = eval_end(c, &r);
  if (rc) return rc;
  return allreduce ? allreduce_out(c) : GPP_OK;
}

int check_variant(int32_t variant) {
  if (variant < GPP_VARIANT_DIV || variant > GPP_KERNEL_ONE_SEED)
    return fail(GPP_ERR_ARG, "unknown variant " + std::to_string(variant) +
                                 " (expected 0=div, 1=rcp, 2=rcp_sq, 3..5 = ladder kernels)");
  return GPP_OK;
}

}  // namespace

namespace {
// After an error on a context with a communicator, abort the communicator
// (ncclCommAbort) so that no peer waits forever on a collective this rank
// will not join; later calls on the context fail with GPP_ERR_NCCL.
int comm_guard(gpp_ctx* c, int rc) {
  if (rc == GPP_OK || !c || !c->comm) return rc;
  CtxLock lock(c);
  if (c->comm) {
    DeviceGuard g(c->device);
    ncclCommAbort(c->comm);
    c->comm = nullptr;
    c->comm_aborted = true;
  }
  return rc;
}

int comm_alive(const gpp_ctx* c) {
  if (c && c->comm_aborted)
    return fail(GPP_ERR_NCCL, "the communicator was aborted after an earlier error");
  return GPP_OK;
}

}  // namespace

extern "C" {

int gpp_abi_version(void) { return GPP_ABI_VERSION; }

const char* gpp_last_error(void) { return g_last_error.c_str(); }

int gpp_device_count(int* count) {
  if (!count) return fail(GPP_ERR_ARG, "count is NULL");
  *count = 0;
  GPP_CUDA(cudaGetDeviceCount(count));
  return GPP_OK;
}

int gpp_create(gpp_ctx** ctx, int device) {
  if (!ctx) return fail(GPP_ERR_ARG, "ctx is NULL");
  *ctx = nullptr;
  if (device < 0) return fail(GPP_ERR_ARG, "device must be >= 0");
  gpp_ctx* c = new (std::nothrow) gpp_ctx();
  if (!c) return fail(GPP_ERR_OOM, "host allocation failed");
  c->device = device;
  *ctx = c;
  return GPP_OK;
}

void gpp_destroy(gpp_ctx* c) {
  if (!c) return;
  if (c->initialized) {
    DeviceGuard g(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->cstream) cudaStreamSynchronize(c->cstream);
    if (c->kstream2) cudaStreamSynchronize(c->kstream2);
    if (c->nstream) cudaStreamSynchronize(c->nstream);
    if (c->comm) ncclCommDestroy(c->comm);
    c->wtilde.release();
    c->eps.release();
    c->aqsn.release();
    c->aqsm.release();
    c->wxb.release();
    c->partials.release();
    c->cpartials.release();
    c->out.release();
    c->counts.release();
    c->stage.release();
    c->ticket.release();
    if (c->h_out) cudaFreeHost(c->h_out);
    if (c->h_counts) cudaFreeHost(c->h_counts);
    if (c->h_wx) cudaFreeHost(c->h_wx);
    for (int k = 0; k < gpp_ctx::kStageSlots; ++k) {
      if (c->h_stage[k]) cudaFreeHost(c->h_stage[k]);
      if (c->stage_ev[k]) cudaEventDestroy(c->stage_ev[k]);
    }
    for (auto& ev : c->ev)
      if (ev) cudaEventDestroy(ev);
    for (auto& ev : c->slab_ev) cudaEventDestroy(ev);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->kstream2) cudaStreamDestroy(c->kstream2);
    if (c->nstream) cudaStreamDestroy(c->nstream);
    if (c->ev_we) cudaEventDestroy(c->ev_we);
    if (c->cstream) cudaStreamDestroy(c->cstream);
    if (c->stream) cudaStreamDestroy(c->stream);
  }
  delete c;
}

}  // extern "C"

namespace {

struct HostProblem {
  int64_t nbands, ngpown, ncouls;
  int32_t nw;
  const double *wtilde, *i_eps, *aqsntemp, *aqsmtemp, *wx;
  int32_t wx_band_indexed;
  int64_t band0, band1;
};

int validate(const gpp_ctx* c, const HostProblem& h) {
  if (!c) return fail(GPP_ERR_ARG, "ctx is NULL");
  if (h.nbands < 1 || h.ngpown < 1 || h.ncouls < 1)
    return fail(GPP_ERR_ARG, "nbands, ngpown and ncouls must all be at least 1");
  if (h.nw < 1) return fail(GPP_ERR_ARG, "nw must be at least 1");
  if (!h.wtilde || !h.i_eps || !h.aqsntemp || !h.aqsmtemp || !h.wx)
    return fail(GPP_ERR_ARG, "input array pointer is NULL");
  // An empty shard (band0 == band1) is allowed: a rank with no bands (more
  // ranks than bands) contributes zeros but still joins the collectives.
  if (h.band0 < 0 || h.band1 > h.nbands || h.band0 > h.band1)
    return fail(GPP_ERR_ARG, "band range [" + std::to_string(h.band0) + ", " +
                                 std::to_string(h.band1) + ") is reversed or outside [0, " +
                                 std::to_string(h.nbands) + "]");
  const int64_t kIntMax = 0x7fffffff;
  if (h.ncouls > kIntMax || h.ngpown > kIntMax || h.nbands > kIntMax ||
      (h.ncouls + gpp::kThreads) * (h.ngpown + gpp::kMaxIgpTile) > (int64_t{1} << 40))
    return fail(GPP_ERR_ARG, "problem dimensions exceed the supported range");
  return GPP_OK;
}

// Size the device buffers and the pinned staging for a problem shard, and
// expand wx to the band-indexed layout on the host (pinned).  No copies yet.
int prepare(gpp_ctx* c, const HostProblem& h) {
  const int64_t nb = h.band1 - h.band0;
  const size_t n_wt = static_cast<size_t>(h.ncouls) * h.ngpown;
  const size_t n_an = static_cast<size_t>(h.ncouls) * nb;
  const size_t n_am = static_cast<size_t>(h.ngpown) * nb;
  const size_t n_wx = static_cast<size_t>(nb) * h.nw;
  GPP_CUDA(c->wtilde.ensure(n_wt));
  GPP_CUDA(c->eps.ensure(n_wt));
  GPP_CUDA(c->aqsn.ensure(n_an));
  GPP_CUDA(c->aqsm.ensure(n_am));
  GPP_CUDA(c->wxb.ensure(n_wx));
  GPP_CUDA(c->out.ensure(4 * static_cast<size_t>(h.nw)));
  GPP_CUDA(c->counts.ensure(2));
  if (c->h_out_cap < 4 * static_cast<size_t>(h.nw)) {
    if (c->h_out) cudaFreeHost(c->h_out);
    c->h_out = nullptr;
    c->h_out_cap = 0;
    GPP_CUDA(cudaMallocHost(&c->h_out, 4 * sizeof(double) * h.nw));
    c->h_out_cap = 4 * static_cast<size_t>(h.nw);
  }
  if (!c->h_counts) GPP_CUDA(cudaMallocHost(&c->h_counts, 2 * sizeof(unsigned long long)));
  if (c->h_wx_cap < n_wx) {
    if (c->h_wx) cudaFreeHost(c->h_wx);
    c->h_wx = nullptr;
    c->h_wx_cap = 0;
    GPP_CUDA(cudaMallocHost(&c->h_wx, n_wx * sizeof(double)));
    c->h_wx_cap = n_wx;
  }
  // The device stream must be done with the staging before it is rewritten.
  GPP_CUDA(cudaStreamSynchronize(c->cstream));
  if (h.wx_band_indexed) {
    std::memcpy(c->h_wx, h.wx + static_cast<size_t>(h.band0) * h.nw, n_wx * sizeof(double));
  } else {
    for (int64_t b = 0; b < nb; ++b)
      std::memcpy(c->h_wx + static_cast<size_t>(b) * h.nw, h.wx, h.nw * sizeof(double));
  }
  double wxmax = 0.0;
  for (size_t k = 0; k < n_wx; ++k) wxmax = std::max(wxmax, std::fabs(c->h_wx[k]));
  bool invariant = true;
  for (size_t k = static_cast<size_t>(h.nw); k < n_wx && invariant; ++k)
    invariant = c->h_wx[k] == c->h_wx[k % h.nw];
  c->wx_band_invariant = invariant;
  c->plan_cache.clear();
  c->canon_cache.clear();
  c->nbands = nb;
  c->ngpown = h.ngpown;
  c->ncouls = h.ncouls;
  c->nw = h.nw;
  c->wxmax = wxmax;
  return GPP_OK;
}

// H2D of the expanded wx (pinned staging) on stream s.
int copy_small_wx(gpp_ctx* c, const HostProblem& h, cudaStream_t s) {
  const int64_t nb = h.band1 - h.band0;
  GPP_CUDA(cudaMemcpyAsync(c->wxb.ptr, c->h_wx, static_cast<size_t>(nb) * h.nw * sizeof(double),
                           cudaMemcpyHostToDevice, s));
  return GPP_OK;
}

// H2D of the small arrays (aqsmtemp shard, expanded wx) on stream s.
int copy_small(gpp_ctx* c, const HostProblem& h, cudaStream_t s) {
  const int64_t nb = h.band1 - h.band0;
  GPP_CUDA(cudaMemcpyAsync(c->aqsm.ptr, h.aqsmtemp + 2 * static_cast<size_t>(h.band0) * h.ngpown,
                           static_cast<size_t>(h.ngpown) * nb * sizeof(double2),
                           cudaMemcpyHostToDevice, s));
  return copy_small_wx(c, h, s);
}

// Whether a host range is page-locked (cudaHostRegister / cudaMallocHost):
// the DMA engines then read it directly.
bool host_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Host threads that pack pageable inputs into the staging ring:
// GPP_HOST_THREADS, else half the cores of this process's share of the node
// (LOCAL_WORLD_SIZE ranks per node under torchrun), at most 8 -- the copy
// saturates PCIe with ~8 (tools/probe_pageable.py: 6.65 ms upload with 8,
// 6.82 with 16, 8.7 with 4 on a 16-core host), and spinning packers must
// not starve the thread that issues the copies and kernels.
int host_threads() {
  static const int n = [] {
    if (const char* e = std::getenv("GPP_HOST_THREADS")) return std::max(1, std::atoi(e));
    int local = 1;
    if (const char* e = std::getenv("LOCAL_WORLD_SIZE")) local = std::max(1, std::atoi(e));
    const int hw = std::max(1, omp_get_num_procs());
    return std::max(1, std::min(8, hw / local / 2));
  }();
  return n;
}

// One staging buffer: 8 MB (GPP_STAGE_MB overrides, for experiments).
size_t stage_bytes() {
  static const size_t n = [] {
    const char* e = std::getenv("GPP_STAGE_MB");
    const long mb = e ? std::max(1L, std::atol(e)) : 8L;
    return static_cast<size_t>(mb) << 20;
  }();
  return n;
}

// Staging buffers in the ring: 4 (GPP_STAGE_SLOTS overrides, <= 16).
int stage_slots() {
  static const int n = [] {
    const char* e = std::getenv("GPP_STAGE_SLOTS");
    return e ? std::max(2, std::min(gpp_ctx::kStageSlots, std::atoi(e))) : 4;
  }();
  return n;
}

int ensure_stage(gpp_ctx* c) {
  if (c->stage_cap >= stage_bytes()) return GPP_OK;
  for (int k = 0; k < stage_slots(); ++k) {
    if (c->h_stage[k]) {
      if (c->stage_ev[k]) GPP_CUDA(cudaEventSynchronize(c->stage_ev[k]));
      cudaFreeHost(c->h_stage[k]);
      c->h_stage[k] = nullptr;
    }
    GPP_CUDA(cudaMallocHost(&c->h_stage[k], stage_bytes()));
    if (!c->stage_ev[k]) GPP_CUDA(cudaEventCreateWithFlags(&c->stage_ev[k], cudaEventDisableTiming));
  }
  c->stage_cap = stage_bytes();
  return GPP_OK;
}

// H2D of rows [i0, i1) of `ncol` columns (column pitch `ld` elements) of a
// complex F-order host array into the device array of the same layout.
// Pinned source: one strided copy.  Pageable source: columns are packed by
// host_threads() threads into the next pinned staging buffer (waiting until
// its previous copy has drained) and copied from there, buffer by buffer, so
// the packing of one buffer overlaps the DMA of the previous ones.
int copy_cols(gpp_ctx* c, double2* dst, const double* src, int64_t ld, int64_t ncol, int64_t i0,
              int64_t i1, bool pinned, cudaStream_t s) {
  const size_t pitch = static_cast<size_t>(ld) * sizeof(double2);
  const size_t width = static_cast<size_t>(i1 - i0) * sizeof(double2);
  if (ncol <= 0 || width == 0) return GPP_OK;
  if (pinned) {
    GPP_CUDA(cudaMemcpy2DAsync(dst + i0, pitch, src + 2 * i0, pitch, width, ncol,
                               cudaMemcpyHostToDevice, s));
    return GPP_OK;
  }
  int rc = ensure_stage(c);
  if (rc) return rc;
  const int64_t per = std::max<int64_t>(1, static_cast<int64_t>(c->stage_cap / width));
  const int nt = host_threads();
  for (int64_t c0 = 0; c0 < ncol; c0 += per) {
    const int64_t c1 = std::min(ncol, c0 + per);
    const int k = c->stage_next;
    c->stage_next = (k + 1) % stage_slots();
    GPP_CUDA(cudaEventSynchronize(c->stage_ev[k]));  // its previous copy has drained
    unsigned char* buf = c->h_stage[k];
    const size_t wbytes = width;
    const int64_t ncols = c1 - c0;
    if (ncols * static_cast<int64_t>(wbytes) >= (int64_t{1} << 20) && nt > 1) {
#pragma omp parallel for num_threads(nt) schedule(static)
      for (int64_t j = 0; j < ncols; ++j)
        std::memcpy(buf + j * wbytes, src + 2 * ((c0 + j) * ld + i0), wbytes);
    } else {
      for (int64_t j = 0; j < ncols; ++j)
        std::memcpy(buf + j * wbytes, src + 2 * ((c0 + j) * ld + i0), wbytes);
    }
    GPP_CUDA(cudaMemcpy2DAsync(dst + c0 * ld + i0, pitch, buf, wbytes, wbytes, ncols,
                               cudaMemcpyHostToDevice, s));
    GPP_CUDA(cudaEventRecord(c->stage_ev[k], s));
    c->staged_bytes += static_cast<uint64_t>(ncols) * wbytes;
  }
  return GPP_OK;
}

// Pinned-ness of the three row-copied inputs (checked once per call).
struct HostPins {
  bool wtilde = false, eps = false, aqsn = false;
};
HostPins host_pins(const HostProblem& h) {
  HostPins p;
  p.wtilde = host_pinned(h.wtilde);
  p.eps = host_pinned(h.i_eps);
  p.aqsn = host_pinned(h.aqsntemp);
  return p;
}

// H2D of the ig rows [i0, i1) of wtilde and i_eps (unless !with_we) and of
// the aqsntemp shard.
int copy_rows(gpp_ctx* c, const HostProblem& h, const HostPins& pins, int64_t i0, int64_t i1,
              cudaStream_t s, bool with_we = true) {
  int rc = GPP_OK;
  if (with_we) {
    rc = copy_cols(c, c->wtilde.ptr, h.wtilde, h.ncouls, h.ngpown, i0, i1, pins.wtilde, s);
    if (!rc) rc = copy_cols(c, c->eps.ptr, h.i_eps, h.ncouls, h.ngpown, i0, i1, pins.eps, s);
  }
  if (!rc)
    rc = copy_cols(c, c->aqsn.ptr, h.aqsntemp + 2 * static_cast<size_t>(h.band0) * h.ncouls,
                   h.ncouls, h.band1 - h.band0, i0, i1, pins.aqsn, s);
  return rc;
}

// Column-split upload of the replicated wtilde / i_eps (band sharding over
// ranks): rank r copies only its igp columns [g0_r, g1_r) over
// its own PCIe link (whole columns: contiguous in F-order), then every rank
// broadcasts its columns to the others over NVLink (one grouped set of
// ncclBroadcast, in place, on nstream).  c->ev_we marks wtilde / eps complete
// on the device.  Per rank the H2D drops from 2 nc ng to 2 nc ng / N complex
// values.  With one rank (GPP_COLUMN_UPLOAD=1, tests) it is a plain copy.
bool column_split(const gpp_ctx* c) {
  static const bool force = [] {
    const char* e = std::getenv("GPP_COLUMN_UPLOAD");
    return e && e[0] == '1';
  }();
  return (c->comm && c->nranks > 1) || force || std::getenv("GPP_COLUMN_SIM") != nullptr;
}

// GPP_COLUMN_SIM=N (timing projection only, tools/probe_shard_e2e.py): on a
// single rank, upload just rank 0's 1/N of the columns and skip the
// broadcasts -- the H2D and compute of one rank of N; the result is wrong.
int column_sim() {
  static const int n = [] {
    const char* e = std::getenv("GPP_COLUMN_SIM");
    return e ? std::max(1, std::atoi(e)) : 1;
  }();
  return n;
}

int upload_we_split(gpp_ctx* c, const HostProblem& h, const HostPins& pins) {
  const bool real = c->comm && c->nranks > 1;
  const int n = real ? c->nranks : column_sim(), me = real ? c->rank : 0;
  auto g0 = [&](int r) { return h.ngpown * r / n; };
  const int64_t a = g0(me), b = g0(me + 1), nc = h.ncouls;
  int rc = copy_cols(c, c->wtilde.ptr + a * nc, h.wtilde + 2 * a * nc, nc, b - a, 0, nc,
                     pins.wtilde, c->cstream);
  if (!rc)
    rc = copy_cols(c, c->eps.ptr + a * nc, h.i_eps + 2 * a * nc, nc, b - a, 0, nc, pins.eps,
                   c->cstream);
  if (rc) return rc;
  GPP_CUDA(cudaEventRecord(c->ev_we, c->cstream));
  if (real) {
    GPP_CUDA(cudaStreamWaitEvent(c->nstream, c->ev_we, 0));
    GPP_NCCL(ncclGroupStart());
    for (int r = 0; r < n; ++r) {
      const size_t off = static_cast<size_t>(g0(r)) * nc;
      const size_t cnt = static_cast<size_t>(g0(r + 1) - g0(r)) * nc * 2;
      if (cnt == 0) continue;
      GPP_NCCL(ncclBroadcast(c->wtilde.ptr + off, c->wtilde.ptr + off, cnt, ncclDouble, r, c->comm,
                             c->nstream));
      GPP_NCCL(ncclBroadcast(c->eps.ptr + off, c->eps.ptr + off, cnt, ncclDouble, r, c->comm,
                             c->nstream));
    }
    GPP_NCCL(ncclGroupEnd());
    GPP_CUDA(cudaEventRecord(c->ev_we, c->nstream));
  }
  return GPP_OK;
}

// ig-slab schedule of the pipelined evaluate, as block offsets.  The copy is
// the critical path (PCIe ~55 GB/s against the kernel's ~0.65 of that time);
// slab s's items run while slab s+1 is in flight, and what follows the last
// byte is the last slab's items.  The production kernel runs canonical items
// (whole rows of up to 512 bands, the balanced tail's last rows in short
// chunks), so the default is slabs of about one wave of rows (resident CTAs /
// igp tiles blocks) and a last slab of the blocks whose rows are all
// balanced-tail rows (short items: little work after the last byte).
// slabs > 0: that many equal slabs.  GPP_SLABS="b0,b1,..." (block counts
// summing to the block total) overrides, for experiments.
std::vector<int> slab_schedule(gpp_ctx* c, const EvalRun& r, int n_blk, int slabs, bool pageable) {
  std::vector<int> sizes;
  if (const char* e = std::getenv("GPP_SLABS")) {
    int sum = 0;
    for (const char* q = e; *q;) {
      char* end = nullptr;
      const long v = std::strtol(q, &end, 10);
      if (end == q || v <= 0) break;
      sizes.push_back(static_cast<int>(v));
      sum += static_cast<int>(v);
      q = *end == ',' ? end + 1 : end;
    }
    if (sum != n_blk) sizes.clear();
  }
  if (sizes.empty() && slabs > 0) {
    const int n = std::min(slabs, n_blk);
    for (int i = 0; i < n; ++i)
      sizes.push_back(static_cast<int>(static_cast<int64_t>(n_blk) * (i + 1) / n -
                                       static_cast<int64_t>(n_blk) * i / n));
  }
  if (sizes.empty()) {
    int per = 8, tail_blocks = 0;
    if (r.sacc && !r.canon.empty()) {
      const Canon& cn = *r.canon[0];
      const long long slots = static_cast<long long>(cn.pl.blocks_per_sm) * c->num_sms;
      per = static_cast<int>(std::max<long long>(1, slots / cn.pl.n_igptile));
      int first_tail_row = cn.n_rows;
      for (const CanonLaunch& L : cn.ls)
        if (L.tail) first_tail_row = std::min(first_tail_row, L.row0);
      tail_blocks = cn.n_rows - ((first_tail_row + cn.pl.n_igptile - 1) / cn.pl.n_igptile) *
                                    cn.pl.n_igptile;
      tail_blocks = std::max(0, tail_blocks / cn.pl.n_igptile);
    }
    // Built from the end: a last slab of max(2, tail) blocks, then slabs of
    // 1, 2, 3, ... waves of rows (resident CTAs / igp tiles blocks), the
    // first slab taking the remainder: every slab's items keep pace with the
    // copy of the next one, and little work follows the last byte
    // (tools/probe_slabs4.py: 6.66 ms pinned / 7.23 ms pageable at the paper
    // size against 6.74-6.90 / 8.2-8.7 for equal slabs of 1-2 waves).
    std::vector<int> rev;
    int sum = 0, k = 1;
    const int last = std::min(n_blk, std::max(2, tail_blocks));
    rev.push_back(last);
    sum = last;
    while (sum < n_blk) {
      const int take = std::min(k * per, n_blk - sum);
      rev.push_back(take);
      sum += take;
      ++k;
    }
    (void)pageable;
    sizes.assign(rev.rbegin(), rev.rend());
  }
  std::vector<int> blk0{0};
  for (int v : sizes) blk0.push_back(blk0.back() + v);
  return blk0;
}

// Wait for stream s.  With a communicator attached, poll instead of
// blocking, so that a failed or aborted peer (ncclCommGetAsyncError) or a
// stuck collective (GPP_NCCL_TIMEOUT_S, default 600 s) surfaces as
// GPP_ERR_NCCL instead of a hang; the caller's guard then aborts the comm.
int wait_stream(gpp_ctx* c, cudaStream_t s) {
  if (!(c->comm && c->nranks > 1)) {
    GPP_CUDA(cudaStreamSynchronize(s));
    return GPP_OK;
  }
  static const double timeout_s = [] {
    const char* e = std::getenv("GPP_NCCL_TIMEOUT_S");
    return e ? std::max(1.0, std::atof(e)) : 600.0;
  }();
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e == cudaSuccess) return GPP_OK;
    if (e != cudaErrorNotReady) return cuda_fail(e, "cudaStreamQuery");
    ncclResult_t st = ncclSuccess;
    GPP_NCCL(ncclCommGetAsyncError(c->comm, &st));
    if (st != ncclSuccess && st != ncclInProgress)
      return fail(GPP_ERR_NCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(st));
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s)
      return fail(GPP_ERR_NCCL, "collective did not complete within GPP_NCCL_TIMEOUT_S");
    std::this_thread::sleep_for(std::chrono::microseconds(10));
  }
}

int finish_run(gpp_ctx* c, double* achtemp, double* asxtemp, int64_t* near_far) {
  int rc = allreduce_out(c);
  if (rc) return rc;
  GPP_CUDA(cudaMemcpyAsync(c->h_out, c->out.ptr, 4 * sizeof(double) * c->nw,
                           cudaMemcpyDeviceToHost, c->stream));
  GPP_CUDA(cudaMemcpyAsync(c->h_counts, c->counts.ptr, 2 * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, c->stream));
  rc = wait_stream(c, c->stream);
  if (rc) return rc;
  std::memcpy(achtemp, c->h_out, 2 * sizeof(double) * c->nw);
  std::memcpy(asxtemp, c->h_out + 2 * c->nw, 2 * sizeof(double) * c->nw);
  if (near_far) {
    near_far[0] = static_cast<int64_t>(c->h_counts[0]);
    near_far[1] = static_cast<int64_t>(c->h_counts[1]);
  }
  return GPP_OK;
}

}  // namespace

extern "C" {

static int gpp_upload_impl(gpp_ctx* c, int64_t nbands, int64_t ngpown, int64_t ncouls, int32_t nw,
               const double* wtilde, const double* i_eps, const double* aqsntemp,
               const double* aqsmtemp, const double* wx, int32_t wx_band_indexed,
               int64_t band0, int64_t band1) {
  CtxLock lock(c);
  const HostProblem h{nbands, ngpown, ncouls, nw, wtilde, i_eps, aqsntemp, aqsmtemp, wx,
                      wx_band_indexed, band0, band1};
  int rc = validate(c, h);
  if (rc) return rc;
  rc = ensure_init(c);
  if (rc) return rc;
  DeviceGuard g(c->device);
  if (!g.ok) return cuda_fail(g.err, "cudaSetDevice");
  c->have_problem = false;
  rc = prepare(c, h);
  if (rc) return rc;
  cudaStream_t s = c->stream;
  rc = copy_small(c, h, s);
  if (rc) return rc;
  rc = copy_rows(c, h, host_pins(h), 0, ncouls, s);
  if (rc) return rc;
  GPP_CUDA(cudaStreamSynchronize(s));
  c->have_problem = true;
  return GPP_OK;
}

static int gpp_evaluate_host_impl(gpp_ctx* c, int32_t variant, int64_t nbands, int64_t ngpown, int64_t ncouls,
                      int32_t nw, const double* wtilde, const double* i_eps,
                      const double* aqsntemp, const double* aqsmtemp, const double* wx,
                      int32_t wx_band_indexed, int64_t band0, int64_t band1, int32_t slabs,
                      double* achtemp, double* asxtemp, int64_t* near_far, float* ms) {
  CtxLock lock(c);
  const HostProblem h{nbands, ngpown, ncouls, nw, wtilde, i_eps, aqsntemp, aqsmtemp, wx,
                      wx_band_indexed, band0, band1};
  int rc = validate(c, h);
  if (rc) return rc;
  rc = check_variant(variant);
  if (rc) return rc;
  if (!achtemp || !asxtemp) return fail(GPP_ERR_ARG, "output pointer is NULL");
  rc = ensure_init(c);
  if (rc) return rc;
  DeviceGuard g(c->device);
  if (!g.ok) return cuda_fail(g.err, "cudaSetDevice");
  c->have_problem = false;
  rc = prepare(c, h);
  if (rc) return rc;
  // ig slabs on 256-ig block boundaries; the canonical items of slab s run as
  // soon as its rows have landed, while slab s+1 is in flight.
  const int n_blk = static_cast<int>((ncouls + gpp::kThreads - 1) / gpp::kThreads);
  const HostPins pins = host_pins(h);
  const bool split = column_split(c);
  GPP_CUDA(cudaEventRecord(c->ev[2], c->cstream));
  rc = copy_small(c, h, c->cstream);
  if (rc) return rc;
  if (split) {
    rc = upload_we_split(c, h, pins);
    if (rc) return rc;
  }
  if (c->nbands == 0) {  // empty shard: no rows to copy, zeros into the collective
    GPP_CUDA(cudaStreamWaitEvent(c->stream, split ? c->ev_we : c->ev[2], 0));
    rc = enqueue_eval(c, variant, near_far != nullptr, nullptr, false);
    if (rc) return rc;
  } else {
    EvalRun r;
    rc = eval_begin(c, variant, near_far != nullptr, nullptr, &r);
    if (rc) return rc;
    if (split) {
      GPP_CUDA(cudaStreamWaitEvent(c->stream, c->ev_we, 0));
      GPP_CUDA(cudaStreamWaitEvent(c->kstream2, c->ev_we, 0));
    }
    const std::vector<int> blk0 = slab_schedule(
        c, r, n_blk, slabs, !(pins.aqsn && (split || (pins.wtilde && pins.eps))));
    const int n_sched = static_cast<int>(blk0.size()) - 1;
    while (static_cast<int>(c->slab_ev.size()) < n_sched + 1) {
      cudaEvent_t e;
      GPP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->slab_ev.push_back(e);
    }
    for (int sl = 0; sl < n_sched; ++sl) {
      const int64_t i0 = static_cast<int64_t>(blk0[sl]) * gpp::kThreads;
      const int64_t i1 =
          std::min<int64_t>(ncouls, static_cast<int64_t>(blk0[sl + 1]) * gpp::kThreads);
      rc = copy_rows(c, h, pins, i0, i1, c->cstream, !split);
      if (rc) return rc;
      GPP_CUDA(cudaEventRecord(c->slab_ev[sl], c->cstream));
      rc = eval_rows(c, &r, blk0[sl], blk0[sl + 1], c->slab_ev[sl]);
      if (rc) return rc;
    }
    rc = eval_end(c, &r);
    if (rc) return rc;
  }
  GPP_CUDA(cudaEventRecord(c->ev[3], c->stream));
  rc = finish_run(c, achtemp, asxtemp, near_far);
  if (rc) return rc;
  c->have_problem = true;
  if (ms) GPP_CUDA(cudaEventElapsedTime(ms, c->ev[2], c->ev[3]));
  return GPP_OK;
}

static int gpp_run_impl(gpp_ctx* c, int32_t variant, double* achtemp, double* asxtemp, int64_t* near_far,
            float* kernel_ms) {
  CtxLock lock(c);
  if (!c) return fail(GPP_ERR_ARG, "ctx is NULL");
  int rc = check_variant(variant);
  if (rc) return rc;
  if (!achtemp || !asxtemp) return fail(GPP_ERR_ARG, "output pointer is NULL");
  if (!c->have_problem) return fail(GPP_ERR_ARG, "no problem uploaded");
  DeviceGuard g(c->device);
  if (!g.ok) return cuda_fail(g.err, "cudaSetDevice");
  GPP_CUDA(cudaEventRecord(c->ev[2], c->stream));
  rc = enqueue_eval(c, variant, near_far != nullptr, nullptr, false);
  if (rc) return rc;
  GPP_CUDA(cudaEventRecord(c->ev[3], c->stream));
  rc = finish_run(c, achtemp, asxtemp, near_far);
  if (rc) return rc;
  if (kernel_ms) GPP_CUDA(cudaEventElapsedTime(kernel_ms, c->ev[2], c->ev[3]));
  return GPP_OK;
}

static int gpp_time_impl(gpp_ctx* c, int32_t variant, int32_t iters, float* total_ms, float* main_ms) {
  CtxLock lock(c);
  if (!c) return fail(GPP_ERR_ARG, "ctx is NULL");
  int rc = check_variant(variant);
  if (rc) return rc;
  if (iters < 1) return fail(GPP_ERR_ARG, "iters must be at least 1");
  if (!c->have_problem) return fail(GPP_ERR_ARG, "no problem uploaded");
  DeviceGuard g(c->device);
  if (!g.ok) return cuda_fail(g.err, "cudaSetDevice");
  std::vector<cudaEvent_t> evs(2 * static_cast<size_t>(iters));
  for (auto& e : evs) GPP_CUDA(cudaEventCreate(&e));
  int result = GPP_OK;
  do {
    cudaError_t e = cudaEventRecord(c->ev[2], c->stream);
    if (e != cudaSuccess) { result = cuda_fail(e, "cudaEventRecord"); break; }
    for (int i = 0; i < iters && result == GPP_OK; ++i)
      result = enqueue_eval(c, variant, false, &evs[2 * static_cast<size_t>(i)], true);
    if (result) break;
    e = cudaEventRecord(c->ev[3], c->stream);
    if (e != cudaSuccess) { result = cuda_fail(e, "gpp_time record"); break; }
    result = wait_stream(c, c->stream);  // polls the communicator's health
    if (result) break;
    float tot = 0.f, mm = 0.f;
    cudaEventElapsedTime(&tot, c->ev[2], c->ev[3]);
    for (int i = 0; i < iters; ++i) {
      float x = 0.f;
      cudaEventElapsedTime(&x, evs[2 * i], evs[2 * i + 1]);
      mm += x;
    }
    if (total_ms) *total_ms = tot;
    if (main_ms) *main_ms = mm;
  } while (0);
  for (auto& e : evs) cudaEventDestroy(e);
  return result;
}

int gpp_plan(int64_t nbands, int64_t ngpown, int64_t ncouls, int32_t nw, int32_t sms,
             int32_t max_launches, int32_t* n_launches, int64_t* launches) {
  if (nbands < 1 || ngpown < 1 || ncouls < 1 || nw < 1 || sms < 1 || !n_launches ||
      (max_launches > 0 && !launches))
    return fail(GPP_ERR_ARG, "gpp_plan: bad argument");
  const int nwg = std::min<int>(nw, max_group(GPP_VARIANT_RCP_SQ));
  const int igp_t = sacc_igp(nwg, ngpown);
  const long long slots = static_cast<long long>(sms) * sacc_blocks_per_sm(nwg, igp_t);
  const int n_igblk = static_cast<int>((ncouls + gpp::kThreads - 1) / gpp::kThreads);
  const int n_igptile = static_cast<int>((ngpown + igp_t - 1) / igp_t);
  const int plan_bchunk = choose_bchunk(n_igblk, n_igptile, nbands, slots, sacc_cap(nwg),
                                       balanced_tail_enabled());
  long long n_slots = 0;
  const std::vector<CanonLaunch> all =
      canon_launches(n_igblk, n_igptile, nbands, nwg, plan_bchunk, slots, &n_slots);
  *n_launches = static_cast<int32_t>(all.size());
  for (int32_t k = 0; k < std::min<int32_t>(max_launches, *n_launches); ++k) {
    const CanonLaunch& L = all[k];
    int64_t* o = launches + 7 * k;
    o[0] = L.row0;
    o[1] = L.n_rows;
    o[2] = L.wb0;
    o[3] = L.wnb;
    o[4] = L.bchunk;
    o[5] = L.n_items;
    o[6] = igp_t;
  }
  return GPP_OK;
}

int gpp_plan_piece(int64_t nbands, int64_t ngpown, int64_t ncouls, int32_t nw, int32_t sms,
                   int32_t blk0, int32_t blk1, int32_t max_launches, int32_t* n_launches,
                   int64_t* launches) {
  if (nbands < 1 || ngpown < 1 || ncouls < 1 || nw < 1 || sms < 1 || !n_launches ||
      (max_launches > 0 && !launches) || blk0 < 0 || blk1 < blk0)
    return fail(GPP_ERR_ARG, "gpp_plan_piece: bad argument");
  const int nwg = std::min<int>(nw, max_group(GPP_VARIANT_RCP_SQ));
  const int igp_t = sacc_igp(nwg, ngpown);
  const long long slots = static_cast<long long>(sms) * sacc_blocks_per_sm(nwg, igp_t);
  const int n_igblk = static_cast<int>((ncouls + gpp::kThreads - 1) / gpp::kThreads);
  const int n_igptile = static_cast<int>((ngpown + igp_t - 1) / igp_t);
  const int plan_bchunk = choose_bchunk(n_igblk, n_igptile, nbands, slots, sacc_cap(nwg),
                                       balanced_tail_enabled());
  long long n_slots = 0;
  const std::vector<CanonLaunch> all =
      canon_launches(n_igblk, n_igptile, nbands, nwg, plan_bchunk, slots, &n_slots);
  const int r0 = std::min(blk0, n_igblk) * n_igptile, r1 = std::min(blk1, n_igblk) * n_igptile;
  int32_t n = 0;
  for (const CanonLaunch& C : all) {
    SaccLaunch L;
    if (!sub_launch(C, r0, r1, &L)) continue;
    if (n < max_launches) {
      int64_t* o = launches + 9 * n;
      o[0] = L.row0;
      o[1] = L.n_rows;
      o[2] = L.wb0;
      o[3] = L.wnb;
      o[4] = L.bchunk;
      o[5] = L.n_items;
      o[6] = igp_t;
      o[7] = C.slot0 - C.row0;  // slot_base
      o[8] = C.n_rows;          // slot_stride
    }
    ++n;
  }
  *n_launches = n;
  return GPP_OK;
}

int gpp_launch_count(gpp_ctx* c, int64_t* launches) {
  CtxLock lock(c);
  if (!c || !launches) return fail(GPP_ERR_ARG, "ctx / launches is NULL");
  *launches = static_cast<int64_t>(c->launches);
  return GPP_OK;
}

int gpp_kernel_info(gpp_ctx* c, int32_t variant, int32_t* registers_per_thread,
                    int32_t* threads_per_block, int32_t* blocks_per_sm, int32_t* grid,
                    int32_t* igp_tile, int32_t* band_chunk) {
  CtxLock lock(c);
  if (!c) return fail(GPP_ERR_ARG, "ctx is NULL");
  int rc = check_variant(variant);
  if (rc) return rc;
  if (!c->have_problem) return fail(GPP_ERR_ARG, "no problem uploaded");
  DeviceGuard g(c->device);
  if (!g.ok) return cuda_fail(g.err, "cudaSetDevice");
  Plan pl;
  rc = make_plan(c, variant, std::min(c->nw, max_group(variant)), false, &pl);
  if (rc) return rc;
  if (registers_per_thread) *registers_per_thread = pl.regs;
  if (threads_per_block) *threads_per_block = gpp::kThreads;
  if (blocks_per_sm) *blocks_per_sm = pl.blocks_per_sm;
  if (grid) *grid = pl.grid;
  if (igp_tile) *igp_tile = pl.igp_t;
  if (band_chunk) *band_chunk = pl.bchunk;
  return GPP_OK;
}

int gpp_comm_unique_id(unsigned char* id128) {
  if (!id128) return fail(GPP_ERR_ARG, "id buffer is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  ncclUniqueId id;
  GPP_NCCL(ncclGetUniqueId(&id));
  std::memcpy(id128, &id, sizeof(id));
  return GPP_OK;
}

int gpp_comm_init(gpp_ctx* c, int nranks, int rank, const unsigned char* id128) {
  CtxLock lock(c);
  if (!c) return fail(GPP_ERR_ARG, "ctx is NULL");
  if (!id128) return fail(GPP_ERR_ARG, "id buffer is NULL");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(GPP_ERR_ARG, "rank " + std::to_string(rank) + " outside [0, " +
                                 std::to_string(nranks) + ")");
  int rc = ensure_init(c);
  if (rc) return rc;
  DeviceGuard g(c->device);
  if (!g.ok) return cuda_fail(g.err, "cudaSetDevice");
  if (c->comm) {
    ncclCommDestroy(c->comm);
    c->comm = nullptr;
  }
  c->nranks = nranks;
  c->rank = rank;
  c->comm_aborted = false;
  // A one-rank communicator is created too (cheap; it exercises the error /
  // abort path on one GPU); the collectives only run with nranks > 1.
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  GPP_NCCL(ncclCommInitRank(&c->comm, nranks, id, rank));
  return GPP_OK;
}

static int gpp_synth_impl(gpp_ctx* c, int64_t nbands, int64_t ngpown, int64_t ncouls, int32_t nw,
              const uint64_t* pcg_state, const double* wx, int64_t band0, int64_t band1) {
  CtxLock lock(c);
  if (!c) return fail(GPP_ERR_ARG, "ctx is NULL");
  if (!pcg_state || !wx) return fail(GPP_ERR_ARG, "pcg_state / wx is NULL");
  // Validate like an upload (the array pointers are not used).
  const double dummy = 0.0;
  const HostProblem h{nbands, ngpown, ncouls, nw, &dummy, &dummy, &dummy, &dummy, wx, 0,
                      band0, band1};
  int rc = validate(c, h);
  if (rc) return rc;
  rc = ensure_init(c);
  if (rc) return rc;
  DeviceGuard g(c->device);
  if (!g.ok) return cuda_fail(g.err, "cudaSetDevice");
  c->have_problem = false;
  rc = prepare(c, h);
  if (rc) return rc;
  const gpp::U128 st{pcg_state[0], pcg_state[1]}, inc{pcg_state[2], pcg_state[3]};
  const unsigned long long nwt = static_cast<unsigned long long>(ncouls) * ngpown;
  const unsigned long long nan_ = static_cast<unsigned long long>(ncouls) * nbands;
  // Draw order of synth_problem (problem.py:136-141): wtilde re, im; i_eps re,
  // im; aqsntemp re, im; aqsmtemp re, im; then wx.
  struct Block {
    unsigned long long offset;
    long long rows, cols, c0, c1;
    double2* dst;
    int comp;
  };
  const Block blocks[8] = {
      {0, ncouls, ngpown, 0, ngpown, c->wtilde.ptr, 0},
      {nwt, ncouls, ngpown, 0, ngpown, c->wtilde.ptr, 1},
      {2 * nwt, ncouls, ngpown, 0, ngpown, c->eps.ptr, 0},
      {3 * nwt, ncouls, ngpown, 0, ngpown, c->eps.ptr, 1},
      {4 * nwt, ncouls, nbands, band0, band1, c->aqsn.ptr, 0},
      {4 * nwt + nan_, ncouls, nbands, band0, band1, c->aqsn.ptr, 1},
      {4 * nwt + 2 * nan_, ngpown, nbands, band0, band1, c->aqsm.ptr, 0},
      {4 * nwt + 2 * nan_ + static_cast<unsigned long long>(ngpown) * nbands, ngpown, nbands,
       band0, band1, c->aqsm.ptr, 1},
  };
  for (const Block& b : blocks) {
    const int grid = static_cast<int>(std::min<long long>((b.rows + 255) / 256, 65535));
    ++c->launches;
    gpp::gpp_synth_kernel<<<grid, 256, 0, c->stream>>>(st, inc, b.offset, b.rows, b.cols, b.c0,
                                                       b.c1, reinterpret_cast<double*>(b.dst),
                                                       b.comp);
    GPP_CUDA(cudaGetLastError());
  }
  rc = copy_small_wx(c, h, c->stream);
  if (rc) return rc;
  GPP_CUDA(cudaStreamSynchronize(c->stream));
  c->have_problem = true;
  return GPP_OK;
}

static int gpp_run_factored_impl(gpp_ctx* c, int32_t variant, double* achtemp, double* asxtemp,
                                 int64_t* near_far, float* ms) {
  CtxLock lock(c);
  if (!c) return fail(GPP_ERR_ARG, "ctx is NULL");
  if (variant < GPP_VARIANT_DIV || variant > GPP_VARIANT_RCP_SQ)
    return fail(GPP_ERR_ARG, "the factored path takes a reference variant (0=div, 1=rcp, 2=rcp_sq)");
  if (!achtemp || !asxtemp) return fail(GPP_ERR_ARG, "output pointer is NULL");
  if (!c->have_problem) return fail(GPP_ERR_ARG, "no problem uploaded");
  if (!c->wx_band_invariant)
    return fail(GPP_ERR_ARG, "the factored path needs a band-invariant wx (the reference's (nw,) vector)");
  DeviceGuard g(c->device);
  if (!g.ok) return cuda_fail(g.err, "cudaSetDevice");
  GPP_CUDA(cudaEventRecord(c->ev[2], c->stream));
  if (c->nbands == 0) {
    int rc = enqueue_eval(c, GPP_VARIANT_RCP_SQ, near_far != nullptr, nullptr, false);
    if (rc) return rc;
  } else {
    std::vector<std::pair<int, int>> groups;
    nw_groups(c->nw, gpp::kMaxNwGroup, &groups);
    const int n_igblk = static_cast<int>((c->ncouls + gpp::kThreads - 1) / gpp::kThreads);
    const int n_igptile = static_cast<int>((c->ngpown + gpp::kFacIgp - 1) / gpp::kFacIgp);
    const long long n_items = static_cast<long long>(n_igblk) * n_igptile;
    bool first = true;
    for (const auto& gr : groups) {
      const int iw0 = gr.first, nwg = gr.second;
      using FacFn = void (*)(const double2*, const double2*, const double2*, const double2*,
                             const double*, int, int, int, int, int, int, long long,
                             unsigned long long, double*, unsigned long long*);
      FacFn fn = nullptr;
#define GPP_FAC_NW(V)                                               \
  switch (nwg) {                                                    \
    case 1: fn = gpp::gpp_factored_kernel<V, 1>; break;             \
    case 2: fn = gpp::gpp_factored_kernel<V, 2>; break;             \
    case 3: fn = gpp::gpp_factored_kernel<V, 3>; break;             \
    default: fn = gpp::gpp_factored_kernel<V, 4>; break;            \
  }
      if (variant == GPP_VARIANT_DIV) {
        GPP_FAC_NW(0)
      } else if (variant == GPP_VARIANT_RCP) {
        GPP_FAC_NW(1)
      } else {
        GPP_FAC_NW(2)
      }
#undef GPP_FAC_NW
      int bps = 0;
      GPP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, reinterpret_cast<const void*>(fn),
                                                             gpp::kThreads, 0));
      const int grid = static_cast<int>(std::max<long long>(
          1, std::min<long long>(static_cast<long long>(std::max(bps, 1)) * c->num_sms, n_items)));
      GPP_CUDA(c->partials.ensure(static_cast<size_t>(grid) * 4 * gpp::kMaxNwGroup));
      GPP_CUDA(c->cpartials.ensure(static_cast<size_t>(grid) * 2));
      fn<<<grid, gpp::kThreads, 0, c->stream>>>(
          c->aqsn.ptr, c->aqsm.ptr, c->wtilde.ptr, c->eps.ptr, c->wxb.ptr, c->nw, iw0,
          static_cast<int>(c->ncouls), static_cast<int>(c->ngpown), static_cast<int>(c->nbands),
          n_igptile, n_items, static_cast<unsigned long long>(c->nbands), c->partials.ptr,
          c->cpartials.ptr);
      GPP_CUDA(cudaGetLastError());
      c->launches += 2;  // fused GEMM + terms, finalize
      pick_finalize(nwg)<<<1, 256, 0, c->stream>>>(c->partials.ptr, c->cpartials.ptr, grid, c->nw,
                                                    iw0, 0, first ? 1 : 0, 1, c->out.ptr,
                                                    c->counts.ptr);
      GPP_CUDA(cudaGetLastError());
      first = false;
    }
  }
  GPP_CUDA(cudaEventRecord(c->ev[3], c->stream));
  int rc = finish_run(c, achtemp, asxtemp, near_far);
  if (rc) return rc;
  if (ms) GPP_CUDA(cudaEventElapsedTime(ms, c->ev[2], c->ev[3]));
  return GPP_OK;
}

int gpp_variant_terms(gpp_ctx* c, int32_t variant, double* sch, double* ssx, uint8_t* near_mask,
                      uint8_t* far_mask) {
  CtxLock lock(c);
  if (!c) return fail(GPP_ERR_ARG, "ctx is NULL");
  if (variant < GPP_VARIANT_DIV || variant > GPP_VARIANT_RCP_SQ)
    return fail(GPP_ERR_ARG, "variant_terms takes a reference variant (0=div, 1=rcp, 2=rcp_sq)");
  if (!sch || !ssx || !near_mask || !far_mask) return fail(GPP_ERR_ARG, "output pointer is NULL");
  if (!c->have_problem) return fail(GPP_ERR_ARG, "no problem uploaded");
  if (!c->wx_band_invariant)
    return fail(GPP_ERR_ARG, "variant_terms needs a band-invariant wx (the reference's (nw,) vector)");
  DeviceGuard g(c->device);
  if (!g.ok) return cuda_fail(g.err, "cudaSetDevice");
  const size_t n = static_cast<size_t>(c->nw) * c->ncouls * c->ngpown;
  DevBuf<double2> d_sch, d_ssx;
  DevBuf<unsigned char> d_near, d_far;
  int rc = GPP_OK;
  do {
    cudaError_t e = d_sch.ensure(n);
    if (e == cudaSuccess) e = d_ssx.ensure(n);
    if (e == cudaSuccess) e = d_near.ensure(n);
    if (e == cudaSuccess) e = d_far.ensure(n);
    if (e != cudaSuccess) { rc = cuda_fail(e, "variant_terms buffers"); break; }
    const long long n_el = c->ncouls * c->ngpown;
    const int grid = static_cast<int>(std::max<long long>(
        1, std::min<long long>(c->num_sms * 8, (n_el + gpp::kThreads - 1) / gpp::kThreads)));
#define GPP_VT(V)                                                                              \
  gpp::gpp_variant_terms_kernel<V><<<grid, gpp::kThreads, 0, c->stream>>>(                     \
      c->wtilde.ptr, c->eps.ptr, c->wxb.ptr, c->nw, c->ncouls, c->ngpown, d_sch.ptr, d_ssx.ptr, \
      d_near.ptr, d_far.ptr)
    if (variant == GPP_VARIANT_DIV) GPP_VT(0);
    else if (variant == GPP_VARIANT_RCP) GPP_VT(1);
    else GPP_VT(2);
#undef GPP_VT
    ++c->launches;
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(sch, d_sch.ptr, n * sizeof(double2), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ssx, d_ssx.ptr, n * sizeof(double2), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(near_mask, d_near.ptr, n, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(far_mask, d_far.ptr, n, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "variant_terms");
  } while (0);
  d_sch.release();
  d_ssx.release();
  d_near.release();
  d_far.release();
  return rc;
}

int gpp_comm_init_all(gpp_ctx** ctxs, int n) {
  CtxLock lock(ctxs, n);
  if (!ctxs || n < 1) return fail(GPP_ERR_ARG, "need at least one context");
  std::vector<int> devs(n);
  for (int i = 0; i < n; ++i) {
    if (!ctxs[i]) return fail(GPP_ERR_ARG, "context " + std::to_string(i) + " is NULL");
    for (int j = 0; j < i; ++j)
      if (ctxs[j]->device == ctxs[i]->device)
        return fail(GPP_ERR_ARG, "contexts must be on distinct devices");
    int rc = ensure_init(ctxs[i]);
    if (rc) return rc;
    devs[i] = ctxs[i]->device;
    if (ctxs[i]->comm) {
      DeviceGuard g(ctxs[i]->device);
      ncclCommDestroy(ctxs[i]->comm);
      ctxs[i]->comm = nullptr;
    }
  }
  for (int i = 0; i < n; ++i) {
    ctxs[i]->nranks = n;
    ctxs[i]->rank = i;
  }
  if (n == 1) return GPP_OK;
  std::vector<ncclComm_t> comms(n);
  GPP_NCCL(ncclCommInitAll(comms.data(), n, devs.data()));
  for (int i = 0; i < n; ++i) ctxs[i]->comm = comms[i];
  return GPP_OK;
}

static int gpp_run_group_impl(gpp_ctx** ctxs, int n, int32_t variant, double* achtemp, double* asxtemp,
                  int64_t* near_far, float* kernel_ms) {
  CtxLock lock(ctxs, n);
  if (!ctxs || n < 1) return fail(GPP_ERR_ARG, "need at least one context");
  int rc = check_variant(variant);
  if (rc) return rc;
  if (!achtemp || !asxtemp) return fail(GPP_ERR_ARG, "output pointer is NULL");
  for (int i = 0; i < n; ++i) {
    if (!ctxs[i] || !ctxs[i]->have_problem)
      return fail(GPP_ERR_ARG, "context " + std::to_string(i) + " has no problem uploaded");
    if (ctxs[i]->nw != ctxs[0]->nw)
      return fail(GPP_ERR_ARG, "contexts hold problems with different nw");
    if (n > 1 && (!ctxs[i]->comm || ctxs[i]->nranks != n))
      return fail(GPP_ERR_ARG, "contexts need gpp_comm_init_all over the same group");
  }
  // Every device's shard first, then one grouped allreduce across them (a
  // single thread must issue all ranks' collectives inside one group).
  for (int i = 0; i < n; ++i) {
    gpp_ctx* c = ctxs[i];
    DeviceGuard g(c->device);
    if (!g.ok) return cuda_fail(g.err, "cudaSetDevice");
    GPP_CUDA(cudaEventRecord(c->ev[2], c->stream));
    rc = enqueue_eval(c, variant, near_far != nullptr, nullptr, false);
    if (rc) return rc;
    GPP_CUDA(cudaEventRecord(c->ev[3], c->stream));
  }
  if (n > 1) {
    GPP_NCCL(ncclGroupStart());
    for (int i = 0; i < n; ++i) {
      gpp_ctx* c = ctxs[i];
      GPP_NCCL(ncclAllReduce(c->out.ptr, c->out.ptr, 4 * c->nw, ncclDouble, ncclSum, c->comm,
                             c->stream));
      GPP_NCCL(ncclAllReduce(c->counts.ptr, c->counts.ptr, 2, ncclUint64, ncclSum, c->comm,
                             c->stream));
    }
    GPP_NCCL(ncclGroupEnd());
  }
  float worst = 0.f;
  for (int i = 0; i < n; ++i) {
    gpp_ctx* c = ctxs[i];
    DeviceGuard g(c->device);
    if (!g.ok) return cuda_fail(g.err, "cudaSetDevice");
    rc = wait_stream(c, c->stream);
    if (rc) return rc;
    float ms = 0.f;
    GPP_CUDA(cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]));
    worst = std::max(worst, ms);
  }
  gpp_ctx* c0 = ctxs[0];
  {
    DeviceGuard g(c0->device);
    if (!g.ok) return cuda_fail(g.err, "cudaSetDevice");
    GPP_CUDA(cudaMemcpy(c0->h_out, c0->out.ptr, 4 * sizeof(double) * c0->nw, cudaMemcpyDeviceToHost));
    GPP_CUDA(cudaMemcpy(c0->h_counts, c0->counts.ptr, 2 * sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost));
  }
  std::memcpy(achtemp, c0->h_out, 2 * sizeof(double) * c0->nw);
  std::memcpy(asxtemp, c0->h_out + 2 * c0->nw, 2 * sizeof(double) * c0->nw);
  if (near_far) {
    near_far[0] = static_cast<int64_t>(c0->h_counts[0]);
    near_far[1] = static_cast<int64_t>(c0->h_counts[1]);
  }
  if (kernel_ms) *kernel_ms = worst;
  return GPP_OK;
}

int gpp_host_register(void* ptr, size_t bytes) {
  if (!ptr || bytes == 0) return fail(GPP_ERR_ARG, "empty host range");
  GPP_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault));
  return GPP_OK;
}

int gpp_host_unregister(void* ptr) {
  if (!ptr) return fail(GPP_ERR_ARG, "ptr is NULL");
  GPP_CUDA(cudaHostUnregister(ptr));
  return GPP_OK;
}

int gpp_fp64_peak(int device, int32_t iters, double* tflops, float* ms) {
  if (device < 0 || iters < 1) return fail(GPP_ERR_ARG, "bad device or iters");
  int n = 0;
  GPP_CUDA(cudaGetDeviceCount(&n));
  if (device >= n) return fail(GPP_ERR_ARG, "device out of range");
  DeviceGuard g(device);
  if (!g.ok) return cuda_fail(g.err, "cudaSetDevice");
  int sms = 0;
  GPP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  double* sink = nullptr;
  GPP_CUDA(cudaMalloc(&sink, 256 * sizeof(double)));
  cudaEvent_t a, b;
  GPP_CUDA(cudaEventCreate(&a));
  GPP_CUDA(cudaEventCreate(&b));
  const int grid = sms * 8;  // 8 x 256 threads = 64 warps per SM
  gpp::fp64_peak_kernel<<<grid, 256>>>(sink, std::max(1, iters / 10), 0.999999, 1e-7);  // warm
  GPP_CUDA(cudaEventRecord(a));
  gpp::fp64_peak_kernel<<<grid, 256>>>(sink, iters, 0.999999, 1e-7);
  GPP_CUDA(cudaEventRecord(b));
  GPP_CUDA(cudaEventSynchronize(b));
  float t = 0.f;
  GPP_CUDA(cudaEventElapsedTime(&t, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  const double flops = 2.0 * 8.0 * static_cast<double>(iters) * grid * 256.0;
  if (tflops) *tflops = flops / (t * 1e-3) / 1e12;
  if (ms) *ms = t;
  return GPP_OK;
}


// ----- public entry points: the implementations above, behind comm_guard ---
int gpp_upload(gpp_ctx* c, int64_t nbands, int64_t ngpown, int64_t ncouls, int32_t nw,
               const double* wtilde, const double* i_eps, const double* aqsntemp,
               const double* aqsmtemp, const double* wx, int32_t wx_band_indexed,
               int64_t band0, int64_t band1) {
  int rc = comm_alive(c);
  if (rc) return rc;
  return comm_guard(c, gpp_upload_impl(c, nbands, ngpown, ncouls, nw, wtilde, i_eps, aqsntemp,
                                       aqsmtemp, wx, wx_band_indexed, band0, band1));
}

int gpp_evaluate_host(gpp_ctx* c, int32_t variant, int64_t nbands, int64_t ngpown, int64_t ncouls,
                      int32_t nw, const double* wtilde, const double* i_eps,
                      const double* aqsntemp, const double* aqsmtemp, const double* wx,
                      int32_t wx_band_indexed, int64_t band0, int64_t band1, int32_t slabs,
                      double* achtemp, double* asxtemp, int64_t* near_far, float* ms) {
  int rc = comm_alive(c);
  if (rc) return rc;
  return comm_guard(c, gpp_evaluate_host_impl(c, variant, nbands, ngpown, ncouls, nw, wtilde,
                                              i_eps, aqsntemp, aqsmtemp, wx, wx_band_indexed,
                                              band0, band1, slabs, achtemp, asxtemp, near_far,
                                              ms));
}

int gpp_run(gpp_ctx* c, int32_t variant, double* achtemp, double* asxtemp, int64_t* near_far,
            float* kernel_ms) {
  int rc = comm_alive(c);
  if (rc) return rc;
  return comm_guard(c, gpp_run_impl(c, variant, achtemp, asxtemp, near_far, kernel_ms));
}

int gpp_time(gpp_ctx* c, int32_t variant, int32_t iters, float* total_ms, float* main_ms) {
  int rc = comm_alive(c);
  if (rc) return rc;
  return comm_guard(c, gpp_time_impl(c, variant, iters, total_ms, main_ms));
}

int gpp_synth(gpp_ctx* c, int64_t nbands, int64_t ngpown, int64_t ncouls, int32_t nw,
              const uint64_t* pcg_state, const double* wx, int64_t band0, int64_t band1) {
  int rc = comm_alive(c);
  if (rc) return rc;
  return comm_guard(c, gpp_synth_impl(c, nbands, ngpown, ncouls, nw, pcg_state, wx, band0, band1));
}

int gpp_run_factored(gpp_ctx* c, int32_t variant, double* achtemp, double* asxtemp,
                     int64_t* near_far, float* ms) {
  int rc = comm_alive(c);
  if (rc) return rc;
  return comm_guard(c, gpp_run_factored_impl(c, variant, achtemp, asxtemp, near_far, ms));
}

static int group_guard(gpp_ctx** ctxs, int n, int rc) {
  for (int i = 0; rc != GPP_OK && ctxs && i < n; ++i) comm_guard(ctxs[i], rc);
  return rc;
}

int gpp_run_group(gpp_ctx** ctxs, int n, int32_t variant, double* achtemp, double* asxtemp,
                  int64_t* near_far, float* kernel_ms) {
  for (int i = 0; ctxs && i < n; ++i) {
    int rc = comm_alive(ctxs[i]);
    if (rc) return rc;
  }
  return group_guard(ctxs, n,
                     gpp_run_group_impl(ctxs, n, variant, achtemp, asxtemp, near_far, kernel_ms));
}

// Device-resident timing of the single-process group: `iters`
// evaluations enqueued back to back on every device, each followed by one
// grouped ncclAllReduce of the partials, no host synchronisation in between;
// total_ms / main_ms = the slowest device's event time of the whole run / of
// its summed main-kernel spans.
static int gpp_time_group_impl(gpp_ctx** ctxs, int n, int32_t variant, int32_t iters,
                               float* total_ms, float* main_ms) {
  if (!ctxs || n < 1) return fail(GPP_ERR_ARG, "need at least one context");
  CtxLock lock(ctxs, n);
  int rc = check_variant(variant);
  if (rc) return rc;
  if (iters < 1) return fail(GPP_ERR_ARG, "iters must be at least 1");
  for (int i = 0; i < n; ++i) {
    if (!ctxs[i] || !ctxs[i]->have_problem)
      return fail(GPP_ERR_ARG, "context " + std::to_string(i) + " has no problem uploaded");
    if (ctxs[i]->nw != ctxs[0]->nw)
      return fail(GPP_ERR_ARG, "contexts hold problems with different nw");
    if (n > 1 && (!ctxs[i]->comm || ctxs[i]->nranks != n))
      return fail(GPP_ERR_ARG, "contexts need gpp_comm_init_all over the same group");
  }
  std::vector<std::vector<cudaEvent_t>> evs(n, std::vector<cudaEvent_t>(2 * static_cast<size_t>(iters)));
  int result = GPP_OK;
  for (int i = 0; i < n && result == GPP_OK; ++i) {
    DeviceGuard g(ctxs[i]->device);
    for (auto& e : evs[i])
      if (result == GPP_OK && cudaEventCreate(&e) != cudaSuccess) result = fail(GPP_ERR_CUDA, "cudaEventCreate");
  }
  for (int i = 0; i < n && result == GPP_OK; ++i) {
    DeviceGuard g(ctxs[i]->device);
    if (cudaEventRecord(ctxs[i]->ev[2], ctxs[i]->stream) != cudaSuccess)
      result = fail(GPP_ERR_CUDA, "cudaEventRecord");
  }
  for (int it = 0; it < iters && result == GPP_OK; ++it) {
    for (int i = 0; i < n && result == GPP_OK; ++i) {
      DeviceGuard g(ctxs[i]->device);
      result = enqueue_eval(ctxs[i], variant, false, &evs[i][2 * static_cast<size_t>(it)], false);
    }
    if (result == GPP_OK && n > 1) {
      ncclResult_t r = ncclGroupStart();
      for (int i = 0; i < n && r == ncclSuccess; ++i) {
        gpp_ctx* c = ctxs[i];
        r = ncclAllReduce(c->out.ptr, c->out.ptr, 4 * c->nw, ncclDouble, ncclSum, c->comm, c->stream);
        if (r == ncclSuccess)
          r = ncclAllReduce(c->counts.ptr, c->counts.ptr, 2, ncclUint64, ncclSum, c->comm, c->stream);
      }
      const ncclResult_t r2 = ncclGroupEnd();
      if (r != ncclSuccess || r2 != ncclSuccess)
        result = fail(GPP_ERR_NCCL, std::string("grouped ncclAllReduce: ") +
                                        ncclGetErrorString(r != ncclSuccess ? r : r2));
    }
  }
  float worst_tot = 0.f, worst_main = 0.f;
  for (int i = 0; i < n && result == GPP_OK; ++i) {
    gpp_ctx* c = ctxs[i];
    DeviceGuard g(c->device);
    if (cudaEventRecord(c->ev[3], c->stream) != cudaSuccess) {
      result = fail(GPP_ERR_CUDA, "cudaEventRecord");
      break;
    }
    result = wait_stream(c, c->stream);
    if (result) break;
    float tot = 0.f, mm = 0.f;
    cudaEventElapsedTime(&tot, c->ev[2], c->ev[3]);
    for (int it = 0; it < iters; ++it) {
      float x = 0.f;
      cudaEventElapsedTime(&x, evs[i][2 * it], evs[i][2 * it + 1]);
      mm += x;
    }
    worst_tot = std::max(worst_tot, tot);
    worst_main = std::max(worst_main, mm);
  }
  for (int i = 0; i < n; ++i) {
    DeviceGuard g(ctxs[i]->device);
    for (auto& e : evs[i])
      if (e) cudaEventDestroy(e);
  }
  if (result == GPP_OK) {
    if (total_ms) *total_ms = worst_tot;
    if (main_ms) *main_ms = worst_main;
  }
  return result;
}

int gpp_time_group(gpp_ctx** ctxs, int n, int32_t variant, int32_t iters, float* total_ms,
                   float* main_ms) {
  for (int i = 0; ctxs && i < n; ++i) {
    int rc = comm_alive(ctxs[i]);
    if (rc) return rc;
  }
  return group_guard(ctxs, n, gpp_time_group_impl(ctxs, n, variant, iters, total_ms, main_ms));
}

}  // extern "C"
