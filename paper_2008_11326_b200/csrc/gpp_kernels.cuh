// gpp_kernels.cuh -- sm_100a FP64 kernels of the GPP self-energy reduction.
//
// The reduction (reference semantics: rooflab/gpp/problem.py:179-208 and
// rooflab/gpp/kernel.py:63-114):
//
//   for band, igp, ig, iw:
//     wdiff = wx[iw, band] - wtilde[ig, igp]
//     delw  = wtilde / wdiff
//     near  = |wdiff| > 0.5 && |delw| < 2          far = !near && |delw| > 1e-12
//     sch   = near ? 0.5 * delw * eps : 0
//     ssx   = near ? delw * eps : far ? -0.25 * eps / |delw| : 0
//     t     = aqsntemp[ig, band] * conj(aqsmtemp[igp, band])
//     achtemp[iw] += sch * t ;  asxtemp[iw] += ssx * t
//
// Work decomposition (one persistent CTA per SM slot, static round-robin
// items so the reduction order -- and therefore the result -- is
// deterministic run to run):
//   item  = (igp tile of IGP_T, ig block of 256, band chunk)
//   thread <-> ig (coalesced along the F-order ig-fastest arrays); the
//   IGP_T (ig, igp) states live in registers; the band loop runs innermost
//   with aqsmtemp[igp tile, band chunk] staged in shared memory (uniform
//   broadcast reads); aqsntemp[ig, band] is streamed from global through a
//   per-thread cp.async ring kAnDepth bands deep, so its latency is covered
//   without holding prefetched values in registers.  Items are ordered
//   igp-tile fastest, so the CTAs resident at one time share the same
//   aqsntemp tile through L2.
//   iw is innermost: t = an conj(am) is formed once per (band, igp, ig) and
//   reused by every frequency from registers (the paper's iw hoist).
// The production kernel is gpp_sacc_kernel (per-(igp, iw) band sums, wx as a
// by-value parameter table, cross-item pipelining); the
// gpp_main_kernel policies are the version-ladder kernels (v0-v7).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gpp {

constexpr int kThreads = 256;     // threads per CTA (= ig per item)
constexpr int kMaxChunk = 128;    // bands per item (upper bound)
#ifndef GPP_ABL
#define GPP_ABL 0  // timing ablations (tools/ablate.sh); 0 in every real build
#endif
#ifndef GPP_SACC_CHUNK
#define GPP_SACC_CHUNK 256
#endif
constexpr int kSaccChunk = GPP_SACC_CHUNK;  // bands per item of gpp_sacc_kernel (upper bound)
// Item capacity (bands) of gpp_sacc_kernel's aqsmtemp staging per frequency
// count: 512 at NW = 2-3 (two-igp tiles; 96-104 KB of shared memory per CTA,
// still two per SM), kSaccChunk at NW = 1 (a three-igp tile).
template <int NW>
constexpr int sacc_cap() { return NW >= 2 ? 2 * kSaccChunk : kSaccChunk; }
constexpr int kMaxIgpTile = 4;    // igp per thread (upper bound)
constexpr int kMaxNwGroup = 4;    // frequencies per launch (host loops groups)
constexpr int kAnDepth = 4;       // aqsntemp bands in flight per thread (cp.async ring)

struct Params {
  const double2* wtilde;   // (ncouls, ngpown) F-order
  const double2* eps;      // (ncouls, ngpown) F-order
  const double2* aqsn;     // (ncouls, nb) F-order, nb = local band count
  const double2* aqsm;     // (ngpown, nb) F-order
  const double* wxb;       // (nb, nw_total): wxb[band * nw_total + iw]
  int ncouls, ngpown, nbands;
  int nw_total, iw0;       // this launch evaluates iw in [iw0, iw0 + NW)
  int igblk0;              // first 256-ig block of this launch (ig slab)
  int band0;               // first (local) band of this launch's band window (gpp_sacc_kernel)
  int n_igblk, n_igptile, bchunk;
  long long n_items;
  // Division by n_igptile / n_rows (below) as multiply-shift (host:
  // fastdiv_init), so that gpp_sacc_kernel decomposes its items on the
  // uniform datapath and the band offset indexing the WxTable stays in a
  // uniform register.
  unsigned long long igpt_mul;
  int igpt_shift;
  // gpp_sacc_kernel enumerates rows [row0, row0 + n_rows) of (igb, igp tile)
  // pairs (tile fastest; row = igb * n_igptile + tile) times band chunks of
  // its window: item = chunk * n_rows + (row - row0).  A whole launch has
  // row0 = 0 and n_rows = n_igblk * n_igptile; a balanced-tail launch covers
  // the last rows of the last chunk in finer chunks (host: enqueue_eval).
  int row0, n_rows;
  unsigned long long rows_mul;
  int rows_shift;
  double wxmax;            // max |wx| over the uploaded bands (regular-item guard)
  // gpp_sacc_kernel writes one row of 4 * NW doubles per (item, warp) into the
  // canonical slot of its (band chunk, row): slot = slot_base + chunk *
  // slot_stride + row (host: the whole-problem plan numbers every item once,
  // so every schedule -- resident, ig slabs, any grid -- writes the same
  // values to the same slots and the finalize sums them in slot order).
  long long slot_base;
  int slot_stride;
  double* partials;                 // [gridDim.x][4 * NW]  (gpp_sacc_kernel: [slot][warp][4 * NW])
  unsigned long long* cpartials;    // [gridDim.x][2]
};

// floor(n / d) for 0 <= n < 2^31 with m = ceil(2^(32+l) / d), l = ceil(log2 d):
// the error term n (m d - 2^(32+l)) < 2^31 d <= 2^(32+l) stays below one unit.
__host__ __device__ __forceinline__ unsigned fastdiv(unsigned n, unsigned long long m, int shift) {
  return static_cast<unsigned>((static_cast<unsigned long long>(n) * m) >> shift);
}
inline void fastdiv_init(unsigned d, unsigned long long* m, int* shift) {
  int l = 0;
  while ((1ull << l) < d) ++l;
  *shift = 32 + l;
  *m = ((1ull << (32 + l)) + d - 1) / d;
}

// wx of one launch's band window, passed by value as a __grid_constant__
// kernel parameter: w[(band - band0) * NW + (iw - iw0)].  The band loop's
// reads of it are warp-uniform with a uniform index, so ptxas serves them
// with LDCU into uniform registers and the DADD / DMUL that consume wx take
// it as a UR operand -- one 64-bit register-file read fewer per use in this
// register-file-read-bound loop, and no shared-memory staging of wx.
constexpr int kWxParam = 1536;  // 12 KB: 512 bands at NW = 3, 768 at 2, 1536 at 1
struct WxTable {
  double w[kWxParam];
};

// ---------------------------------------------------------------------------
// FP64 primitives.  rcp/rsqrt start from the MUFU.RCP64H / MUFU.RSQ64H
// approximations and refine with DFMA Newton steps (no IEEE slow path).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double rcp_approx(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
__device__ __forceinline__ double rsqrt_approx(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
// 1/d to ~1 ulp: one cubic Newton step, r(1 + e + e^2) with e = 1 - d r.
__device__ __forceinline__ double rcp_refined(double d) {
  double r = rcp_approx(d);
  double e = fma(-d, r, 1.0);
  e = fma(e, e, e);
  return fma(e, r, r);
}

// cp.async (LDGSTS) of one 16-byte aqsntemp element into this thread's slot
// of the shared-memory ring.  Each thread only ever reads the slots it filled
// itself, so cp.async.wait_group alone orders the copy before the read; no
// CTA barrier is needed.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Bit pattern of 1e24: |delw|^2 > 1e-24  <=>  d / |wt|^2 < 1e24.
constexpr unsigned long long kBits1e24 = 0x44EA784379D99DB4ull;

// ---------------------------------------------------------------------------
// Policies: per-(ig, igp) register state and per-(band, igp, ig) work.
// Acc holds two complex sums per frequency plus near/far counters.
// ---------------------------------------------------------------------------
template <int NW>
struct Acc {
  double2 a[NW];
  double2 b[NW];
  unsigned nn, nf;
};

// Branch selection shared by the fast formulations.  Decisions are integer
// compares on the bit patterns of non-negative doubles (ALU pipe, not the
// FP64 pipe):
//   near <=> bits(d) > bits(qn)
//   far  <=> !near && bits(x) - 1 < bits(1e24) - 1      (x in (0, 1e24))
// Both branch bodies are computed for every instance and only their scalar
// multipliers are selected -- no divergence.  (PTX selp keeps ptxas from
// turning the far select into a branch.)
template <bool COUNT, int NW>
__device__ __forceinline__ void select_branches(double d, long long qbits, double x, double inv,
                                                double g, double& in, double& gf, Acc<NW>& acc) {
  const long long dbits = __double_as_longlong(d);
  const long long xbits = __double_as_longlong(x);
  if constexpr (COUNT) {
    asm("{\n\t.reg .pred pn, pf;\n\t.reg .u64 xm1;\n\t"
        "setp.gt.s64 pn, %4, %5;\n\t"
        "sub.u64 xm1, %6, 1;\n\t"
        "setp.lt.and.u64 pf, xm1, %7, !pn;\n\t"
        "selp.f64 %0, %8, 0d0000000000000000, pn;\n\t"
        "selp.f64 %1, %9, 0d0000000000000000, pf;\n\t"
        "@pn add.u32 %2, %2, 1;\n\t"
        "@pf add.u32 %3, %3, 1;\n\t}"
        : "=d"(in), "=d"(gf), "+r"(acc.nn), "+r"(acc.nf)
        : "l"(dbits), "l"(qbits), "l"(xbits), "l"(kBits1e24 - 1ull), "d"(inv), "d"(g));
  } else {
    asm("{\n\t.reg .pred pn, pf;\n\t.reg .u64 xm1;\n\t"
        "setp.gt.s64 pn, %2, %3;\n\t"
        "sub.u64 xm1, %4, 1;\n\t"
        "setp.lt.and.u64 pf, xm1, %5, !pn;\n\t"
        "selp.f64 %0, %6, 0d0000000000000000, pn;\n\t"
        "selp.f64 %1, %7, 0d0000000000000000, pf;\n\t}"
        : "=d"(in), "=d"(gf)
        : "l"(dbits), "l"(qbits), "l"(xbits), "l"(kBits1e24 - 1ull), "d"(inv), "d"(g));
  }
}

// sqrt(x) from the MUFU.RSQ64H seed r (rel. error ~2^-20, measured).
//   STEPS = 1: one coupled Newton step            4 FP64, rel. error ~1e-12
//   STEPS = 2: two coupled Newton steps           7 FP64, ~1 ulp
//   STEPS = 3: one cubic step r (1 + e/2 + 3e^2/8), e = 1 - x r^2,
//              then sqrt = x r                    5 FP64, ~1 ulp
template <int STEPS>
__device__ __forceinline__ double sqrt_nr(double x) {
  const double r = rsqrt_approx(x);
  if constexpr (STEPS == 3) {
    const double t = x * r;                 // sqrt(x) (1 + O(e))
    const double e = fma(-t, r, 1.0);
    const double p = fma(e, 0.375, 0.5);
    const double q = e * p;
    return fma(t, q, t);
  } else {
    double g = x * r;
    double h = 0.5 * r;
    double e = fma(-g, h, 0.5);
    g = fma(g, e, g);
    if constexpr (STEPS >= 2) {
      h = fma(h, e, h);
      double res = fma(-g, g, x);
      g = fma(res, h, g);
    }
    return g;
  }
}

// RCP_SQ, optimised (the paper's v8 re-derived for Blackwell).
//   d     = |wdiff|^2 = (wx - wt.re)^2 + wt.im^2          (1 DADD + 1 DFMA)
//   inv   = 1/d                                          (MUFU + 3 DFMA)
//   num   = wt * conj(wdiff) = wx * wt - |wt|^2
//   delw  = num * inv,  |delw|^2 = |wt|^2 / d
//   near  <=> d > 0.25  &&  |wt|^2 < 4 d  <=>  d > max(0.25, |wt|^2/4) = qn
//   far   <=> !near && d/|wt|^2 < 1e24
//   sum a += near * inv * num * (eps t)                   -> ach = a/2
//   sum b += far  * sqrt(d/|wt|^2) * (eps t)              -> asx = a - b/4
// ALG 0 forms y = num * (eps t) per instance (6 FP64);  ALG 1 forms
// P = wt*(eps t) and Q = |wt|^2 (eps t) once per (band, igp, ig) and then
// y = wx P - Q per instance (2 DFMA), which pays off from nw = 2 on.
// These are the intermediate kernels of the version ladder
// (GPP_KERNEL_SQ_SPLIT = <0, 2>, GPP_KERNEL_IW_HOIST = <1, 3>).
template <int ALG, int SQRT_STEPS>
struct FastPolicyT {
  struct St {
    double wtr, wti, wti2, wt2, qn, iwt2, er, ei;
  };
  static constexpr bool kHasFastPath = false;
  __device__ __forceinline__ static bool regular(const St&, double) { return false; }

  __device__ __forceinline__ static St make(double2 wt, double2 e, bool valid) {
    St s;
    s.wtr = wt.x;
    s.wti = wt.y;
    s.wti2 = wt.y * wt.y;
    s.wt2 = fma(wt.x, wt.x, s.wti2);
    s.qn = valid ? fmax(0.25, 0.25 * s.wt2) : __longlong_as_double(0x7FF0000000000000ll);
    // x = d * iwt2 must be 0 (never far) on padded lanes and for wt = 0
    // (delw = 0 is degenerate), so those lanes carry iwt2 = 0, not inf.
    s.iwt2 = (valid && s.wt2 > 0.0) ? 1.0 / s.wt2 : 0.0;
    s.er = valid ? e.x : 0.0;
    s.ei = valid ? e.y : 0.0;
    return s;
  }

  template <int NW, bool COUNT, bool FAST>
  __device__ __forceinline__ static void tuple(const St& s, double tr, double ti,
                                               const double (&wx)[NW], Acc<NW>& acc) {
    // eps * t, shared by every frequency.
    const double etr = fma(s.er, tr, -s.ei * ti);
    const double eti = fma(s.er, ti, s.ei * tr);
    const long long qbits = __double_as_longlong(s.qn);
    double pr = 0.0, pi = 0.0, qr = 0.0, qi = 0.0;
    if constexpr (ALG >= 1) {
      pr = fma(s.wtr, etr, -s.wti * eti);
      pi = fma(s.wtr, eti, s.wti * etr);
      qr = s.wt2 * etr;
      qi = s.wt2 * eti;
    }
#pragma unroll
    for (int iw = 0; iw < NW; ++iw) {
      const double wdre = wx[iw] - s.wtr;
      const double d = fma(wdre, wdre, s.wti2);
      const double x = d * s.iwt2;
      double yre, yim;
      if constexpr (ALG >= 1) {
        yre = fma(wx[iw], pr, -qr);
        yim = fma(wx[iw], pi, -qi);
      } else {
        const double nre = fma(s.wtr, wdre, -s.wti2);
        const double nim = s.wti * wx[iw];
        yre = fma(nre, etr, -nim * eti);
        yim = fma(nre, eti, nim * etr);
      }
      double in, gf;
      const double inv = rcp_refined(d);
      const double g = sqrt_nr<SQRT_STEPS>(x);
      select_branches<COUNT>(d, qbits, x, inv, g, in, gf, acc);
      acc.a[iw].x = fma(in, yre, acc.a[iw].x);
      acc.a[iw].y = fma(in, yim, acc.a[iw].y);
      acc.b[iw].x = fma(gf, etr, acc.b[iw].x);
      acc.b[iw].y = fma(gf, eti, acc.b[iw].y);
    }
  }
};
// RCP_SQ, production kernel (ALG 3).  Differences from FastPolicyT:
//  * One MUFU.RSQ64H seed serves both branches: r = rsqrt(d) refined by one
//    cubic step gives sqrt(d) = d r and 1/d = r^2 (~1-2 ulp), so an instance
//    costs one MUFU and 7 FP64 for both reciprocal and square root.
//  * The far body is sqrt(d) * (|wt|^-1 eps t): the 1/|wt| factor is applied
//    once per (band, igp, ig) instead of forming x = d/|wt|^2 per instance.
//  * Regular items: when no instance of an item can be degenerate -- wt.im != 0
//    (so d > 0) and |wt|^2 > 1e-24 (max|wx| + |wt|)^2 (so |delw| > 1e-12) --
//    far is exactly !near and the 64-bit far compare disappears.  Items that
//    are not regular (and the counting kernel) take the general path, which
//    evaluates the full far test.
// The optimisations were chosen against the measured register-file read
// model of the loop (tools/sass_rf.py): the kernel is bound by
// operand reads, not by the FP64 pipe, so ALU and FP64 instructions both
// count.
struct FastPolicy3 {
  struct St {
    double wtr, wti, wti2, wt2, qn, rwt, er, ei;
  };
  static constexpr bool kHasFastPath = true;

  __device__ __forceinline__ static St make(double2 wt, double2 e, bool valid) {
    St s;
    s.wtr = wt.x;
    s.wti = wt.y;
    s.wti2 = wt.y * wt.y;
    s.wt2 = fma(wt.x, wt.x, s.wti2);
    s.qn = valid ? fmax(0.25, 0.25 * s.wt2) : __longlong_as_double(0x7FF0000000000000ll);
    // Padded lanes and wt == 0 carry rwt = 0: never far in the general path
    // (x = 0) and a zero far term in the regular path.
    s.rwt = (valid && s.wt2 > 0.0) ? 1.0 / sqrt(s.wt2) : 0.0;
    s.er = valid ? e.x : 0.0;
    s.ei = valid ? e.y : 0.0;
    return s;
  }
  // No instance of this (ig, igp) can be degenerate for any wx with
  // |wx| <= wxmax.  (Padded lanes: qn = inf and eps = 0, so they contribute
  // nothing on either path.)
  __device__ __forceinline__ static bool regular(const St& s, double wxmax) {
    if (s.qn == __longlong_as_double(0x7FF0000000000000ll)) return true;
    if (s.wti == 0.0) return false;
    const double m = wxmax + sqrt(s.wt2);
    return s.wt2 > 1.000001e-24 * m * m;
  }

  template <int NW, bool COUNT, bool FAST>
  __device__ __forceinline__ static void tuple(const St& s, double tr, double ti,
                                               const double (&wx)[NW], Acc<NW>& acc) {
    const double etr = fma(s.er, tr, -s.ei * ti);
    const double eti = fma(s.er, ti, s.ei * tr);
    const double pr = fma(s.wtr, etr, -s.wti * eti);
    const double pi = fma(s.wtr, eti, s.wti * etr);
    const double qr = s.wt2 * etr;
    const double qi = s.wt2 * eti;
    const long long qbits = __double_as_longlong(s.qn);
    if constexpr (FAST && !COUNT) {
      const double efr = s.rwt * etr;
      const double efi = s.rwt * eti;
#pragma unroll
      for (int iw = 0; iw < NW; ++iw) {
        const double wdre = wx[iw] - s.wtr;
        const double d = fma(wdre, wdre, s.wti2);
        const double r = rsqrt_approx(d);
        const double t = d * r;
        const double e = fma(-t, r, 1.0);
        const double pe = fma(e, 0.375, 0.5);
        const double q = e * pe;
        const double rr = fma(r, q, r);  // 1/sqrt(d)
        const double sq = fma(t, q, t);  // sqrt(d)
        const double inv = rr * rr;      // 1/d
        const double yre = fma(wx[iw], pr, -qr);
        const double yim = fma(wx[iw], pi, -qi);
        double in, gf;
        asm("{\n\t.reg .pred pn;\n\t"
            "setp.gt.s64 pn, %2, %3;\n\t"
            "selp.f64 %0, %4, 0d0000000000000000, pn;\n\t"
            "selp.f64 %1, 0d0000000000000000, %5, pn;\n\t}"
            : "=d"(in), "=d"(gf)
            : "l"(__double_as_longlong(d)), "l"(qbits), "d"(inv), "d"(sq));
        acc.a[iw].x = fma(in, yre, acc.a[iw].x);
        acc.a[iw].y = fma(in, yim, acc.a[iw].y);
        acc.b[iw].x = fma(gf, efr, acc.b[iw].x);
        acc.b[iw].y = fma(gf, efi, acc.b[iw].y);
      }
    } else {
      const double iwt2 = s.rwt * s.rwt;
#pragma unroll
      for (int iw = 0; iw < NW; ++iw) {
        const double wdre = wx[iw] - s.wtr;
        const double d = fma(wdre, wdre, s.wti2);
        const double inv = rcp_refined(d);
        const double x = d * iwt2;
        const double yre = fma(wx[iw], pr, -qr);
        const double yim = fma(wx[iw], pi, -qi);
        const double g = sqrt_nr<3>(x);
        double in, gf;
        select_branches<COUNT>(d, qbits, x, inv, g, in, gf, acc);
        acc.a[iw].x = fma(in, yre, acc.a[iw].x);
        acc.a[iw].y = fma(in, yim, acc.a[iw].y);
        acc.b[iw].x = fma(gf, etr, acc.b[iw].x);
        acc.b[iw].y = fma(gf, eti, acc.b[iw].y);
      }
    }
  }
};

using FastPolicy = FastPolicy3;

// DIV / RCP / RCP_SQ "as written": the reference's per-instance formulas
// (kernel.py:68-95) with IEEE division and sqrt, both branch bodies and two
// complex accumulations per instance (a = ach, b = asx).  These are the
// paper's v0/v1/v3 arithmetic on the same traversal, kept for the version
// ladder and for evaluate_variant(problem, "div" | "rcp").
template <int VARIANT>
struct PlainPolicy {
  struct St {
    double wtr, wti, er, ei;
    bool valid;
  };
  static constexpr bool kHasFastPath = false;

  __device__ __forceinline__ static St make(double2 wt, double2 e, bool valid) {
    St s;
    s.wtr = wt.x;
    s.wti = wt.y;
    s.er = valid ? e.x : 0.0;
    s.ei = valid ? e.y : 0.0;
    s.valid = valid;
    return s;
  }
  __device__ __forceinline__ static bool regular(const St&, double) { return false; }

  template <int NW, bool COUNT, bool FAST>
  __device__ __forceinline__ static void tuple(const St& s, double tr, double ti,
                                               const double (&wx)[NW], Acc<NW>& acc) {
#pragma unroll
    for (int iw = 0; iw < NW; ++iw) {
      const double wdr = wx[iw] - s.wtr;
      const double wdi = -s.wti;
      double dr, di;  // delw
      if (VARIANT == 0) {
        // Library-style complex division wt / wdiff (Smith's scaling).
        if (fabs(wdr) >= fabs(wdi)) {
          const double rat = wdi / wdr;
          const double den = wdr + wdi * rat;
          dr = (s.wtr + s.wti * rat) / den;
          di = (s.wti - s.wtr * rat) / den;
        } else {
          const double rat = wdr / wdi;
          const double den = wdr * rat + wdi;
          dr = (s.wtr * rat + s.wti) / den;
          di = (s.wti * rat - s.wtr) / den;
        }
      } else {
        const double den = wdr * wdr + wdi * wdi;
        const double inv = 1.0 / den;
        const double rr = wdr * inv, ri = -wdi * inv;  // conj(wdiff) * inv
        dr = s.wtr * rr - s.wti * ri;
        di = s.wtr * ri + s.wti * rr;
      }
      bool near, far;
      double delwr;
      if (VARIANT == 2) {
        const double wsq = wdr * wdr + wdi * wdi;
        const double dsq = dr * dr + di * di;
        near = (wsq > 0.25) && (dsq < 4.0);
        far = !near && (dsq > 1e-24);
        delwr = sqrt(dsq);
      } else {
        const double wabs = hypot(wdr, wdi);
        delwr = hypot(dr, di);
        near = (wabs > 0.5) && (delwr < 2.0);
        far = !near && (delwr > 1e-12);
      }
      near = near && s.valid;
      far = far && s.valid;
      const double pr = dr * s.er - di * s.ei;
      const double pi = dr * s.ei + di * s.er;
      double schr = 0.0, schi = 0.0, ssxr = 0.0, ssxi = 0.0;
      if (near) {
        schr = 0.5 * pr;
        schi = 0.5 * pi;
        ssxr = pr;
        ssxi = pi;
      } else if (far) {
        ssxr = -0.25 * s.er / delwr;
        ssxi = -0.25 * s.ei / delwr;
      }
      acc.a[iw].x += schr * tr - schi * ti;
      acc.a[iw].y += schr * ti + schi * tr;
      acc.b[iw].x += ssxr * tr - ssxi * ti;
      acc.b[iw].y += ssxr * ti + ssxi * tr;
      if (COUNT) {
        acc.nn += near;
        acc.nf += far;
      }
    }
  }
};

// ---------------------------------------------------------------------------
// Main kernel.
// ---------------------------------------------------------------------------
// Deterministic block reduction of the per-thread accumulators: warp xor-tree,
// then the warps in order; one row of 4*NW doubles (+2 counts, scaled by
// count_scale) per CTA.
template <int NW, bool COUNT>
__device__ __forceinline__ void block_reduce_write(const Acc<NW>& acc, double* partials,
                                                   unsigned long long* cpartials,
                                                   unsigned long long count_scale) {
  __shared__ double s_red[kThreads / 32][4 * NW];
  __shared__ unsigned long long s_cred[kThreads / 32][2];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  double v[4 * NW];
#pragma unroll
  for (int iw = 0; iw < NW; ++iw) {
    v[4 * iw + 0] = acc.a[iw].x;
    v[4 * iw + 1] = acc.a[iw].y;
    v[4 * iw + 2] = acc.b[iw].x;
    v[4 * iw + 3] = acc.b[iw].y;
  }
  unsigned long long cn = acc.nn, cf = acc.nf;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < 4 * NW; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
    cn += __shfl_xor_sync(0xffffffffu, cn, off);
    cf += __shfl_xor_sync(0xffffffffu, cf, off);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 4 * NW; ++k) s_red[warp][k] = v[k];
    s_cred[warp][0] = cn;
    s_cred[warp][1] = cf;
  }
  __syncthreads();
  if (tid < 4 * NW) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) sum += s_red[w][tid];
    partials[static_cast<size_t>(blockIdx.x) * (4 * NW) + tid] = sum;
  } else if (COUNT && tid < 4 * NW + 2) {
    const int c = tid - 4 * NW;
    unsigned long long sum = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) sum += s_cred[w][c];
    cpartials[static_cast<size_t>(blockIdx.x) * 2 + c] = sum * count_scale;
  }
}

// The band loop of one item: aqsntemp streamed through the per-thread
// cp.async ring, aqsmtemp / wx read from shared memory (uniform broadcasts).
template <class P, int NW, int IGP_T, bool COUNT, bool FAST>
__device__ __forceinline__ void band_loop(const double2* anp, int ncouls, int nb,
                                          double2 (&s_an)[kAnDepth][kThreads],
                                          const double2 (&s_am)[kMaxChunk][IGP_T],
                                          const double (&s_wx)[kMaxChunk][NW],
                                          const typename P::St (&st)[IGP_T], Acc<NW>& acc) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int s = 0; s < kAnDepth - 1; ++s) {
    if (s < nb) cp_async16(&s_an[s][tid], anp + static_cast<size_t>(s) * ncouls);
    cp_async_commit();
  }
  for (int bb = 0; bb < nb; ++bb) {
    const int pf = bb + kAnDepth - 1;
    if (pf < nb) cp_async16(&s_an[pf % kAnDepth][tid], anp + static_cast<size_t>(pf) * ncouls);
    cp_async_commit();
    cp_async_wait<kAnDepth - 1>();
    const double2 an = s_an[bb % kAnDepth][tid];
    double wx[NW];
#pragma unroll
    for (int iw = 0; iw < NW; ++iw) wx[iw] = s_wx[bb][iw];
#pragma unroll
    for (int j = 0; j < IGP_T; ++j) {
      const double2 am = s_am[bb][j];
      // t = an * conj(am)
      const double tr = fma(an.x, am.x, an.y * am.y);
      const double ti = fma(an.y, am.x, -an.x * am.y);
      P::template tuple<NW, COUNT, FAST>(st[j], tr, ti, wx, acc);
    }
  }
  cp_async_wait<0>();
}

template <class P, int NW, int IGP_T, bool COUNT>
__global__ void __launch_bounds__(kThreads, 2) gpp_main_kernel(const Params p) {
  __shared__ double2 s_am[kMaxChunk][IGP_T];
  __shared__ double s_wx[kMaxChunk][NW];
  __shared__ __align__(16) double2 s_an[kAnDepth][kThreads];

  Acc<NW> acc;
#pragma unroll
  for (int iw = 0; iw < NW; ++iw) {
    acc.a[iw] = make_double2(0.0, 0.0);
    acc.b[iw] = make_double2(0.0, 0.0);
  }
  acc.nn = 0;
  acc.nf = 0;

  const int tid = threadIdx.x;
  for (long long item = blockIdx.x; item < p.n_items; item += gridDim.x) {
    const int igpt = static_cast<int>(item % p.n_igptile);
    const long long rest = item / p.n_igptile;
    const int igb = static_cast<int>(rest % p.n_igblk);
    const int bc = static_cast<int>(rest / p.n_igblk);
    const int ig = (p.igblk0 + igb) * kThreads + tid;
    const bool vig = ig < p.ncouls;
    const int igc = vig ? ig : p.ncouls - 1;
    const int b0 = bc * p.bchunk;
    const int nb = min(p.bchunk, p.nbands - b0);

    typename P::St st[IGP_T];
#pragma unroll
    for (int j = 0; j < IGP_T; ++j) {
      const int igp = igpt * IGP_T + j;
      const bool v = vig && igp < p.ngpown;
      const size_t off = static_cast<size_t>(min(igp, p.ngpown - 1)) * p.ncouls + igc;
      st[j] = P::make(__ldg(p.wtilde + off), __ldg(p.eps + off), v);
    }

    // Block-uniform choice of the regular (no degenerate instance possible)
    // fast path; the barrier also orders this item's staging after the
    // previous item's shared-memory reads.
    bool thread_regular = true;
#pragma unroll
    for (int j = 0; j < IGP_T; ++j) thread_regular = thread_regular && P::regular(st[j], p.wxmax);
    const bool item_regular =
        __syncthreads_and(P::kHasFastPath && !COUNT && thread_regular) != 0;
    for (int k = tid; k < nb * IGP_T; k += kThreads) {
      const int bb = k / IGP_T, j = k - bb * IGP_T;
      const int igp = igpt * IGP_T + j;
      s_am[bb][j] = igp < p.ngpown
                        ? __ldg(p.aqsm + static_cast<size_t>(b0 + bb) * p.ngpown + igp)
                        : make_double2(0.0, 0.0);
    }
    for (int k = tid; k < nb * NW; k += kThreads) {
      const int bb = k / NW, iw = k - bb * NW;
      s_wx[bb][iw] = __ldg(p.wxb + static_cast<size_t>(b0 + bb) * p.nw_total + p.iw0 + iw);
    }
    __syncthreads();

    const double2* anp = p.aqsn + static_cast<size_t>(b0) * p.ncouls + igc;
    if (item_regular)
      band_loop<P, NW, IGP_T, COUNT, true>(anp, p.ncouls, nb, s_an, s_am, s_wx, st, acc);
    else
      band_loop<P, NW, IGP_T, COUNT, false>(anp, p.ncouls, nb, s_an, s_am, s_wx, st, acc);
  }

  block_reduce_write<NW, COUNT>(acc, p.partials, p.cpartials, 1ull);
}

// ---------------------------------------------------------------------------
// Production kernel: per-(igp, iw) band sums with the (ig, igp) constants
// applied once per item.
//
// For one (ig, igp) the near term of every instance is
//     inv (wx wt - |wt|^2) eps t = (eps wt) [inv wx t] - (eps |wt|^2) [inv t]
// and the far term sqrt(d/|wt|^2) eps t = (eps / |wt|) [sqrt(d) t], where
// only the bracketed factors change with the band.  The band loop therefore
// accumulates, per igp of the tile and per frequency,
//     S1 += (inv wx) t,   S2 += inv t,   Sf += sqrt(d) t
// and the item epilogue multiplies by eps wt, eps |wt|^2 and eps / |wt|.
// Every instance still evaluates its own d, 1/d, sqrt(d), branch decision and
// accumulation (nothing is hoisted across bands; wx may depend on the band).
// Against FastPolicy3 this drops eps*t, wt*(eps t), |wt|^2 (eps t) and
// |wt|^-1 (eps t) from every (band, igp, ig) tuple: 9 % fewer register-file
// reads per instance at nw = 3 and 21 % at nw = 2 (tools/sass_rf.py).  The
// per-thread ach/asx accumulators live in shared memory (updated once per
// item) to leave the registers to the S sums.
// ---------------------------------------------------------------------------
// Shared memory of gpp_sacc_kernel (dynamic: 88-104 KB, two CTAs per SM).
// The aqsmtemp tile and the (wtilde, eps) of the thread's ig are double
// buffered: item k+1's are copied (cp.async) while item k's bands run, and
// item k+1's first aqsntemp bands enter the ring during item k's last
// iterations, so an item boundary exposes no load latency.
template <int NW, int IGP_T>
struct SaccSmem {
  double2 an[kAnDepth][kThreads];          // aqsntemp ring, one slot per band in flight
  double2 am[2][sacc_cap<NW>()][IGP_T];    // aqsmtemp[igp tile, band chunk]
  double2 we[2][IGP_T][2][kThreads];       // [buf][j][wtilde | eps][thread]
};

struct SaccItem {
  int igpt, igb, b0, nb;
};

__device__ __forceinline__ SaccItem sacc_item(const Params& p, unsigned item) {
  SaccItem it;
  const unsigned bcu = fastdiv(item, p.rows_mul, p.rows_shift);
  const unsigned row = item - bcu * static_cast<unsigned>(p.n_rows) + static_cast<unsigned>(p.row0);
  const unsigned igb = fastdiv(row, p.igpt_mul, p.igpt_shift);
  it.igpt = static_cast<int>(row - igb * p.n_igptile);
  it.igb = static_cast<int>(igb);
  it.b0 = static_cast<int>(bcu) * p.bchunk;
  it.nb = min(p.bchunk, p.nbands - it.b0);
  return it;
}

// The canonical slot of an item (Params::slot_base).
__device__ __forceinline__ long long sacc_slot(const Params& p, unsigned item) {
  const unsigned bcu = fastdiv(item, p.rows_mul, p.rows_shift);
  const unsigned row = item - bcu * static_cast<unsigned>(p.n_rows) + static_cast<unsigned>(p.row0);
  return p.slot_base + static_cast<long long>(bcu) * p.slot_stride + row;
}

// This thread's ig for an item (clamped to a valid column for padded lanes).
__device__ __forceinline__ int sacc_igc(const Params& p, const SaccItem& it) {
  return min((p.igblk0 + it.igb) * kThreads + static_cast<int>(threadIdx.x), p.ncouls - 1);
}

// Issue (no commit) the copies of an item's aqsmtemp tile (cooperative) and of
// this thread's wtilde / eps into buffer `buf`.
template <int NW, int IGP_T>
__device__ __forceinline__ void sacc_stage(const Params& p, const SaccItem& it,
                                           SaccSmem<NW, IGP_T>& sm, int buf) {
  const int tid = threadIdx.x;
  // Thread t stages column j = t % IGP_T of bands t / IGP_T, + kThreads /
  // IGP_T, ...: a fixed igp per thread and a strided walk over the bands.
  constexpr int kStep = kThreads / IGP_T;
  const int j = tid % IGP_T, igp = it.igpt * IGP_T + j;
  if (tid < kStep * IGP_T) {
    int bb = tid / IGP_T;
    if (igp < p.ngpown) {
      const double2* src = p.aqsm + static_cast<size_t>(p.band0 + it.b0 + bb) * p.ngpown + igp;
      const size_t stride = static_cast<size_t>(kStep) * p.ngpown;
      for (; bb < it.nb; bb += kStep, src += stride) cp_async16(&sm.am[buf][bb][j], src);
    } else {
      for (; bb < it.nb; bb += kStep) sm.am[buf][bb][j] = make_double2(0.0, 0.0);
    }
  }
  const int igc = sacc_igc(p, it);
#pragma unroll
  for (int j = 0; j < IGP_T; ++j) {
    const int igp = min(it.igpt * IGP_T + j, p.ngpown - 1);
    const size_t off = static_cast<size_t>(igp) * p.ncouls + igc;
    cp_async16(&sm.we[buf][j][0][tid], p.wtilde + off);
    cp_async16(&sm.we[buf][j][1][tid], p.eps + off);
  }
}

// One band of the S-sum recurrence for all IGP_T x NW instances of this thread.
template <int NW, int IGP_T, bool COUNT, bool FAST>
__device__ __forceinline__ void sacc_band(const double2 an, const double2 (&am)[IGP_T],
                                          const double (&wx)[NW], const double (&wtr)[IGP_T],
                                          const double (&wti2)[IGP_T], const double (&qn)[IGP_T],
                                          double2 (&S1)[IGP_T][NW], double2 (&S2)[IGP_T][NW],
                                          double2 (&Sf)[IGP_T][NW], Acc<1>& cnt) {
#pragma unroll
  for (int j = 0; j < IGP_T; ++j) {
    const double tr = fma(an.x, am[j].x, an.y * am[j].y);  // t = an * conj(am)
    const double ti = fma(an.y, am[j].x, -an.x * am[j].y);
    const long long qbits = __double_as_longlong(qn[j]);
    double iwt2 = 0.0;
    if constexpr (!FAST) {
      // Padded lanes (qn = +inf) and wt = 0 get x = 0: never far.
      const double wt2 = fma(wtr[j], wtr[j], wti2[j]);
      iwt2 = (wt2 > 0.0 && qbits != 0x7FF0000000000000ll) ? 1.0 / wt2 : 0.0;
    }
#pragma unroll
    for (int iw = 0; iw < NW; ++iw) {
      const double wdre = wx[iw] - wtr[j];
      const double d = fma(wdre, wdre, wti2[j]);
      double in, gf;
      if constexpr (FAST && !COUNT) {
        // One rsqrt seed, one cubic step: 1/d = rr^2, sqrt(d) = t (1 + q).
        // MUFU.RSQ64H writes only the high word; pair it with the (dead)
        // low word of wdre instead of a zeroed register.  The low word
        // perturbs the 2^-20 seed by < 2^-20 relative, which the cubic step
        // absorbs (its error is O(e^3)).
        double r;
        asm("{\n\t.reg .b32 wl, wh, rl, rh;\n\t.reg .f64 s;\n\t"
            "mov.b64 {wl, wh}, %1;\n\t"
            "rsqrt.approx.ftz.f64 s, %2;\n\t"
            "mov.b64 {rl, rh}, s;\n\t"
            "mov.b64 %0, {wl, rh};\n\t}"
            : "=d"(r) : "d"(wdre), "d"(d));
#if GPP_ABL & 4
        r = d;  // ablation: no MUFU seed dependency
#endif
        const double t = d * r;
        const double e = fma(-t, r, 1.0);
        const double pe = fma(e, 0.375, 0.5);
        const double q = e * pe;
        const double rr = fma(r, q, r);
        const double sq = fma(t, q, t);
        const double inv = rr * rr;
        // near ? (inv, 0) : (0, sq), selecting only the HIGH words: the
        // deselected value keeps its low word, i.e. becomes a subnormal
        // below 2^-1042.  Its products vanish below half an ulp of any
        // partial sum above ~1e-290 that they join (the selected terms are
        // >= ~1e-300 unless |wx - wt| > 1e150), so the sums are unchanged
        // (tools/ab_select.sh: bitwise equal to the exact-select build); it
        // halves the selects (2 SEL instead of 4 FSEL per instance).
        asm("{\n\t.reg .pred pn;\n\t.reg .b32 il, ih, gl, gh;\n\t"
            "setp.gt.s64 pn, %2, %3;\n\t"
            "mov.b64 {il, ih}, %4;\n\t"
            "mov.b64 {gl, gh}, %5;\n\t"
            "selp.b32 ih, ih, 0, pn;\n\t"
            "selp.b32 gh, 0, gh, pn;\n\t"
            "mov.b64 %0, {il, ih};\n\t"
            "mov.b64 %1, {gl, gh};\n\t}"
            : "=d"(in), "=d"(gf)
            : "l"(__double_as_longlong(d)), "l"(qbits), "d"(inv), "d"(sq));
#if GPP_ABL & 1  // ablation: no branch selection
        in = inv;
        gf = sq;
#endif
#ifdef GPP_EXACT_SELECT  // A/B reference build (tools/ab_select.sh): full 64-bit selects
        asm("{\n\t.reg .pred pn;\n\t"
            "setp.gt.s64 pn, %2, %3;\n\t"
            "selp.f64 %0, %4, 0d0000000000000000, pn;\n\t"
            "selp.f64 %1, 0d0000000000000000, %5, pn;\n\t}"
            : "=d"(in), "=d"(gf)
            : "l"(__double_as_longlong(d)), "l"(qbits), "d"(inv), "d"(sq));
#endif
      } else {
        // General path: full far test on x = d/|wt|^2; gf = sqrt(x)
        // already carries the 1/|wt| factor.
        const double inv = rcp_refined(d);
        const double x = d * iwt2;
        const double g = sqrt_nr<3>(x);
        select_branches<COUNT>(d, qbits, x, inv, g, in, gf, cnt);
      }
      const double s1 = in * wx[iw];
      S1[j][iw].x = fma(s1, tr, S1[j][iw].x);
      S1[j][iw].y = fma(s1, ti, S1[j][iw].y);
      S2[j][iw].x = fma(in, tr, S2[j][iw].x);
      S2[j][iw].y = fma(in, ti, S2[j][iw].y);
#if !(GPP_ABL & 2)  // ablation 2: no far-branch accumulation
      Sf[j][iw].x = fma(gf, tr, Sf[j][iw].x);
      Sf[j][iw].y = fma(gf, ti, Sf[j][iw].y);
#endif
    }
  }
}

// The band loop of one item.  Ring slot of band bb: (ro + bb) % kAnDepth.
// Every iteration commits exactly one cp.async group and waits for the group
// of its own band (kAnDepth - 1 groups back), so the ring stays continuous
// across items:
//   - main phase (pf = bb + kAnDepth - 1 < nb): prefetch this item's band pf;
//   - tail phase: prefetch the NEXT item's band pf - nb into the same ring
//     (when this item has at least kAnDepth - 1 bands; a shorter item leaves
//     the next one to prime its ring itself);
//   - iteration 0's group also carries the next item's aqsmtemp tile and
//     wtilde / eps (issued just before the loop).
template <int NW, int IGP_T, bool COUNT, bool FAST>
__device__ __forceinline__ void sacc_band_loop(const Params& p, const WxTable& wxt,
                                               SaccSmem<NW, IGP_T>& sm, int buf, unsigned ro,
                                               const SaccItem& it, const double2* anp,
                                               bool has_next, const SaccItem& nx,
                                               const double (&wtr)[IGP_T],
                                               const double (&wti2)[IGP_T],
                                               const double (&qn)[IGP_T],
                                               double2 (&S1)[IGP_T][NW], double2 (&S2)[IGP_T][NW],
                                               double2 (&Sf)[IGP_T][NW], Acc<1>& cnt) {
  const int tid = threadIdx.x;
  const int nb = it.nb, wx0 = it.b0 * NW;
  const size_t ncouls = static_cast<size_t>(p.ncouls);
  const int nmain = max(nb - (kAnDepth - 1), 0);
  // Prefetch address advanced incrementally (one 64-bit add per band).
  const double2* pfp = anp + static_cast<size_t>(kAnDepth - 1) * ncouls;
  // The next item's staging joins iteration 0's commit group.
  if (has_next) sacc_stage(p, nx, sm, buf ^ 1);
  int wxo = wx0;
  // Main phase unrolled by the ring depth: the four ring slots of a round
  // are fixed per item, so no slot arithmetic in the loop.
  const int nmain4 = nmain & ~(kAnDepth - 1);
  double2* slot[kAnDepth];
#pragma unroll
  for (int k = 0; k < kAnDepth; ++k) slot[k] = &sm.an[(ro + k) % kAnDepth][tid];
  for (int b4 = 0; b4 < nmain4; b4 += kAnDepth) {
#pragma unroll
    for (int k = 0; k < kAnDepth; ++k) {
      const int bb = b4 + k;
      cp_async16(slot[(k + kAnDepth - 1) % kAnDepth], pfp);
      pfp += ncouls;
      cp_async_commit();
      cp_async_wait<kAnDepth - 1>();
      const double2 an = *slot[k];
      double wx[NW];
#pragma unroll
      for (int iw = 0; iw < NW; ++iw) wx[iw] = wxt.w[wxo + iw];
      wxo += NW;
      double2 am[IGP_T];
#pragma unroll
      for (int j = 0; j < IGP_T; ++j) am[j] = sm.am[buf][bb][j];
      sacc_band<NW, IGP_T, COUNT, FAST>(an, am, wx, wtr, wti2, qn, S1, S2, Sf, cnt);
    }
  }
  for (int bb = nmain4; bb < nmain; ++bb) {
    cp_async16(&sm.an[(ro + bb + kAnDepth - 1) % kAnDepth][tid], pfp);  // unsigned: a mask
    pfp += ncouls;
    cp_async_commit();
    cp_async_wait<kAnDepth - 1>();
    const double2 an = sm.an[(ro + bb) % kAnDepth][tid];
    double wx[NW];
#pragma unroll
    for (int iw = 0; iw < NW; ++iw) wx[iw] = wxt.w[wxo + iw];
    wxo += NW;
    double2 am[IGP_T];
#pragma unroll
    for (int j = 0; j < IGP_T; ++j) am[j] = sm.am[buf][bb][j];
    sacc_band<NW, IGP_T, COUNT, FAST>(an, am, wx, wtr, wti2, qn, S1, S2, Sf, cnt);
  }
  // The next item's column pointer is formed only here, so it is not live
  // (two registers) across the main phase.
  const double2* nx_anp =
      p.aqsn + static_cast<size_t>(p.band0 + nx.b0) * p.ncouls + sacc_igc(p, nx);
  for (int bb = nmain; bb < nb; ++bb) {
    const int pf = bb + kAnDepth - 1;
    if (pf < nb)
      cp_async16(&sm.an[(ro + pf) % kAnDepth][tid], pfp);
    else if (has_next && nb >= kAnDepth - 1 && pf - nb < nx.nb)
      cp_async16(&sm.an[(ro + pf) % kAnDepth][tid], nx_anp + static_cast<size_t>(pf - nb) * ncouls);
    pfp += ncouls;
    cp_async_commit();
    cp_async_wait<kAnDepth - 1>();
    const double2 an = sm.an[(ro + bb) % kAnDepth][tid];
    double wx[NW];
#pragma unroll
    for (int iw = 0; iw < NW; ++iw) wx[iw] = wxt.w[wx0 + bb * NW + iw];
    double2 am[IGP_T];
#pragma unroll
    for (int j = 0; j < IGP_T; ++j) am[j] = sm.am[buf][bb][j];
    sacc_band<NW, IGP_T, COUNT, FAST>(an, am, wx, wtr, wti2, qn, S1, S2, Sf, cnt);
  }
}

template <int NW, int IGP_T>
constexpr size_t sacc_smem_bytes() {
  return sizeof(SaccSmem<NW, IGP_T>);
}

// Resident CTAs per SM the production kernel is compiled for: two-igp tiles
// (and the one-frequency kernel) fit 128 registers and run two CTAs per SM;
// the 3- and 4-igp tiles at nw 2-3 take up to 255 registers and run one CTA
// (8 warps) per SM -- fewer warps, but 9-12 independent instances per warp
// and band, and the tuple / ring work amortised over more igp
// (tools/probe_variants_sweep.py: 1.6-5.5 % faster per column).
template <int NW, int IGP_T>
constexpr int sacc_min_blocks() { return (NW >= 2 && IGP_T >= 3) ? 1 : 2; }
// Register budget per instantiation: 128 for two CTAs per SM; for the
// one-CTA tiles the cap that measured fastest over the aspect-ratio sweep
// (tools/probe_variants_sweep.py over builds with GPP_R<nw><igp>): a cap
// below 255 changes ptxas's schedule (and whether wx stays on the uniform
// datapath): nw 3 / 4-igp at 240: 1.1-1.6 % faster than at 255; nw 2 /
// 3-igp at 184: 2 % faster; the others fastest at 255 (the RF model's
// predicted gains for caps on the 3-igp nw-3 tile did not materialise).
#ifndef GPP_R33
#define GPP_R33 255
#endif
#ifndef GPP_R34
#define GPP_R34 240
#endif
#ifndef GPP_R23
#define GPP_R23 184
#endif
#ifndef GPP_R24
#define GPP_R24 255
#endif
template <int NW, int IGP_T>
constexpr int sacc_maxnreg() {
  return sacc_min_blocks<NW, IGP_T>() == 2 ? 128
         : (NW == 3 && IGP_T == 3)         ? GPP_R33
         : (NW == 3 && IGP_T == 4)         ? GPP_R34
         : (NW == 2 && IGP_T == 3)         ? GPP_R23
                                           : GPP_R24;
}

template <int NW, int IGP_T, bool COUNT>
__global__ void __maxnreg__((sacc_maxnreg<NW, IGP_T>()))
    gpp_sacc_kernel(const __grid_constant__ Params p,
                                                               const __grid_constant__ WxTable wxt) {
  extern __shared__ __align__(16) unsigned char sacc_smem_raw[];
  SaccSmem<NW, IGP_T>& sm = *reinterpret_cast<SaccSmem<NW, IGP_T>*>(sacc_smem_raw);
  const int tid = threadIdx.x;
  Acc<1> cnt;
  cnt.nn = 0;
  cnt.nf = 0;

  // n_items < 2^31 (host-checked): items decompose by multiply-shift.
  const unsigned n_items = static_cast<unsigned>(p.n_items);
  unsigned item = blockIdx.x;
  // First item: stage buffer 0 (its own group).
  if (item < n_items) sacc_stage(p, sacc_item(p, item), sm, 0);
  cp_async_commit();
  int buf = 0;
  unsigned ro = 0;
  bool primed = false;  // this item's first bands are already in the ring
  bool deep = true;     // its staging group is older than the last kAnDepth - 1 groups

  while (item < n_items) {
    // Decomposed afresh from the uniform item index every iteration (not
    // carried), so the band offset stays on the uniform datapath.
    const SaccItem it = sacc_item(p, item);
    const double2* anp =
        p.aqsn + static_cast<size_t>(p.band0 + it.b0) * p.ncouls + sacc_igc(p, it);
    if (!primed) {
      // Prime the ring (first item, or after an item too short to do it).
      cp_async_wait<0>();
      ro = 0;
#pragma unroll
      for (int s = 0; s < kAnDepth - 1; ++s) {
        if (s < it.nb) cp_async16(&sm.an[s][tid], anp + static_cast<size_t>(s) * p.ncouls);
        cp_async_commit();
      }
      deep = true;
    }
    const unsigned nitem = item + gridDim.x;
    const bool has_next = nitem < n_items;
    const SaccItem nx = sacc_item(p, has_next ? nitem : item);
    const int ig = (p.igblk0 + it.igb) * kThreads + tid;
    const bool vig = ig < p.ncouls;

    // This item's staging has landed (per thread); the barrier publishes the
    // aqsmtemp tile and retires the previous item's reads of the other buffer.
    if (deep)
      cp_async_wait<kAnDepth - 1>();
    else
      cp_async_wait<0>();
    double wtr[IGP_T], wti2[IGP_T], qn[IGP_T];
    bool thread_regular = true;
#pragma unroll
    for (int j = 0; j < IGP_T; ++j) {
      const int igp = it.igpt * IGP_T + j;
      const bool v = vig && igp < p.ngpown;
      const double2 wt = sm.we[buf][j][0][tid];
      wtr[j] = wt.x;
      wti2[j] = wt.y * wt.y;
      const double wt2 = fma(wt.x, wt.x, wti2[j]);
      qn[j] = v ? fmax(0.25, 0.25 * wt2) : __longlong_as_double(0x7FF0000000000000ll);
      // Regular: no instance can be degenerate.  |delw| = |wt| / |wdiff| >=
      // |wt| / (wxmax + |wt|), which exceeds 1e-12 whenever |wt| >= 1e-11
      // wxmax -- a sqrt-free sufficient condition (the per-item prologue
      // sits on the critical path of every item).
      thread_regular = thread_regular && (!v || (wt.y != 0.0 && wt2 >= 1e-22 * p.wxmax * p.wxmax));
    }
    const bool item_regular = __syncthreads_and(!COUNT && thread_regular) != 0;

    double2 S1[IGP_T][NW], S2[IGP_T][NW], Sf[IGP_T][NW];
#pragma unroll
    for (int j = 0; j < IGP_T; ++j)
#pragma unroll
      for (int iw = 0; iw < NW; ++iw) {
        S1[j][iw] = make_double2(0.0, 0.0);
        S2[j][iw] = make_double2(0.0, 0.0);
        Sf[j][iw] = make_double2(0.0, 0.0);
      }
    if (item_regular)
      sacc_band_loop<NW, IGP_T, COUNT, true>(p, wxt, sm, buf, ro, it, anp, has_next, nx, wtr,
                                             wti2, qn, S1, S2, Sf, cnt);
    else
      sacc_band_loop<NW, IGP_T, COUNT, false>(p, wxt, sm, buf, ro, it, anp, has_next, nx, wtr,
                                              wti2, qn, S1, S2, Sf, cnt);

    // Item epilogue: apply the (ig, igp) constants once (wtilde / eps from
    // the staged buffer: no load latency here).
    double a[4 * NW];
#pragma unroll
    for (int k = 0; k < 4 * NW; ++k) a[k] = 0.0;
#pragma unroll
    for (int j = 0; j < IGP_T; ++j) {
      const int igp = it.igpt * IGP_T + j;
      const bool v = vig && igp < p.ngpown;
      const double2 wt = sm.we[buf][j][0][tid];
      const double2 e = v ? sm.we[buf][j][1][tid] : make_double2(0.0, 0.0);
      const double wt2 = fma(wt.x, wt.x, wt.y * wt.y);
      const double c1r = e.x * wt.x - e.y * wt.y, c1i = e.x * wt.y + e.y * wt.x;  // eps wt
      const double c2r = e.x * wt2, c2i = e.y * wt2;                              // eps |wt|^2
      // 1/|wt| from the rsqrt seed and two Newton steps (~1 ulp): the IEEE
      // sqrt + division would cost more than a band iteration per item.
      // Regular items have wt2 > 0.
      double rw = 1.0;
      if (item_regular) {
        const double r0 = rsqrt_approx(wt2);
        const double h = 0.5 * wt2;
        const double r1 = r0 * fma(-h * r0, r0, 1.5);
        rw = r1 * fma(-h * r1, r1, 1.5);
      }
      const double cfr = e.x * rw, cfi = e.y * rw;                                // eps / |wt|
#pragma unroll
      for (int iw = 0; iw < NW; ++iw) {
        const double2 u = S1[j][iw], w = S2[j][iw], f = Sf[j][iw];
        a[4 * iw + 0] += (c1r * u.x - c1i * u.y) - (c2r * w.x - c2i * w.y);
        a[4 * iw + 1] += (c1r * u.y + c1i * u.x) - (c2r * w.y + c2i * w.x);
        a[4 * iw + 2] += cfr * f.x - cfi * f.y;
        a[4 * iw + 3] += cfr * f.y + cfi * f.x;
      }
    }
    // This item's warp partial: xor tree over the lanes (lane 0's fixed
    // association), one row of 4 * NW doubles into the item's canonical slot.
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int k = 0; k < 4 * NW; ++k) a[k] += __shfl_xor_sync(0xffffffffu, a[k], off);
    // Lane 0 stores the row with predicated stores (no branch: a divergent
    // region inside the item loop costs the band loop its uniform-datapath
    // wx indexing).
    {
      unsigned tid_l;  // read afresh: not held across the band loop
      asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid_l));
      const unsigned leader = (tid_l & 31) == 0;
      double2* dst = reinterpret_cast<double2*>(
          p.partials + (sacc_slot(p, item) * (kThreads / 32) + (tid_l >> 5)) * (4 * NW));
#pragma unroll
      for (int k = 0; k < 2 * NW; ++k)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t"
                     "@p st.global.v2.f64 [%1], {%2, %3};\n\t}"
                     ::"r"(leader), "l"(dst + k), "d"(a[2 * k]), "d"(a[2 * k + 1]) : "memory");
    }

    if (!has_next) break;
    // The staging group (iteration 0) is older than the last kAnDepth - 1
    // groups only if the item ran at least kAnDepth bands.
    deep = it.nb >= kAnDepth;
    primed = it.nb >= kAnDepth - 1;
    ro = (ro + static_cast<unsigned>(it.nb)) % kAnDepth;
    buf ^= 1;
    item = nitem;
  }
  cp_async_wait<0>();

  if constexpr (COUNT) {
    const int lane = tid & 31, warp = tid >> 5;
    __syncthreads();
    // The aqsntemp ring is idle now: reuse it for the per-warp counts.
    unsigned long long* s_cnt = reinterpret_cast<unsigned long long*>(&sm.an[0][0]);
    unsigned long long cn = cnt.nn, cf = cnt.nf;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      cn += __shfl_xor_sync(0xffffffffu, cn, off);
      cf += __shfl_xor_sync(0xffffffffu, cf, off);
    }
    if (lane == 0) {
      s_cnt[2 * warp] = cn;
      s_cnt[2 * warp + 1] = cf;
    }
    __syncthreads();
    if (tid < 2) {  // integer counts: one atomic per CTA (order-free, exact)
      unsigned long long sum = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) sum += s_cnt[2 * w + tid];
      atomicAdd(p.cpartials + tid, sum);
    }
  }
}

// Sum the per-CTA partials in a fixed order and form achtemp/asxtemp for the
// frequency group [iw0, iw0 + NW).  out: [ach(2 nw_total) | asx(2 nw_total)],
// counts: [near, far] (accumulated over frequency groups: `first` zeroes).
template <int NW>
__global__ void __launch_bounds__(256) gpp_finalize_kernel(const double* partials,
                                                           const unsigned long long* cpartials,
                                                           int nparts, int nw_total, int iw0,
                                                           int fast, int first, int counted,
                                                           double* out,
                                                           unsigned long long* counts) {
  // One coalesced pass: thread t owns column k = t % K of the [nparts][K]
  // partials and rows t / K, t / K + L, ... (L = 256 / K lanes per column);
  // the L column sums then add in a fixed order.  Deterministic for a given
  // nparts, and a single barrier instead of one tree per column.
  constexpr int K = 4 * NW, L = 256 / K;
  __shared__ double s[L][K];
  __shared__ unsigned long long sc[128][2];
  const int tid = threadIdx.x;
  if (tid < L * K) {
    const int k = tid % K, r0 = tid / K;
    double acc = 0.0;
    for (int i = r0; i < nparts; i += L) acc += partials[static_cast<size_t>(i) * K + k];
    s[r0][k] = acc;
  }
  if (counted) {
    const int c = tid & 1, r0 = tid >> 1;
    unsigned long long acc = 0;
    for (int i = r0; i < nparts; i += 128) acc += cpartials[static_cast<size_t>(i) * 2 + c];
    sc[r0][c] = acc;
  }
  __syncthreads();
  __shared__ double s_sum[K];
  __shared__ unsigned long long s_csum[2];
  if (tid < K) {
    double v = 0.0;
    for (int r = 0; r < L; ++r) v += s[r][tid];
    s_sum[tid] = v;
  } else if (tid >= 32 && tid < 34) {
    unsigned long long v = 0;
    if (counted)
      for (int r = 0; r < 128; ++r) v += sc[r][tid - 32];
    s_csum[tid - 32] = v;
  }
  __syncthreads();
  const double* sum = s_sum;
  const unsigned long long* csum = s_csum;
  if (tid == 0) {
    for (int iw = 0; iw < NW; ++iw) {
      const double ar = sum[4 * iw + 0], ai = sum[4 * iw + 1];
      const double br = sum[4 * iw + 2], bi = sum[4 * iw + 3];
      double achr, achi, asxr, asxi;
      if (fast) {
        achr = 0.5 * ar;
        achi = 0.5 * ai;
        asxr = fma(-0.25, br, ar);
        asxi = fma(-0.25, bi, ai);
      } else {
        achr = ar;
        achi = ai;
        asxr = br;
        asxi = bi;
      }
      out[2 * (iw0 + iw) + 0] = achr;
      out[2 * (iw0 + iw) + 1] = achi;
      out[2 * nw_total + 2 * (iw0 + iw) + 0] = asxr;
      out[2 * nw_total + 2 * (iw0 + iw) + 1] = asxi;
    }
    counts[0] = (first ? 0ull : counts[0]) + csum[0];
    counts[1] = (first ? 0ull : counts[1]) + csum[1];
  }
}

// Finalize of the production kernel: sums the canonical (slot, warp) rows in
// slot order and forms achtemp / asxtemp for the frequency group [iw0, iw0 +
// NW).  Two stages in one launch: block b sums the slots [b * spb, (b + 1) *
// spb) (fixed lanes per column, fixed combine order) into stage[b]; the last
// block to finish (atomic ticket, self-resetting) sums stage[0..gridDim) in
// order and writes out / counts.  The reduction tree depends only on the slot
// count, so the result is bitwise the same for every schedule of the items.
// counts: [near, far] summed from the per-CTA integer rows (any order).
template <int NW>
__global__ void __launch_bounds__(256) gpp_slot_finalize_kernel(
    const double* __restrict__ partials, long long n_slots, int spb, double* stage,
    unsigned* ticket, const unsigned long long* cpartials, int n_cparts, int nw_total, int iw0,
    int first, int counted, double* out, unsigned long long* counts) {
  constexpr int K = 4 * NW, V = (kThreads / 32) * K, L = 256 / V, L2 = 256 / K;
  __shared__ double s_red[L][V];
  __shared__ double s_red2[L2][K];
  __shared__ double s_sum[K];
  __shared__ unsigned long long sc[128][2];
  __shared__ unsigned long long s_csum[2];
  __shared__ bool s_last;
  const int tid = threadIdx.x;
  const long long s0 = static_cast<long long>(blockIdx.x) * spb;
  const long long s1 = min(n_slots, s0 + spb);
  if (tid < L * V) {
    const int c = tid % V, l = tid / V;
    double acc = 0.0;
    for (long long sl = s0 + l; sl < s1; sl += L) acc += partials[sl * V + c];
    s_red[l][c] = acc;
  }
  __syncthreads();
  if (tid < K) {
    double v = 0.0;
    for (int l = 0; l < L; ++l)
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) v += s_red[l][w * K + tid];
    stage[static_cast<size_t>(blockIdx.x) * K + tid] = v;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicInc(ticket, gridDim.x - 1) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // Last block: the stage rows in a fixed order (L2 reads: other blocks wrote them).
  {
    const int c = tid % K, l = tid / K;
    if (l < L2) {
      double acc = 0.0;
      for (int b = l; b < static_cast<int>(gridDim.x); b += L2)
        acc += __ldcg(stage + static_cast<size_t>(b) * K + c);
      s_red2[l][c] = acc;
    }
  }
  if (counted) {
    const int c = tid & 1, r0 = tid >> 1;
    unsigned long long acc = 0;
    for (int i = r0; i < n_cparts; i += 128) acc += cpartials[static_cast<size_t>(i) * 2 + c];
    sc[r0][c] = acc;
  }
  __syncthreads();
  if (tid < K) {
    double v = 0.0;
    for (int l = 0; l < L2; ++l) v += s_red2[l][tid];
    s_sum[tid] = v;
  } else if (tid >= 32 && tid < 34) {
    unsigned long long v = 0;
    if (counted)
      for (int r = 0; r < 128; ++r) v += sc[r][tid - 32];
    s_csum[tid - 32] = v;
  }
  __syncthreads();
  if (tid == 0) {
    for (int iw = 0; iw < NW; ++iw) {
      const double ar = s_sum[4 * iw + 0], ai = s_sum[4 * iw + 1];
      const double br = s_sum[4 * iw + 2], bi = s_sum[4 * iw + 3];
      out[2 * (iw0 + iw) + 0] = 0.5 * ar;
      out[2 * (iw0 + iw) + 1] = 0.5 * ai;
      out[2 * nw_total + 2 * (iw0 + iw) + 0] = fma(-0.25, br, ar);
      out[2 * nw_total + 2 * (iw0 + iw) + 1] = fma(-0.25, bi, ai);
    }
    counts[0] = (first ? 0ull : counts[0]) + s_csum[0];
    counts[1] = (first ? 0ull : counts[1]) + s_csum[1];
  }
}

// Factored evaluation (the reference's production algorithm,
// rooflab/gpp/kernel.py:98-114), valid when wx does not depend on the band:
// the band sum is factored out of the branch terms,
//     W[ig, igp] = sum_band aqsntemp[ig, band] conj(aqsmtemp[igp, band])
// (kernel.py:108), then ach[iw] = sum sch[iw, ig, igp] W, asx likewise.
// One fused kernel: an item is (256-ig block, 8-igp tile).  The band GEMM runs
// on the FP64 tensor cores (DMMA.8x8x4, mma.sync.m8n8k4.f64): warp w owns
// ig rows [32w, 32w + 32) of the block as four 8x8 (ig x igp) tiles, and a
// complex multiply-add is four real MMAs (Wr += Ar Br + Ai Bi, Wi += Ai Br -
// Ar Bi) over 4 bands per step, fragments loaded straight from the
// column-major arrays (lane (g, q): ig row g, band q; aqsmtemp column g) with
// a one-step register prefetch.  The epilogue forms variant V's branch terms
// per (iw, ig, igp) exactly as PlainPolicy<V> does (kernel.py:63-95) for the
// 4 x 2 (ig, igp) entries of W each lane holds, and contracts them -- W never
// goes to memory.  A different algorithm from the per-instance nest (it
// exploits the band invariance of the reference's wx): time to solution,
// never a roofline figure.  Counts are scaled by nb, the band
// count W summed over (kernel.py:130-137).
constexpr int kFacIgp = 8;  // igp per item (one MMA n-tile)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int V, int NW>
__global__ void __launch_bounds__(kThreads, 2) gpp_factored_kernel(
    const double2* __restrict__ aqsn, const double2* __restrict__ aqsm,
    const double2* __restrict__ wtilde, const double2* __restrict__ eps,
    const double* __restrict__ wx0, int nw_total, int iw0, int ncouls, int ngpown, int nbands,
    int n_igptile, long long n_items, unsigned long long nb_scale, double* partials,
    unsigned long long* cpartials) {
  // This thread's ach / asx partials across its items (shared memory, so the
  // registers stay with the W fragments).
  __shared__ double s_acc[4 * NW][kThreads];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
#pragma unroll
  for (int k = 0; k < 4 * NW; ++k) s_acc[k][tid] = 0.0;
  unsigned n_near = 0, n_far = 0;
  const size_t nc = static_cast<size_t>(ncouls), ng = static_cast<size_t>(ngpown);
  for (long long item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int igpt = static_cast<int>(item % n_igptile);
    const int igb = static_cast<int>(item / n_igptile);
    const int ig_base = igb * kThreads + warp * 32;
    // A rows of this lane (clamped: rows past ncouls are masked in the epilogue).
    const double2* ap[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) ap[s] = aqsn + min(ig_base + 8 * s + g, ncouls - 1);
    const double2* bp = aqsm + min(igpt * kFacIgp + g, ngpown - 1);
    double wr[4][2], wi[4][2];
#pragma unroll
    for (int s = 0; s < 4; ++s) wr[s][0] = wr[s][1] = wi[s][0] = wi[s][1] = 0.0;
    // Band step k0: this lane's band is k0 + q (zero past nbands).  The main
    // loop runs while the prefetched step is whole (no guards); the last
    // one or two steps take the guarded path.
    const double2* pa[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) pa[s] = ap[s] + q * nc;
    const double2* pb = bp + q * ng;
    const size_t sa = 4 * nc, sb = 4 * ng;
    double2 a_cur[4], b_cur;
    {
      const bool v = q < nbands;
#pragma unroll
      for (int s = 0; s < 4; ++s) a_cur[s] = v ? __ldg(pa[s]) : make_double2(0.0, 0.0);
      b_cur = v ? __ldg(pb) : make_double2(0.0, 0.0);
    }
    int k0 = 0;
    for (; k0 + 8 <= nbands; k0 += 4) {
      double2 a_nxt[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        pa[s] += sa;
        a_nxt[s] = __ldg(pa[s]);
      }
      pb += sb;
      const double2 b_nxt = __ldg(pb);
      const double nbi = -b_cur.y;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        dmma(wr[s], a_cur[s].x, b_cur.x);   // Ar Br
        dmma(wr[s], a_cur[s].y, b_cur.y);   // + Ai Bi
        dmma(wi[s], a_cur[s].y, b_cur.x);   // Ai Br
        dmma(wi[s], a_cur[s].x, nbi);       // - Ar Bi
      }
#pragma unroll
      for (int s = 0; s < 4; ++s) a_cur[s] = a_nxt[s];
      b_cur = b_nxt;
    }
    for (; k0 < nbands; k0 += 4) {
      double2 a_nxt[4], b_nxt;
      const bool vn = k0 + 4 + q < nbands;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        pa[s] += sa;
        a_nxt[s] = vn ? __ldg(pa[s]) : make_double2(0.0, 0.0);
      }
      pb += sb;
      b_nxt = vn ? __ldg(pb) : make_double2(0.0, 0.0);
      const double nbi = -b_cur.y;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        dmma(wr[s], a_cur[s].x, b_cur.x);
        dmma(wr[s], a_cur[s].y, b_cur.y);
        dmma(wi[s], a_cur[s].y, b_cur.x);
        dmma(wi[s], a_cur[s].x, nbi);
      }
#pragma unroll
      for (int s = 0; s < 4; ++s) a_cur[s] = a_nxt[s];
      b_cur = b_nxt;
    }
    Acc<NW> acc;
#pragma unroll
    for (int iw = 0; iw < NW; ++iw) {
      acc.a[iw] = make_double2(s_acc[4 * iw + 0][tid], s_acc[4 * iw + 1][tid]);
      acc.b[iw] = make_double2(s_acc[4 * iw + 2][tid], s_acc[4 * iw + 3][tid]);
    }
    acc.nn = n_near;
    acc.nf = n_far;
    double wx[NW];
#pragma unroll
    for (int iw = 0; iw < NW; ++iw) wx[iw] = __ldg(wx0 + iw0 + iw);
    // Accumulator (s, i): ig = ig_base + 8 s + g, igp = igpt * 8 + 2 q + i.
#pragma unroll
    for (int s = 0; s < 4; ++s) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int ig = ig_base + 8 * s + g, igp = igpt * kFacIgp + 2 * q + i;
        const bool v = ig < ncouls && igp < ngpown;
        const size_t off = static_cast<size_t>(min(igp, ngpown - 1)) * nc + min(ig, ncouls - 1);
        const typename PlainPolicy<V>::St st =
            PlainPolicy<V>::make(__ldg(wtilde + off), __ldg(eps + off), v);
        PlainPolicy<V>::template tuple<NW, true, false>(st, wr[s][i], wi[s][i], wx, acc);
      }
    }
#pragma unroll
    for (int iw = 0; iw < NW; ++iw) {
      s_acc[4 * iw + 0][tid] = acc.a[iw].x;
      s_acc[4 * iw + 1][tid] = acc.a[iw].y;
      s_acc[4 * iw + 2][tid] = acc.b[iw].x;
      s_acc[4 * iw + 3][tid] = acc.b[iw].y;
    }
    n_near = acc.nn;
    n_far = acc.nf;
  }
  Acc<NW> acc;
#pragma unroll
  for (int iw = 0; iw < NW; ++iw) {
    acc.a[iw] = make_double2(s_acc[4 * iw + 0][tid], s_acc[4 * iw + 1][tid]);
    acc.b[iw] = make_double2(s_acc[4 * iw + 2][tid], s_acc[4 * iw + 3][tid]);
  }
  acc.nn = n_near;
  acc.nf = n_far;
  block_reduce_write<NW, true>(acc, partials, cpartials, nb_scale);
}

// ---------------------------------------------------------------------------
// Device-side synthesis: numpy's PCG64 (128-bit LCG, XSL-RR output) and
// Generator.uniform, bit-exact with synth_problem (rooflab/gpp/problem.py:
// 109-156).  The host passes the generator state after seeding; every thread
// jumps to its first draw with the O(log n) LCG advance and then steps.
// ---------------------------------------------------------------------------
struct U128 {
  unsigned long long lo, hi;
};
__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}
__device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}
constexpr unsigned long long kPcgMulHi = 0x2360ED051FC65DA4ull;
constexpr unsigned long long kPcgMulLo = 0x4385DF649FCCF645ull;

// state after `delta` further steps (pcg_advance_lcg_128).
__device__ __forceinline__ U128 pcg_advance(U128 state, U128 inc, unsigned long long delta) {
  U128 acc_mult{1ull, 0ull}, acc_plus{0ull, 0ull};
  U128 cur_mult{kPcgMulLo, kPcgMulHi}, cur_plus = inc;
  while (delta) {
    if (delta & 1ull) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, U128{1ull, 0ull}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  return add128(mul128(acc_mult, state), acc_plus);
}

// One draw: step, XSL-RR output, 53-bit double in [0, 1).
__device__ __forceinline__ double pcg_next_double(U128& state, U128 inc) {
  state = add128(mul128(state, U128{kPcgMulLo, kPcgMulHi}), inc);
  const unsigned long long x = state.hi ^ state.lo;
  const unsigned rot = static_cast<unsigned>(state.hi >> 58);
  const unsigned long long out = (x >> rot) | (x << ((64u - rot) & 63u));
  return static_cast<double>(out >> 11) * (1.0 / 9007199254740992.0);
}

// Fill one real or imaginary component of an F-order complex matrix whose
// draws are laid out C-order over (rows, cols) starting at draw `offset`;
// only columns [c0, c1) are produced, at dst[(i + (c - c0) * rows)].  Thread
// i owns row i: one jump, then sequential steps along its row, so for a
// fixed column the warp writes consecutive rows (coalesced).
__global__ void __launch_bounds__(256) gpp_synth_kernel(U128 state0, U128 inc,
                                                        unsigned long long offset, long long rows,
                                                        long long cols, long long c0, long long c1,
                                                        double* dst, int comp) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    U128 s = pcg_advance(state0, inc, offset + static_cast<unsigned long long>(i * cols + c0));
    for (long long c = c0; c < c1; ++c) {
      const double u = pcg_next_double(s, inc);
      dst[2 * (i + (c - c0) * rows) + comp] = fma(2.0, u, -1.0);  // uniform(-1, 1)
    }
  }
}

// variant_terms (rooflab/gpp/kernel.py:63-95) on the device: per (iw, ig,
// igp) the branch terms sch, ssx and the decision masks of variant V, laid
// out (nw, ncouls, ngpown) in C order as the reference returns them.
// wtilde/eps are F-order (ig fastest), so element (ig, igp) = e % nc, e / nc.
template <int V>
__global__ void __launch_bounds__(kThreads) gpp_variant_terms_kernel(
    const double2* __restrict__ wtilde, const double2* __restrict__ eps,
    const double* __restrict__ wx0, int nw, long long ncouls, long long ngpown, double2* sch,
    double2* ssx, unsigned char* near_out, unsigned char* far_out) {
  const long long n_el = ncouls * ngpown;
  for (long long e = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x; e < n_el;
       e += static_cast<long long>(gridDim.x) * kThreads) {
    const long long ig = e % ncouls, igp = e / ncouls;
    const typename PlainPolicy<V>::St st = PlainPolicy<V>::make(__ldg(wtilde + e), __ldg(eps + e), true);
    for (int iw = 0; iw < nw; ++iw) {
      // One instance with t = 1: acc.a = sch, acc.b = ssx.
      Acc<1> acc;
      acc.a[0] = make_double2(0.0, 0.0);
      acc.b[0] = make_double2(0.0, 0.0);
      acc.nn = 0;
      acc.nf = 0;
      const double wx[1] = {__ldg(wx0 + iw)};
      PlainPolicy<V>::template tuple<1, true, false>(st, 1.0, 0.0, wx, acc);
      const long long o = (static_cast<long long>(iw) * ncouls + ig) * ngpown + igp;
      sch[o] = acc.a[0];
      ssx[o] = acc.b[0];
      near_out[o] = static_cast<unsigned char>(acc.nn);
      far_out[o] = static_cast<unsigned char>(acc.nf);
    }
  }
}

// FP64 pipe peak: 8 independent DFMA chains per thread, a = a * a + c.
// One register operand per DFMA keeps the operand collector out of the way
// (a DFMA with three distinct register operands runs at 2/3 rate on B200,
// measured by tools/fp64_issue_probe.cu), so this measures the FP64 pipe.
__global__ void __launch_bounds__(256) fp64_peak_kernel(double* sink, int iters, double b,
                                                        double c) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = (threadIdx.x * 1e-3 + k) * b * 1e-4;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], a[k], c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1.2345e300) sink[threadIdx.x] = s;  // never true; defeats DCE
}

}  // namespace gpp
