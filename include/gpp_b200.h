/*
 * gpp_b200.h -- C ABI of the B200-native GPP self-energy library
 * (libgpp_b200.so, built from paper_2008_11326_b200/csrc/).
 *
 * The reference (`rooflab`, pure Python) has no FFI: its drop-in seam is the
 * Python function
 *     evaluate_variant(problem: GPPProblem, variant: str) -> GPPResult
 *         rooflab/gpp/kernel.py:98-114
 * called by run_version (rooflab/gpp/runner.py:249-286), with the oracle
 * reference_result (rooflab/gpp/problem.py:179-208) and the branch
 * statistics branch_stats (rooflab/gpp/kernel.py:130-137) beside it.
 * This header is the boundary those calls cross on the B200 path; the
 * ctypes shim paper_2008_11326_b200/_lib.py binds every entry point below,
 * and INTEGRATION.md shows the binding a rooflab maintainer would add.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Complex arrays are interleaved
 *     (re, im) float64, column-major (Fortran order) exactly as numpy holds
 *     the reference's GPPProblem arrays (problem.py:50-61).
 *   - Every int-returning call returns a GPP_* status; on failure
 *     gpp_last_error() returns a thread-local message.
 *   - Host input buffers are borrowed for the duration of the call only and
 *     never written.  Outputs go to caller-allocated host buffers.
 *   - Distinct contexts may be used concurrently (the reference allows
 *     concurrent independent runs); calls on one shared context
 *     are serialised by a per-context lock.
 *   - Reproducible: every evaluation of the same inputs and variant returns
 *     the same bits, whichever entry point (gpp_evaluate_host's pipelined
 *     first call, gpp_run on the resident problem, any slab count) -- the
 *     production kernel runs a canonical item schedule and its finalize sums
 *     the items in a fixed order.
 *   - With a communicator attached, an error aborts it (ncclCommAbort), so
 *     peers fail (GPP_ERR_NCCL) instead of waiting on a collective; waits
 *     poll ncclCommGetAsyncError and time out after GPP_NCCL_TIMEOUT_S.
 *   - There is no CPU fallback: without a working CUDA device every compute
 *     entry point fails with GPP_ERR_CUDA.
 */
#ifndef GPP_B200_H
#define GPP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GPP_ABI_VERSION 1

/* Status codes.  The shim raises GPP_ERR_ARG as DomainError and the others as
 * GPUError; both derive from RooflabError (rooflab/errors.py:8-21), so the
 * reference CLI's exit-1 mapping (rooflab/cli.py:341-343) is preserved. */
#define GPP_OK 0
#define GPP_ERR_ARG 1
#define GPP_ERR_CUDA 2
#define GPP_ERR_NCCL 3
#define GPP_ERR_OOM 4

/* Arithmetic variants, rooflab/gpp/kernel.py:30 VARIANTS = (div, rcp, rcp_sq).
 * DIV and RCP evaluate the per-instance formulas as the reference writes them
 * (kernel.py:68-95, IEEE division and sqrt); RCP_SQ is the optimised
 * squared-magnitude / reciprocal-multiply kernel (the paper's v8). */
#define GPP_VARIANT_DIV 0
#define GPP_VARIANT_RCP 1
#define GPP_VARIANT_RCP_SQ 2

/* Intermediate rcp_sq kernels of the B200 version ladder (the paper's
 * optimisation steps re-derived, rooflab/gpp/runner.py:75-115); same results
 * as GPP_VARIANT_RCP_SQ, kept so each step can be measured:
 *   SQ_SPLIT  squared-magnitude predicates as integer compares, separate
 *             MUFU seeds for 1/d and sqrt, per-instance y    (paper v3-v4)
 *   IW_HOIST  eps*t, wt*(eps*t), |wt|^2 (eps*t) formed once per (band, igp,
 *             ig) and reused across frequencies              (paper v5-v6)
 *   ONE_SEED  one rsqrt seed for 1/d and sqrt(d), regular-item fast path
 *             (far == !near)                                  (paper v7)
 * GPP_VARIANT_RCP_SQ is the final kernel: per-(igp, iw) band sums, the
 * (ig, igp) constants applied once per item (paper v8). */
#define GPP_KERNEL_SQ_SPLIT 3
#define GPP_KERNEL_IW_HOIST 4
#define GPP_KERNEL_ONE_SEED 5

typedef struct gpp_ctx gpp_ctx;

/* ABI revision (GPP_ABI_VERSION) of the loaded library. */
int gpp_abi_version(void);

/* Thread-local message describing the last failure on this thread. */
const char* gpp_last_error(void);

/* Number of visible CUDA devices. */
int gpp_device_count(int* count);

/* Create a context bound to one CUDA device.  Lazy: no CUDA call is made
 * until the first upload, so argument validation works without a GPU. */
int gpp_create(gpp_ctx** ctx, int device);
void gpp_destroy(gpp_ctx* ctx);

/* Copy one problem (or the band shard [band0, band1) of it) to the device.
 * An empty shard (band0 == band1, e.g. more ranks than bands) is allowed: it
 * contributes zeros and still joins the collectives.
 * Replaces the array hand-off into evaluate_variant (kernel.py:98) and the
 * GPPProblem fields (problem.py:50-71).
 *   wtilde, i_eps : (ncouls, ngpown) complex, F-order  -> 2*ncouls*ngpown doubles
 *   aqsntemp      : (ncouls, nbands) complex, F-order  (whole array; only the
 *                   shard's columns are copied)
 *   aqsmtemp      : (ngpown, nbands) complex, F-order  (whole array)
 *   wx            : nw doubles (wx_band_indexed == 0, the reference's (NW,)
 *                   vector, problem.py:70), or an (nw, nbands) F-order array
 *                   (wx_band_indexed != 0, BerkeleyGW's wx_array(iw, n1)).
 * The device always stores wx band-indexed, so the kernel evaluates every
 * (band, igp, ig, iw) instance (no band-invariance shortcut).
 * nw may be any value >= 1; the library processes it in groups of <= 4. */
int gpp_upload(gpp_ctx* ctx, int64_t nbands, int64_t ngpown, int64_t ncouls, int32_t nw,
               const double* wtilde, const double* i_eps, const double* aqsntemp,
               const double* aqsmtemp, const double* wx, int32_t wx_band_indexed,
               int64_t band0, int64_t band1);

/* Evaluate the uploaded problem.  Replaces evaluate_variant (kernel.py:98-114)
 * and, through near_far, branch_stats (kernel.py:130-137).
 *   achtemp, asxtemp : 2*nw doubles each (complex, interleaved)
 *   near_far         : nullable; receives [near, far] instance counts over
 *                      the evaluated (band, igp, ig, iw) instances
 *   kernel_ms        : nullable; device time of the compute kernels (CUDA
 *                      events), excluding the collective and the D2H copy
 * With a communicator attached (gpp_comm_init) the per-rank partial sums and
 * counts are combined with ncclAllReduce before they are returned. */
int gpp_run(gpp_ctx* ctx, int32_t variant, double* achtemp, double* asxtemp,
            int64_t* near_far, float* kernel_ms);

/* Synthesize the problem on the device instead of uploading it: the arrays
 * synth_problem(nbands, ngpown, ncouls, seed, nw) draws (rooflab/gpp/
 * problem.py:109-156, numpy PCG64 + Generator.uniform), bit-exact, for the
 * band shard [band0, band1).  pcg_state = {state.lo, state.hi, inc.lo,
 * inc.hi} of np.random.default_rng(seed) right after seeding; wx = the nw
 * frequencies (drawn on the host, they are the last nw draws).  The
 * branch-margin scan (problem.py:159-176) is not run. */
int gpp_synth(gpp_ctx* ctx, int64_t nbands, int64_t ngpown, int64_t ncouls, int32_t nw,
              const uint64_t* pcg_state, const double* wx, int64_t band0, int64_t band1);

/* Upload + evaluate in one call, with the host->device copy pipelined
 * against the computation: the ig rows of wtilde / i_eps / aqsntemp are
 * copied in ig slabs on a copy stream, and the kernel for slab s starts as
 * soon as its rows have landed, while slab s+1 is in flight.  `slabs` > 0:
 * that many equal slabs; <= 0: slabs tapering towards single 256-ig blocks
 * at the end, so that little computation follows the last copy.  Arguments as gpp_upload + gpp_run; `ms` (nullable) receives the
 * device time from the first copy to the end of the computation.  Host
 * arrays should be page-locked (gpp_host_register) for the copies to be
 * asynchronous.  Afterwards the problem is resident, as after gpp_upload.
 * This is the end-to-end path of evaluate_variant on a problem that is not
 * yet on the device (kernel.py:98-114). */
int gpp_evaluate_host(gpp_ctx* ctx, int32_t variant, int64_t nbands, int64_t ngpown,
                      int64_t ncouls, int32_t nw, const double* wtilde, const double* i_eps,
                      const double* aqsntemp, const double* aqsmtemp, const double* wx,
                      int32_t wx_band_indexed, int64_t band0, int64_t band1, int32_t slabs,
                      double* achtemp, double* asxtemp, int64_t* near_far, float* ms);

/* Factored evaluation of the uploaded problem: the reference's own
 * production algorithm (rooflab/gpp/kernel.py:98-114) -- the band sum
 * W = aqsntemp conj(aqsmtemp)^T and the contraction of the variant's branch
 * terms per (iw, ig, igp) with W, fused in one hand-written FP64 kernel
 * (gpp_factored_kernel: the GEMM on the DMMA tensor cores, W stays in registers).  Only valid for a band-invariant
 * wx (GPP_ERR_ARG otherwise).  A different algorithm from the per-instance
 * nest gpp_run evaluates: time to solution, not a roofline figure.  With a
 * communicator attached the partials are all-reduced as in gpp_run. */
int gpp_run_factored(gpp_ctx* ctx, int32_t variant, double* achtemp, double* asxtemp,
                     int64_t* near_far, float* ms);

/* variant_terms (rooflab/gpp/kernel.py:63-95) of the uploaded problem: the
 * per-(iw, ig, igp) branch terms sch, ssx (complex, interleaved) and the
 * near / far decision masks (0/1 bytes), C-order (nw, ncouls, ngpown) as the
 * reference returns them.  Band-invariant wx only (GPP_ERR_ARG otherwise). */
int gpp_variant_terms(gpp_ctx* ctx, int32_t variant, double* sch, double* ssx, uint8_t* near_mask,
                      uint8_t* far_mask);

/* Device-resident timing: `iters` back-to-back evaluations on the context's
 * stream (compute kernels + finalize + allreduce when attached, no host
 * copies).  total_ms = event time of the whole run; main_ms = summed event
 * time of the main reduction kernel launches alone. */
int gpp_time(gpp_ctx* ctx, int32_t variant, int32_t iters, float* total_ms, float* main_ms);

/* Launch shape of the main kernel for the uploaded problem. */
int gpp_kernel_info(gpp_ctx* ctx, int32_t variant, int32_t* registers_per_thread,
                    int32_t* threads_per_block, int32_t* blocks_per_sm, int32_t* grid,
                    int32_t* igp_tile, int32_t* band_chunk);

/* The production kernel's canonical launch schedule for a whole (unsharded,
 * un-slabbed) evaluation of the first frequency group on a GPU with `sms`
 * SMs: pure host logic, no device needed.  Each launch is 7 values: row0,
 * n_rows (rows of (256-ig block, igp tile) pairs), band0, nbands (its band
 * window), bchunk (bands per item), n_items (items = chunk * n_rows + row -
 * row0, the first n_items of them) and the igp tile (2-4 igp per thread, the
 * tile of least padded cost for ngpown; 1 or 2 resident CTAs per SM).
 * Writes at most max_launches entries; *n_launches is the full count. */
int gpp_plan(int64_t nbands, int64_t ngpown, int64_t ncouls, int32_t nw, int32_t sms,
             int32_t max_launches, int32_t* n_launches, int64_t* launches);

/* The production kernel's launches for one ig slab (256-ig blocks [blk0,
 * blk1)) of the pipelined evaluate: the canonical items of gpp_plan whose rows
 * lie in the slab, as sub-launches of 9 values each -- row0, n_rows, band0,
 * nbands, bchunk, n_items, igp tile, slot_base, slot_stride; item k runs rows
 * row0 + k % n_rows, band chunk k / n_rows, and writes canonical slot
 * slot_base + chunk * slot_stride + row.  Pure host logic: the CPU tests
 * check that any slab partition runs exactly the canonical items, each into
 * its canonical slot (the basis of the bitwise reproducibility). */
int gpp_plan_piece(int64_t nbands, int64_t ngpown, int64_t ncouls, int32_t nw, int32_t sms,
                   int32_t blk0, int32_t blk1, int32_t max_launches, int32_t* n_launches,
                   int64_t* launches);

/* Number of kernels this context has launched so far (every compute,
 * finalize, synthesis and factored-path launch): the bench's gpu_launches is
 * the difference across its timed region. */
int gpp_launch_count(gpp_ctx* ctx, int64_t* launches);

/* NCCL plumbing for band sharding across ranks (one process per GPU).
 * The unique id (128 bytes) is created on rank 0 and broadcast by the host
 * (torch.distributed in the Python driver). */
int gpp_comm_unique_id(unsigned char* id128);
int gpp_comm_init(gpp_ctx* ctx, int nranks, int rank, const unsigned char* id128);

/* Single-process multi-GPU (the survey's ncclCommInitAll design): one
 * context per device in ONE process, all in one NCCL clique.  Upload each
 * context's band shard with gpp_upload(..., band0, band1), then
 * gpp_run_group evaluates every shard, combines the partials with one grouped
 * ncclAllReduce and returns the totals (kernel_ms = slowest device). */
int gpp_comm_init_all(gpp_ctx** ctxs, int n);
int gpp_run_group(gpp_ctx** ctxs, int n, int32_t variant, double* achtemp, double* asxtemp,
                  int64_t* near_far, float* kernel_ms);

/* Device-resident timing of the single-process group: `iters` evaluations
 * enqueued back to back on every device, each followed by one grouped
 * ncclAllReduce of the partials, with no host synchronisation in between.
 * total_ms / main_ms: the slowest device's event time of the whole run / of
 * its summed main-kernel spans (the bench's N-GPU timing without torchrun). */
int gpp_time_group(gpp_ctx** ctxs, int n, int32_t variant, int32_t iters, float* total_ms,
                   float* main_ms);

/* Page-lock an existing host buffer so uploads from it run at DMA speed.
 * (Not required: pageable inputs are packed into the library's pinned
 * staging ring by host threads, overlapped with the DMA.) */
int gpp_host_register(void* ptr, size_t bytes);
int gpp_host_unregister(void* ptr);

/* FP64 (DFMA) pipe microbenchmark: independent FMA chains on every SM.
 * Returns the achieved FP64 TFLOP/s (2 flops per DFMA) and the device time. */
int gpp_fp64_peak(int device, int32_t iters, double* tflops, float* ms);

#ifdef __cplusplus
}
#endif

#endif /* GPP_B200_H */
