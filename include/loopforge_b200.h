/*
 * loopforge_b200.h -- C ABI of the B200 executor for Fortran-ingested,
 * transformed loopforge kernels.
 *
 * The reference has no plugin/operator registry; its two
 * execution boundaries are
 *   (1) interpret(kernel, env) -> env
 *       /root/reference/pkg/src/loopforge/interp.py:323-400, and
 *   (2) the C function emitted by emit(kernel, "c") and called by the test
 *       harness  /root/reference/pkg/src/loopforge/codegen.py:511-527
 *       (signature) and /root/reference/pkg/tests/c_oracle.py:59-74 (call).
 * Each entry point below replaces one emitted function: the leading
 * arguments are exactly the emitted-C parameters (kernel.args in declaration
 * order -- arrays as pointers, const iff not an output, scalars by value --
 * then the remaining integer parameters sorted by name, codegen.py:511-527),
 * except that pointers are DEVICE pointers.  Two arguments are appended: the
 * logical launch geometry derived from the kernel's g.N/l.N tags and the
 * CUDA stream to launch on.
 *
 * Conventions
 *   - Every entry returns LFB_OK (0) or an LFB_ERR_* code; the text of the
 *     last error on the calling thread is available from lfb_last_error().
 *     LFB_ERR_UNSUPPORTED maps to loopforge.errors.CodegenError
 *     (codegen.py:470-472, 574-577), LFB_ERR_LAUNCH / LFB_ERR_ARG to
 *     InterpError (interp.py:103-112).
 *   - Launches are asynchronous and stream ordered; nothing synchronises.
 *   - The caller owns all device memory; no entry allocates or frees caller
 *     buffers.  Scratch (the SEM norm partials) is caller provided.
 *   - Index arithmetic inside kernels is 64-bit (the emitted C uses int and
 *     overflows past 2^31 elements, SURVEY.md §7 hard part 2).
 *   - geom->variant 0 results are bitwise identical to the reference's
 *     execution of the same kernel for fill, axpy and semlap; matvec's
 *     default (split-j) and semlap variants 50/51/61 (fused multiply-adds)
 *     are within the north star's fp64 bound (1e-12 relative), matvec
 *     variants 1/3 bitwise; sgemm / dgemm tensor-core paths are within the
 *     fp32 / fp64 tolerances, their variant 1 bitwise.
 */
#ifndef LOOPFORGE_B200_H
#define LOOPFORGE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LFB_ABI_VERSION 1

enum {
    LFB_OK = 0,
    LFB_ERR_UNSUPPORTED = 1, /* -> CodegenError */
    LFB_ERR_LAUNCH = 2,      /* -> InterpError  */
    LFB_ERR_ARG = 3          /* -> InterpError  */
};

/* cudaStream_t without pulling in the CUDA headers. */
typedef struct CUstream_st *lfb_stream;

/* Logical launch geometry (paper_1503_07659_b200/launch.py), i.e. what the
 * reference's OpenCL prologue would index with get_group_id/get_local_id
 * (codegen.py:580-612).  A NULL geometry means "untransformed kernel": the
 * executor picks its own decomposition. */
typedef struct lfb_launch {
    int32_t abi_version;      /* must be LFB_ABI_VERSION                    */
    int32_t guard;            /* 1 iff the reference emits an OpenCL guard   */
    int64_t group_extent[3];  /* extents of the g.0..g.2 inames; 0 in
                                 group_extent[0] = no parallel tags
                                 (untransformed kernel): the executor
                                 chooses the decomposition               */
    int32_t local_extent[3];  /* extents of the l.0..l.2 inames              */
    int32_t npts;             /* semlap: points per direction (order + 1)    */
    int32_t sm_count;         /* 0: query the device                         */
    int32_t ctas_per_sm;      /* 0: kernel default                           */
    int32_t variant;          /* 0: default kernel variant                   */
    int32_t reserved;
    double *sumsq;            /* semlap: if non-NULL receives sum(w*w)       */
    double *workspace;        /* semlap: >= lfb_semlap_workspace() doubles   */
    int64_t workspace_len;
} lfb_launch;

int lfb_abi_version(void);
const char *lfb_last_error(void);
/* SMs of the current device (148 on B200), or -1. */
int lfb_device_sm_count(void);

/* fill: out[i] = a                      emitted: void fill(double *out, double a, int n)
 * reference: tests/test_fortran.py:13-27, tests/test_codegen.py:217-234   */
int lfb_fill_f64(double *out, double a, int n,
                 const lfb_launch *geom, lfb_stream stream);
int lfb_fill_f32(float *out, float a, int n,
                 const lfb_launch *geom, lfb_stream stream);

/* axpy: y[i] = y[i] + alpha*x[i]        emitted: void axpy(double *y, double const *x, double alpha, int n)
 * reference: SURVEY.md Appendix B                                         */
int lfb_axpy_f64(double *y, const double *x, double alpha, int n,
                 const lfb_launch *geom, lfb_stream stream);
int lfb_axpy_f32(float *y, const float *x, float alpha, int n,
                 const lfb_launch *geom, lfb_stream stream);

/* matvec: y[i] = sum_j a[i + n*j]*x[j], sequential j, s starts at 0
 *                                       emitted: void matvec(double *y, double const *a, double const *x, int n)
 * reference: SURVEY.md Appendix B (extract_subst + precompute on x)
 * geom->variant: 0 split-j (4 column parts summed in order; fp64 within
 * 1e-12) when n >= 256, 1 bitwise direct loads, 2 split-j only, 3 bitwise
 * TMA kernel                                                              */
int lfb_matvec_f64(double *y, const double *a, const double *x, int n,
                   const lfb_launch *geom, lfb_stream stream);

/* semlap: tensor-product SEM Laplacian, geom->npts points per direction
 *                                       emitted: void semlap(double *w, double const *u, double const *d, double const *g, int nelt)
 * reference: SURVEY.md Appendix A; layouts u,w (n,n,n,nelt) strides
 * (1,n,n^2,n^3), d (n,n) strides (1,n), g (6,n,n,n,nelt) strides
 * (1,6,6n,6n^2,6n^3) -- fortran.py:638-658 column-major lowering.
 * geom->variant: 0 bitwise (the tuned kernel per order), 50 DFMA mode
 * (fp64 within 1e-12 per point), 51 FP64 tensor cores (DMMA, n = 9..16),
 * 60 / 61 two columns per thread (bitwise / DFMA, n = 7, 9..12), other
 * numbers: tuning alternatives (tests/test_gpu_parity.py)               */
int lfb_semlap_f64(double *w, const double *u, const double *d,
                   const double *g, int nelt,
                   const lfb_launch *geom, lfb_stream stream);
/* doubles of workspace lfb_semlap_f64 needs when geom->sumsq != NULL */
int64_t lfb_semlap_workspace(int npts, int nelt, const lfb_launch *geom);

/* dssum: SEM direct-stiffness summation Q Q^T on element-local w (the
 * semlap layout) over a structured box of ex x ey x ez elements of n points
 * per direction -- SURVEY.md §8(f) row 4, not a reference entry point (the
 * reference operator is element-local, interp.py:385-399; this is the
 * assembly step an SEM solver applies after it).  Global nodes with
 * zlo <= Z <= zhi (Z = ez_elem (n-1) + k).  mode 0: every node shared by
 * 2/4/8 elements gets the sum of its copies, formed left to right in
 * ascending element order; 1: that sum into plane_out[X + (ex(n-1)+1) Y],
 * no write-back (a rank's top interface plane); 2: start from plane_in, add
 * the copies, write back and into plane_out (the upper rank of an
 * interface); 3: write plane_in into the copies.  Modes 1-3 take one
 * element plane (zlo == zhi, a multiple of n-1).  Deterministic; bitwise
 * the single-domain result when the ranks chain modes 1 -> 2 -> 3.  Bits
 * 4 and up of mode select a kernel variant (tuning; 0 = the default, every
 * variant bitwise equal). */
int lfb_dssum_f64(double *w, int n, int ex, int ey, int ez, int zlo,
                  int zhi, int mode, const double *plane_in,
                  double *plane_out, lfb_stream stream);

/* sgemm: c[i,j] = c[i,j] + alpha*b[k,j]*a[i,k] over ascending k, all
 * column major: a (m,l), b (l,n), c (m,n)
 *                                       emitted: void sgemm(float alpha, float const *a, float const *b, float *c, int l, int m, int n)
 * reference: tests/test_fortran.py:72-103 (real*4 variant)                */
int lfb_sgemm_f32(float alpha, const float *a, const float *b, float *c,
                  int l, int m, int n,
                  const lfb_launch *geom, lfb_stream stream);
/* doubles of workspace the tensor-core sgemm needs (tf32 hi/lo operand
 * split, geom->workspace); 0 if the shape cannot use tensor cores
 * (m % 128, n % 256, l % 32 != 0).  geom->variant: 0 tensor cores when
 * possible else the bit-exact CUDA-core kernel, 1 bit-exact, 2 tensor only */
int64_t lfb_sgemm_workspace(int l, int m, int n);

/* dgemm: the same kernel in real*8 -- the reference's own DGEMM test
 * (tests/test_fortran.py:72-103)
 * emitted (codegen.py:511-527: kernel.args in declaration order, then the
 * remaining params sorted by name):
 *   void dgemm(double alpha, double const *a, double const *b, double *c,
 *              int l, int m, int n)
 * -- the same order as this entry.  geom->variant: 0 the FP64
 * tensor cores (DMMA; tolerance parity, fp64 within 1e-12) when m % 128,
 * n % 128, l % 16 == 0 and a, b are 16-byte aligned, else the bit-exact
 * CUDA-core kernel; 1 bit-exact; 2 tensor cores only                     */
int lfb_dgemm_f64(double alpha, const double *a, const double *b, double *c,
                  int l, int m, int n,
                  const lfb_launch *geom, lfb_stream stream);

/* Generic path: CUDA C++ generated from a kernel's
 * schedule by paper_1503_07659_b200/cudagen.py -- g.N -> blockIdx, l.N ->
 * threadIdx, workgroup temporaries -> __shared__ with real barriers -- the
 * executable counterpart of the OpenCL text the reference only prints
 * (codegen.py:580-612, 707-710).  Compiled for sm_100a by NVRTC (dlopen'ed),
 * loaded and launched through the driver API.
 *
 * lfb_rtc_compile: cubin == NULL queries the size into *cubin_len; otherwise
 * writes at most *cubin_len bytes.  Compiler diagnostics -> lfb_last_error. */
typedef struct lfb_module_st *lfb_module;
int lfb_rtc_compile(const char *src, const char *prog_name,
                    const char *const *opts, int nopts, void *cubin,
                    int64_t *cubin_len);
int lfb_module_load(const void *cubin, int64_t len, const char *kernel_name,
                    lfb_module *out);
/* grid/block: 3 extents each (the g.N / l.N extents); args: cuLaunchKernel
 * argument pointers in the generated kernel's parameter order. */
int lfb_module_launch(lfb_module m, const int64_t *grid, const int32_t *block,
                      int32_t smem, void **args, lfb_stream stream);
int lfb_module_unload(lfb_module m);
/* Tensor map (TMA descriptor, 128 bytes into *map) for a precompute
 * footprint of a column-major argument array (transforms.py:669-674 gives the
 * box): dtype 0 f64, 1 f32, 2 i32; dims[rank] extents (dim 0 contiguous),
 * strides_bytes[rank-1] for dims 1.., box[rank], swizzle 0/32/64/128.
 * LFB_ERR_UNSUPPORTED when the array violates the tensor-map rules (16-B
 * aligned base and strides); the generated kernel then fetches
 * cooperatively. */
int lfb_tmap_encode(void *map, int dtype, int rank, const int64_t *dims,
                    const int64_t *strides_bytes, const int32_t *box,
                    int swizzle_bytes, const void *base);

/* Microbenchmark used by bench.py to state the FP64 issue ceiling the SEM
 * kernel runs against: iters x 8 independent DMUL+DADD chains per thread. */
int lfb_probe_fp64(double *out, int iters, int blocks, int threads,
                   lfb_stream stream);
/* The SEM kernel's HBM access mix without its arithmetic (read u + 6 g,
 * write w per point): the streaming ceiling at a given footprint. */
int lfb_probe_stream(double *w, const double *u, const double *g,
                     int64_t npoints, lfb_stream stream);

#ifdef __cplusplus
}
#endif

#endif /* LOOPFORGE_B200_H */
