/*
 * tnc.h -- C ABI of the B200 tensor-network contraction engine (libtnc.so).
 *
 * Drop-in boundary for the amplitude-evaluation path of the reference
 * package `tnsim` (arXiv 2011.02621, /root/reference/pkg/src/tnsim):
 *
 *   tnc_contract_pair   replaces tnsim.tensor.contract_pair
 *                       (pkg/src/tnsim/tensor.py:100-115), batched over a
 *                       bitstring axis, optional conjugation of b (used by the
 *                       per-node overlap of network.py:109-122).
 *   tnc_project         replaces the per-node physical contraction of
 *                       build_overlap_network (network.py:95-126) for
 *                       product-state bras -- a gather of the projected
 *                       variant -- fused with slice_network's cut-leg
 *                       restriction (network.py:218-243) and a leg permutation.
 *   tnc_step            one Contract(C^{i1..im}, C^{im+1}) of
 *                       contract_along_path (network.py:246-268), batched over
 *                       (bitstring x slice).
 *   tnc_slice_sum       the slice loop's sum (network.py:334-339).
 *   tnc_contract_path   a whole planned path: project, every step, slice sum
 *                       (compute_amplitude's contraction, network.py:294-344).
 *
 * All pointers are CUDA device pointers unless stated; `stream` is a
 * cudaStream_t passed as void*.  Complex numbers are interleaved (re, im)
 * pairs of float (TNC_C64) or double (TNC_C128).  Every call returns 0 on
 * success or a negative TNC_E* code; tnc_last_error() describes the last
 * failure on the calling thread.  No entry point falls back to the host.
 */
#ifndef TNC_H_
#define TNC_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TNC_C64  0
#define TNC_C128 1

#define TNC_OK              0
#define TNC_E_INVALID      -1   /* bad descriptor / argument                 */
#define TNC_E_CUDA         -2   /* CUDA launch or runtime failure            */
#define TNC_E_UNSUPPORTED  -3   /* shape outside every kernel's envelope     */
#define TNC_E_NODEVICE     -4   /* no sm_100 device visible                  */

#define TNC_MAX_LEGS 40        /* legs of one tensor (after slicing)        */
#define TNC_MAX_CUTS 16        /* cut legs touching one site tensor         */

/* kernel selection for tnc_step (field `kernel`) */
#define TNC_K_AUTO     0
#define TNC_K_GENERIC  1   /* tiled SIMT, arbitrary strides (any shape)      */
#define TNC_K_SKINNY   2   /* bandwidth kernel, A rows contiguous, K,N <= 64 */
#define TNC_K_TC       3   /* tcgen05 3xTF32 (c64) / DMMA (c128) GEMM path   */

/* Where a site-tensor operand lives for one batch element z:
 *   ptr + z * zstride + sel[z / slices_per_b] * vstride
 *       + sum_c ((s / cut_div[c]) % cut_ext[c]) * cut_stride[c]
 * with s = s0 + z % slices_per_b.  sel == NULL selects variant 0. */
typedef struct {
  const void*    ptr;
  const int32_t* sel;
  int64_t        zstride;
  int64_t        vstride;
  int64_t        nvariants;   /* number of variants behind sel (0 = unknown) */
  int32_t        ncut;
  int32_t        _pad;
  int64_t        cut_stride[TNC_MAX_CUTS];
  int64_t        cut_div[TNC_MAX_CUTS];
  int64_t        cut_ext[TNC_MAX_CUTS];
} tnc_site;

/* One path step: out[z] = contract(acc[z], site(z)).
 * Row index f in [0, M) is mixed-radix over the free legs of acc (dims f_dim,
 * outermost first) and lands at  acc + f_astride.f  /  out + f_cstride.f.
 * Shared index k in [0, K) reads acc at a_koff[k] and the site at b_koff[k];
 * new index n in [0, N) reads the site at b_noff[n] and writes out at c_noff[n].
 * Tables are device arrays of int64. */
typedef struct {
  int32_t  dtype;
  int32_t  kernel;
  int64_t  Z;
  int64_t  slices_per_b;
  int64_t  s0;
  const void* acc;  int64_t acc_zstride;
  void*       out;  int64_t out_zstride;
  tnc_site site;
  int64_t  M;
  int32_t  nf;
  int32_t  c_n_contig;      /* 1 if c_noff[n] == n (rows may still be mapped) */
  int64_t  f_dim[TNC_MAX_LEGS];
  int64_t  f_astride[TNC_MAX_LEGS];
  int64_t  f_cstride[TNC_MAX_LEGS];
  int64_t  K;
  int64_t  N;
  const int64_t* a_koff;
  const int64_t* b_koff;
  const int64_t* b_noff;
  const int64_t* c_noff;
  int32_t  a_rows_contig;   /* 1 if a_koff[k] == k and f_astride.f == f*K   */
  int32_t  c_rows_contig;   /* 1 if c_noff[n] == n and f_cstride.f == f*N   */
  int32_t  b_dense;         /* 1 if b_koff[k] == k*N and b_noff[n] == n      */
  int32_t  conj_b;          /* 1: contract with conj(site)                  */
  /* Optional per-batch-element magnitude bounds (complex64; NULL = none):
   * amax_out[z] <- max over out[z] of |re|, |im| (zeroed and written by the
   * step), amax_in[z] = the same for acc[z] (the previous step's amax_out).
   * With amax_in, tensor-core GEMM steps scale and split their operands into
   * fp16 hi/lo pairs (two-fold MMA rate, same ~2^-22 product accuracy). */
  float*       amax_out;
  const float* amax_in;
  /* Optional structure of the new legs (nn = 0: unknown): n in [0, N) is
   * mixed-radix over n_dim (outermost first) and c_noff[n] = n_cstride.n.
   * Lets the tensor-core epilogue store result tiles with TMA. */
  int32_t  nn;
  int32_t  _pad2;
  int64_t  n_dim[TNC_MAX_LEGS];
  int64_t  n_cstride[TNC_MAX_LEGS];
} tnc_step_desc;

/* Gather: out[z][i] = site(z)[ sum_j digit_j(i) * src_stride[j] ], i mixed-radix
 * over dims (outermost first); optional conjugation. */
typedef struct {
  int32_t  dtype;
  int32_t  conj;
  int64_t  Z;
  int64_t  slices_per_b;
  int64_t  s0;
  tnc_site site;
  void*    out;
  int64_t  out_zstride;
  int32_t  nd;
  int32_t  _pad;
  int64_t  dim[TNC_MAX_LEGS];
  int64_t  src_stride[TNC_MAX_LEGS];
} tnc_project_desc;

/* amp[b] (+)= sum_{j < slices_per_b} x[(b * slices_per_b + j) * x_zstride], b < B. */
typedef struct {
  int32_t  dtype;
  int32_t  accumulate;      /* 0: overwrite amp, 1: add into amp           */
  int64_t  B;
  int64_t  slices_per_b;
  const void* x;
  int64_t  x_zstride;
  void*    amp;
} tnc_slice_sum_desc;

/* A whole planned path over one (bitstring x slice) chunk. */
typedef struct {
  tnc_project_desc     first;
  int32_t              nsteps;
  int32_t              _pad;
  const tnc_step_desc* steps;     /* host array of nsteps descriptors        */
  tnc_slice_sum_desc   reduce;
} tnc_path_desc;

int  tnc_version(void);                      /* ABI version (major*100+minor) */
/* sizeof of the descriptor structs, for binding checks:
 * 0 tnc_site, 1 tnc_step_desc, 2 tnc_project_desc, 3 tnc_slice_sum_desc, 4 tnc_path_desc */
size_t tnc_struct_size(int which);
int  tnc_device_check(void);                 /* TNC_OK if an sm_100 device is current */
const char* tnc_last_error(void);

int  tnc_project(const tnc_project_desc* d, void* stream);
int  tnc_step(const tnc_step_desc* d, void* stream);
int  tnc_slice_sum(const tnc_slice_sum_desc* d, void* stream);
int  tnc_contract_path(const tnc_path_desc* d, void* stream);

/* tensor.py:100 contract_pair, batched: for every z < batch,
 *   out[z] = sum over paired axes of a[z] * (conj_b ? conj(b[z]) : b[z])
 * a: rank a_rank dims a_dims (row-major, z-stride a_zstride; 0 broadcasts),
 * b likewise; pairs (pair_a[i], pair_b[i]); result axes = unpaired a axes then
 * unpaired b axes, optionally permuted by out_perm (NULL = identity), written
 * row-major with z-stride out_zstride.  `workspace` must hold
 * tnc_contract_pair_workspace(...) bytes of device memory. */
size_t tnc_contract_pair_workspace(int a_rank, const int64_t* a_dims, int b_rank, const int64_t* b_dims,
                                   int npairs, const int32_t* pair_a, const int32_t* pair_b);
int  tnc_contract_pair(int dtype, int64_t batch,
                       const void* a, int a_rank, const int64_t* a_dims, int64_t a_zstride,
                       const void* b, int b_rank, const int64_t* b_dims, int64_t b_zstride,
                       int npairs, const int32_t* pair_a, const int32_t* pair_b,
                       const int32_t* out_perm, int conj_b,
                       void* out, int64_t out_zstride,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Reusable pairwise plan: the layout analysis and offset tables of
 * tnc_contract_pair computed once (device tables owned by the plan), so a path
 * step or a benchmark loop launches only the kernel.  Execute is asynchronous
 * on `stream`. */
typedef struct tnc_pair_plan tnc_pair_plan;
int  tnc_pair_plan_create(int dtype, int a_rank, const int64_t* a_dims, int b_rank, const int64_t* b_dims,
                          int npairs, const int32_t* pair_a, const int32_t* pair_b,
                          const int32_t* out_perm, int conj_b, tnc_pair_plan** plan);
int  tnc_pair_plan_execute(const tnc_pair_plan* plan, int64_t batch,
                           const void* a, int64_t a_zstride, const void* b, int64_t b_zstride,
                           void* out, int64_t out_zstride, void* stream);
int  tnc_pair_plan_kernel(const tnc_pair_plan* plan);   /* TNC_K_SKINNY (tiled) or TNC_K_GENERIC */
void tnc_pair_plan_destroy(tnc_pair_plan* plan);

#ifdef __cplusplus
}
#endif
#endif /* TNC_H_ */
