/*
 * tk_b200.h -- C ABI of the B200-native tilekit kernels (libtilekit_b200.so).
 *
 * This is the drop-in boundary.  The reference (tilekit, a header-only C++20
 * library) has no FFI of its own; its public entry points are the inline
 * functions listed next to each declaration below.  The C++ headers in
 * include/tilekit/ keep those signatures verbatim and forward here, so a
 * caller of the reference recompiles unchanged.  Anything else (Python
 * ctypes, another language's FFI) binds these symbols directly; see
 * INTEGRATION.md.
 *
 * Conventions
 *  - plain pointers and sizes only; no C++ or torch types.
 *  - matrices are column-major (element (i,j) at i + j*rows), 4-D tensors are
 *    row-major NHWC (inputs/outputs) and HWCK (filters), exactly the
 *    reference layouts (tensor.hpp:12-111).
 *  - every function returns TK_OK or an error code; the message is
 *    available from tk_last_error() (thread-local).  Codes map 1:1 onto the
 *    reference exception classes (errors.hpp:9-59).
 *  - "host" entry points take HOST buffers and do the device copies inside;
 *    "_dev" entry points take caller-owned DEVICE buffers and an explicit
 *    cudaStream_t (passed as void*), launch asynchronously and allocate
 *    nothing once their workspace is provided.
 *  - there is no CPU fallback: without a usable sm_100 GPU every compute
 *    entry point returns TK_ERR_CUDA.
 */
#ifndef TK_B200_H_
#define TK_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TK_ABI_VERSION 1

#if defined(__GNUC__)
#define TK_API __attribute__((visibility("default")))
#else
#define TK_API
#endif

/* Status codes: one per reference exception class (errors.hpp:16-56). */
enum tk_status {
  TK_OK = 0,
  TK_ERR_SHAPE = 1,      /* ShapeError      */
  TK_ERR_CONFIG = 2,     /* ConfigError     */
  TK_ERR_PARSE = 3,      /* ParseError      */
  TK_ERR_CAPABILITY = 4, /* CapabilityError */
  TK_ERR_CONTRACT = 5,   /* ContractError   */
  TK_ERR_IO = 6,         /* IoError         */
  TK_ERR_TUNING = 7,     /* TuningError     */
  TK_ERR_CUDA = 8        /* device failure / no B200 (no reference twin) */
};

/* Arithmetic of the contraction.  The reference is FP32 with separate
 * multiply and add roundings; TK_PREC_FP32_EXACT reproduces it bit for bit
 * (FMUL+FADD, ascending k, no split-K).  The tensor-core precisions are the
 * B200 extension and are judged with max_scaled_error (numeric.hpp:39-56). */
enum tk_precision {
  TK_PREC_FP32_EXACT = 0, /* SIMT, bit-identical to gemm_naive/conv2d_naive */
  TK_PREC_TF32 = 1,       /* tcgen05 kind::tf32, fp32 accumulate            */
  TK_PREC_BF16 = 2,       /* tcgen05 kind::f16 (bf16 operands), fp32 accum. */
  TK_PREC_3XTF32 = 3      /* split-precision tf32 (hi/lo, three MMAs)       */
};

/* GemmShape (config.hpp:19-37).  op: 0 = Op::Identity, 1 = Op::Transpose. */
typedef struct tk_gemm_shape {
  size_t m, n, k;
  float alpha, beta;
  int op_a, op_b;
} tk_gemm_shape;

/* GemmConfig (config.hpp:42-65): h x w register tile, r x c work-group. */
typedef struct tk_gemm_config {
  size_t reg_rows, reg_cols; /* h, w */
  size_t wg_rows, wg_cols;   /* r, c */
  int use_local_memory;      /* _loc  */
  int double_buffer;         /* _db   */
  size_t k_step;
} tk_gemm_config;

/* DeviceSpec (device.hpp:20-50).  name may be NULL. */
typedef struct tk_device_spec {
  const char* name;
  size_t cache_line_bytes;
  size_t local_memory_bytes;
  size_t compute_units;
  size_t register_budget;
  size_t max_workgroup_size;
} tk_device_spec;

/* ConvShape (config.hpp:137-195).  padding: 0 = Valid, 1 = Same. */
typedef struct tk_conv_shape {
  size_t batch, in_rows, in_cols, channels, features;
  size_t window_rows, window_cols, stride;
  int padding;
} tk_conv_shape;

/* ConvAlgoParams (config.hpp:198-241).
 * algo: 0 = Naive, 1 = Tiled, 2 = Im2col, 3 = Winograd. */
typedef struct tk_conv_params {
  int algo;
  size_t tile_rows, tile_cols;
  size_t channel_vector, feature_vector;
} tk_conv_params;

/* B200 execution options (the extension struct of SURVEY.md 8(b); the
 * reference structs stay untouched).  Zero-initialised = reference
 * semantics: exact FP32, library-chosen kernel shape. */
typedef struct tk_exec_options {
  int precision;     /* enum tk_precision                                  */
  int tc_tile_n;     /* tensor-core N tile of a GEMM (0 = auto; 64..256)   */
  int tc_stages;     /* smem pipeline depth (0 = auto, else 2..8)          */
  int tc_cluster;    /* 0 = auto, 1 = one SM (UMMA M 128), 2 = SM pair     */
  int tc_mode;       /* conv operand path: enum tk_tc_mode                  */
  int tc_split;      /* 0 = cost model, 1 = never split K (no split-K, no
                        wave tail), n > 1 = n K-splits where supported     */
  int io;            /* TK_IO_* flags: activations kept in HBM as bf16
                        (BF16 precision, im2col algorithm): the in / out
                        pointers of the conv calls then address bf16 NHWC
                        tensors (element counts unchanged)                 */
  int reserved[1];
} tk_exec_options;

/* tk_exec_options.io: a BF16 network keeps its activations in bf16 between
 * layers -- the producing layer's epilogue writes bf16 (TK_IO_OUT_BF16) and
 * the consuming layer reads it without a conversion pass (TK_IO_IN_BF16). */
enum tk_io_flags {
  TK_IO_FP32 = 0,
  TK_IO_IN_BF16 = 1,
  TK_IO_OUT_BF16 = 2
};

/* Tensor-core convolution operand paths (tk_exec_options.tc_mode); a mode
 * (or tc_cluster) the shape cannot use is rejected with TK_ERR_CAPABILITY. */
enum tk_tc_mode {
  TK_TC_AUTO = 0,
  TK_TC_HALO = 1,      /* one halo box per channel chunk, taps as views    */
  TK_TC_PIXN = 2,      /* features on the MMA M side, pixel boxes on N     */
  TK_TC_PIXM = 3,      /* pixels on M, features on N                       */
  TK_TC_GATHER = 4,    /* producer warps build the pixel operand           */
  TK_TC_POINTWISE = 5, /* 1x1: plain GEMM on the NHWC input                */
  TK_TC_IM2COL = 6     /* pixels on M gathered by im2col-mode TMA          */
};

/* Kernel family a convolution call runs (tk_conv_plan_info.kernel); the
 * tensor-core values equal the tk_tc_mode of the operand path. */
enum tk_kernel_kind {
  TK_KERNEL_EXACT = 0,        /* FP32 SIMT implicit GEMM, bit-exact          */
  TK_KERNEL_TC_HALO = 1,
  TK_KERNEL_TC_PIXN = 2,
  TK_KERNEL_TC_PIXM = 3,
  TK_KERNEL_TC_GATHER = 4,
  TK_KERNEL_TC_POINTWISE = 5,
  TK_KERNEL_TC_IM2COL = 6,
  TK_KERNEL_WINOGRAD = 7,     /* transforms + batched transform-domain GEMM */
  TK_KERNEL_TC_HALO_NARROW = 8 /* C <= 16 bytes per pixel: padded 16-byte pixels, one
                                  halo box per stride phase, two taps per MMA */
};

/* The plan of one convolution call (tk_conv2d_plan_info): what
 * tk_conv2d_dev / tk_conv2d_run_dev will launch for this shape, algorithm
 * and options.  `precision` is the arithmetic the contraction actually runs
 * in -- it differs from the request when a path has no kernel for it (the
 * gather producers and the Winograd batched GEMM compute BF16 requests in
 * TF32). */
typedef struct tk_conv_plan_info {
  int kernel;              /* enum tk_kernel_kind                            */
  int precision;           /* effective enum tk_precision                    */
  int requested_precision; /* tk_exec_options.precision of the call          */
  int cta_group;           /* SMs per tensor-core tile (1 or 2); 1 for SIMT  */
  int tile_m, tile_n;      /* MMA tile (TC) or CTA output tile (SIMT)        */
  int splits;              /* split-K partial sums (1 = none)                */
  int tail_pieces;         /* stream-K tail: max pieces per tile (0 = none)  */
  int imgs, flat;          /* pixN: whole images per tile / flat-row tiles   */
  int box_w, box_h;        /* pixel box of the box / halo modes              */
  int halo_resident;       /* halo: filter slice resident in shared memory   */
  int winograd_m;          /* 2 or 4 for TK_KERNEL_WINOGRAD, else 0          */
  int tuned;               /* 1: knobs from the loaded tuning DB             */
  int reserved[3];
} tk_conv_plan_info;

/* The plan of one GEMM call (tk_gemm_plan_info): what tk_gemm_dev will run
 * for this shape, config and options (operands assumed 16-byte aligned). */
typedef struct tk_gemm_plan {
  int kernel;              /* TK_KERNEL_EXACT, or TK_KERNEL_TC_IM2COL's neighbour
                              TK_KERNEL_TC_PLAIN (9): the tensor-core GEMM      */
  int precision;           /* effective enum tk_precision                    */
  int requested_precision; /* tk_exec_options.precision of the call          */
  int cta_group;           /* SMs per tensor-core tile (1 or 2); 1 for SIMT  */
  int tile_m, tile_n;      /* MMA tile (TC) or CTA output tile (SIMT)        */
  int splits;              /* split-K partial sums (1 = none)                */
  int tail_pieces;         /* stream-K tail: max pieces per tile (0 = none)  */
  int a_in_place, b_in_place; /* operand read where it lies (no pack pass)   */
  int k_depth;             /* contraction depth of the MMAs (3 kp: 3xTF32)   */
  int tuned;               /* 1: knobs from the loaded tuning DB             */
  int reserved[4];
} tk_gemm_plan;
#define TK_KERNEL_TC_PLAIN 9

/* ---- library --------------------------------------------------------- */
TK_API const char* tk_last_error(void);
TK_API int tk_abi_version(void);
/* Number of usable sm_100 devices (0 when none; never an error). */
TK_API int tk_device_count(void);
/* DeviceSpec describing the current B200 (cudaGetDeviceProperties):
 * 128 B lines, 227 KiB opt-in shared memory, 148 SMs, 255 registers,
 * 1024 threads.  Kept out of builtin_devices(). */
TK_API int tk_b200_device_spec(tk_device_spec* out);
/* Kernels launched by this library since load (all streams); used by the
 * bench to report gpu_launches. */
TK_API uint64_t tk_launch_count(void);
TK_API int tk_synchronize(void);

/* ---- validation (host-only, no GPU needed) ---------------------------- */
/* validate_config (gemm.hpp:103-146): writes the "; "-joined violation
 * list (or "valid") into msg and sets *ok. */
TK_API int tk_validate_gemm_config(const tk_gemm_config* cfg, const tk_device_spec* dev,
                            int* ok, char* msg, size_t msg_cap);
/* local_mem_elems (gemm.hpp:71-80). */
TK_API int tk_local_mem_elems(const tk_gemm_config* cfg, const tk_device_spec* dev,
                       size_t* elems);

/* ---- GEMM ------------------------------------------------------------- */
/* gemm_tiled (gemm.hpp:308-445).  a/b are the STORED operands (m x k or
 * k x m when transposed, etc.), c is m x n, out is m x n.  c is not read
 * when beta == 0.  Host buffers. */
TK_API int tk_gemm_tiled(const tk_gemm_shape* shape, const tk_gemm_config* cfg,
                  const tk_device_spec* dev, const float* a, const float* b,
                  const float* c, float* out);
/* gemm_naive (gemm.hpp:194-213): same arithmetic on the GPU. */
TK_API int tk_gemm_naive(const tk_gemm_shape* shape, const float* a, const float* b,
                  const float* c, float* out);
/* gemm_batched_strided (gemm.hpp:451-479); *multiplies gets the count. */
TK_API int tk_gemm_batched_strided(const float* a, size_t stride_a, const float* b,
                            size_t stride_b, float* c, size_t stride_c,
                            size_t batch, size_t m, size_t n, size_t k,
                            uint64_t* multiplies);
/* Device-buffer GEMM.  cfg may be NULL (library choice); opts may be NULL
 * (exact FP32).  Tensor-core precisions ignore cfg. */
/* What tk_gemm_dev would run for (shape, cfg, opts): kernel family,
 * effective precision, CTA group, tile, split-K, stream-K tail, which
 * operands are read in place, whether a tuning-DB record chose the knobs.
 * Nothing is launched or allocated. */
TK_API int tk_gemm_plan_info(const tk_gemm_shape* shape, const tk_gemm_config* cfg,
                             const tk_exec_options* opts, tk_gemm_plan* out);
TK_API int tk_gemm_dev(const tk_gemm_shape* shape, const tk_gemm_config* cfg,
                const tk_exec_options* opts, const float* d_a, const float* d_b,
                const float* d_c, float* d_out, void* stream);
/* gemm with B200 execution options on HOST buffers (precision etc.). */
TK_API int tk_gemm_ex(const tk_gemm_shape* shape, const tk_exec_options* opts, const float* a,
                      const float* b, const float* c, float* out);
/* gemm_batched_strided (gemm.hpp:451-479) on device buffers: C_g = A_g B_g,
 * column-major members at the given element strides, C zeroed (not read).
 * opts->precision FP32_EXACT: the bit-exact SIMT path; TF32 / BF16: one
 * batched tensor-core GEMM (A_g packed K-major, B_g read in place when it
 * can be); 3XTF32: the split-precision GEMM per member. */
TK_API int tk_gemm_batched_strided_dev(const float* d_a, size_t stride_a,
                                const float* d_b, size_t stride_b, float* d_c,
                                size_t stride_c, size_t batch, size_t m,
                                size_t n, size_t k, const tk_exec_options* opts,
                                void* stream);

/* ---- convolution ------------------------------------------------------ */
/* conv2d selector (winograd.hpp:304-314) and the per-algorithm entry
 * points (conv.hpp:74, :136, :320, :353; winograd.hpp:169).  Host buffers:
 * in NHWC, filt HWCK, out NHWC (batch x out_rows x out_cols x features). */
TK_API int tk_conv2d(const tk_conv_shape* shape, const tk_conv_params* params,
              const float* in, const float* filt, float* out);
TK_API int tk_conv2d_naive(const tk_conv_shape* shape, const float* in,
                    const float* filt, float* out);
TK_API int tk_conv2d_tiled(const tk_conv_shape* shape, const tk_conv_params* params,
                    const float* in, const float* filt, float* out);
/* conv2d_im2col with an explicit GEMM config + device (conv.hpp:320-351). */
TK_API int tk_conv2d_im2col(const tk_conv_shape* shape, const tk_gemm_config* cfg,
                     const tk_device_spec* dev, const float* in,
                     const float* filt, float* out);
/* conv2d_winograd (winograd.hpp:169-301); stats may be NULL. */
TK_API int tk_conv2d_winograd(const tk_conv_shape* shape, const tk_conv_params* params,
                       const float* in, const float* filt, float* out,
                       uint64_t* batched_multiplies, size_t* tiles);
/* im2col (conv.hpp:255-300): column-major (N*OH*OW) x (R*S*C). */
TK_API int tk_im2col(const tk_conv_shape* shape, const float* in, float* patches);
/* filter_matrix (conv.hpp:304-317): HWCK -> column-major (R*S*C) x K. */
TK_API int tk_filter_matrix(size_t r, size_t s, size_t c, size_t k, const float* filt,
                     float* mat);

/* Device-buffer convolution through the selector.  workspace may be NULL
 * (library-owned, grown on first use; not allocation-free then). */
TK_API int tk_conv2d_dev(const tk_conv_shape* shape, const tk_conv_params* params,
                  const tk_exec_options* opts, const float* d_in,
                  const float* d_filt, float* d_out, void* d_workspace,
                  size_t workspace_bytes, void* stream);
TK_API int tk_conv2d_workspace_size(const tk_conv_shape* shape,
                             const tk_conv_params* params,
                             const tk_exec_options* opts, size_t* bytes);
/* Same as tk_conv2d but with the exec options (host buffers). */
TK_API int tk_conv2d_ex(const tk_conv_shape* shape, const tk_conv_params* params,
                 const tk_exec_options* opts, const float* in,
                 const float* filt, float* out);
/* The same convolution in two phases on caller-provided workspace:
 * prepare = the filter-side work (tensor-core filter repack, Winograd filter
 * transform) -- it reads only d_filt, so it may run on another stream and
 * overlap earlier work; run = everything that reads the input, ordered after
 * prepare on the same workspace. */
TK_API int tk_conv2d_prepare_dev(const tk_conv_shape* shape, const tk_conv_params* params,
                                 const tk_exec_options* opts, const float* d_filt,
                                 void* d_workspace, size_t workspace_bytes, void* stream);
TK_API int tk_conv2d_run_dev(const tk_conv_shape* shape, const tk_conv_params* params,
                             const tk_exec_options* opts, const float* d_in, const float* d_filt,
                             float* d_out, void* d_workspace, size_t workspace_bytes,
                             void* stream);
/* The plan tk_conv2d_dev would run (host-side only: no GPU work, usable
 * without a GPU for the shape/option logic). */
TK_API int tk_conv2d_plan_info(const tk_conv_shape* shape, const tk_conv_params* params,
                               const tk_exec_options* opts, tk_conv_plan_info* out);
TK_API int tk_im2col_dev(const tk_conv_shape* shape, const float* d_in,
                  float* d_patches, void* stream);

/* ---- tuning DB (lookup_best on the launch path, tuner.hpp:684-694) ------ */
/* Load (merge) the tuner's NDJSON DB: for each (problem key, algorithm,
 * precision) the fastest valid record's tensor-core knobs are kept.  A
 * conv (im2col algorithm) or GEMM call on tensor cores whose
 * tk_exec_options leave every knob automatic then runs with those knobs
 * instead of the built-in rules.  device: keep only records of this device
 * name (NULL = any).  *records = records kept. */
TK_API int tk_tuning_db_load(const char* path, const char* device, size_t* records);
TK_API int tk_tuning_db_clear(void);
TK_API int tk_tuning_db_size(size_t* entries);

/* ---- benchmarking (the tuner's device clock) --------------------------- */
/* Upload the given HOST inputs once, run `warmup` untimed and `samples`
 * timed launches of the device path (CUDA events on a private stream) and
 * write each sample's duration in nanoseconds to ns[samples].  cfg may be
 * NULL (library default); opts may be NULL (exact FP32).  c may be NULL
 * when beta == 0.  Used by tilekit::benchmark_config (tuner.hpp). */
TK_API int tk_bench_gemm(const tk_gemm_shape* shape, const tk_gemm_config* cfg,
                         const tk_exec_options* opts, const float* a, const float* b,
                         const float* c, int warmup, int samples, int64_t* ns);
TK_API int tk_bench_conv2d(const tk_conv_shape* shape, const tk_conv_params* params,
                           const tk_exec_options* opts, const float* in, const float* filt,
                           int warmup, int samples, int64_t* ns);

#ifdef __cplusplus
}
#endif

#endif /* TK_B200_H_ */
