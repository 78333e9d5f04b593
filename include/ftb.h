/*
 * ftb.h — C ABI of the B200-native FTuner hot path (libftb.so).
 *
 * The reference (mktune 0.1.0, /root/reference/pkg/src/mktune) is a pure
 * Python package with no FFI. These entry points are what a ctypes/cffi
 * binding of that package's hot path binds instead; each one names the
 * reference interface it replaces. Conventions:
 *   - every function returns an ftb_status; 0 = success;
 *   - status codes map 1:1 onto mktune.errors (errors.py:10-47):
 *       FTB_INPUT_ERROR -> InputError, FTB_CAPACITY_ERROR -> CapacityError,
 *       FTB_EMPTY_RESULT -> EmptyResultError, FTB_MISSING_METRICS ->
 *       MissingMetricsError, FTB_INTERNAL_ERROR -> InternalError;
 *     FTB_CUDA_ERROR is new (device failures have no reference analogue);
 *   - the message of the last failure on the calling thread is returned by
 *     ftb_last_error();
 *   - buffers are caller-owned; handles (ftb_exec*, ftb_planner*) are owned by
 *     the library and released with the matching *_destroy call;
 *   - no torch types: device pointers are plain void*, streams are the
 *     cudaStream_t value cast to void*.
 */
#ifndef FTB_H_
#define FTB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t ftb_status;
enum {
  FTB_OK = 0,
  FTB_INPUT_ERROR = 2,      /* errors.py:14-22 InputError (exit code 2)          */
  FTB_EMPTY_RESULT = 1,     /* errors.py:29-39 EmptyResultError (exit code 1)    */
  FTB_INTERNAL_ERROR = 3,   /* errors.py:46-47 InternalError (exit code 3)       */
  FTB_CAPACITY_ERROR = 4,   /* errors.py:25-26 CapacityError                     */
  FTB_MISSING_METRICS = 5,  /* errors.py:42-43 MissingMetricsError              */
  FTB_CUDA_ERROR = 6        /* new: CUDA runtime / driver failure                */
};

/* Thread-local message of the last failing call (NUL-terminated, truncated). */
size_t ftb_last_error(char* buf, size_t n);
/* Optional: the field name attached to the last InputError (errors.py:20-22). */
size_t ftb_last_error_field(char* buf, size_t n);

/* ------------------------------------------------------------------------ */
/* Program (compose/select output)                                          */
/* ------------------------------------------------------------------------ */

/* Axis order follows the operator spec: space axes then reduce axes.
 *   Dense: (i, j, k)        C[i,j]   = sum_k A[i,k] B[k,j]
 *   BMM  : (b, i, j, k)     C[b,i,j] = sum_k A[b,i,k] B[b,k,j]
 * A program is the reference's ProgramPlan (combine.py:30-55): one or two
 * uKernels, each with a repetition count along the main axis tau; non-tau
 * tiles are uniform across parts (combine.py:118-123). */
#define FTB_MAX_AXES 8
typedef struct {
  int32_t n_space;                    /* 2 (dense) or 3 (bmm)                    */
  int32_t n_reduce;                   /* 1                                       */
  int32_t tau;                        /* index of tau among the space axes       */
  int32_t n_parts;                    /* 1 or 2                                  */
  int64_t reg[2][FTB_MAX_AXES];       /* register tiles (space axes)             */
  int64_t smem[2][FTB_MAX_AXES];      /* shared-memory tiles (space + reduce)    */
  int64_t count[2];                   /* repetitions along tau                   */
  double sia;                         /* score attached by ranking (scoring.py:126) */
} ftb_program;

/* ------------------------------------------------------------------------ */
/* Planner (enumerate -> annotate -> filter -> relax -> compose -> rank)     */
/* ------------------------------------------------------------------------ */

/* HardwareDescriptor (hardware.py:35-66): the 9 integer fields, plus the
 * B200 legality extension (0 = parity mode, exactly the reference). With
 * legality = 1 the tile rules derive from the tcgen05 fields (0 = the sm_100a
 * value): lane tiles are multiples of the largest MMA M atom (up to two
 * slabs) or span a short axis; column tiles are the widest MMA N
 * (mma_n_max, which a double-buffered accumulator must fit twice in
 * tmem_columns) or span a short axis; reduce tiles are whole TMA swizzle
 * atoms (tma_swizzle_bytes / elem_bytes elements). */
typedef struct {
  int64_t num_cores, regs_per_core, smem_per_core_bytes;
  int64_t global_bw_bytes_per_s, shared_bw_bytes_per_s, peak_flops;
  int64_t default_active_blocks, active_blocks_per_core, align_elems;
  int32_t legality;   /* 0 = parity (reference), 1 = tcgen05 tile legality */
  int32_t reserved;
  int64_t tmem_columns;       /* 512 */
  int64_t mma_m_max;          /* 128: largest M of the cta_group::1 kind::f16 atoms */
  int64_t mma_n_step;         /* 16  */
  int64_t mma_n_max;          /* 256 */
  int64_t tma_swizzle_bytes;  /* 128 */
} ftb_hw;

/* A bound WorkloadInstance (workload.py:187-220) flattened. Axis indices
 * run over the spec's space axes then its reduce axes (axis_names order of
 * ukernel.py:250-252). */
#define FTB_MAX_INPUTS 4
typedef struct {
  int32_t n_space, n_reduce;
  int32_t major;                                  /* space index of the major axis (ukernel.py:93-95) */
  int32_t n_inputs;
  int32_t input_naxes[FTB_MAX_INPUTS];
  int32_t input_axes[FTB_MAX_INPUTS][FTB_MAX_AXES];
  int32_t elem_bytes, flops_per_point;
  int64_t extent[FTB_MAX_AXES];
  int32_t dynamic[FTB_MAX_AXES];
  char axis_name[FTB_MAX_AXES][16];
} ftb_instance;

typedef struct { int64_t num, den; } ftb_frac;

/* FilterParams + SweepParams (filtering.py:77-128, :237-250). */
typedef struct {
  ftb_frac eps_min, eps_max, lam_min, lam_max, eps_step, lam_step;
  double psi;
  int64_t rest_regs;
  int64_t candidate_cap;   /* < 0 = no cap (None) */
} ftb_params;

typedef struct { double c0, c1, c2; } ftb_coeffs;   /* SiaCoeffs (scoring.py:23-38) */

enum { FTB_RELAX_NONE = 0, FTB_RELAX_DROP_INTENSITY = 1, FTB_RELAX_DROP_SATURATION = 2,
       FTB_RELAX_WIDEN = 3, FTB_RELAX_DROP_SWEEP = 4 };

/* ShapeResult provenance (filtering.py:253-264, :334-348). */
typedef struct {
  int64_t n_align, n_cross, n_filter, n_final;
  int32_t relaxation;      /* FTB_RELAX_*                                 */
  int32_t widen;           /* N of "widen-sweep-N"                        */
  int32_t truncated;
  int32_t tau;             /* select_main_axis (combine.py:58-68)         */
  ftb_frac sweep_used[6];  /* eps_min, eps_max, lam_min, lam_max, eps_step, lam_step */
  int32_t stage;           /* set ranked by ftb_plan_batch: 0 final; B200-mode fallback
                              rungs 1 filter, 2 cross, 3 align (extension)          */
  int32_t reserved;
  double seconds;
} ftb_compile_report;

/* Columnar candidate set (CandidateSet, ukernel.py:219-313) owned by the library. */
typedef struct ftb_cands ftb_cands;

/* enumerate_ukernels (ukernel.py:341-437): canonical order, cap truncation. */
ftb_status ftb_enumerate(const ftb_hw* hw, const ftb_instance* inst, int64_t cap,
                         ftb_cands** out, int32_t* truncated);
/* compile_shape (filtering.py:270-348): the final set with cached metrics. */
ftb_status ftb_compile_shape(const ftb_hw* hw, const ftb_instance* inst, const ftb_params* p,
                             ftb_cands** out, ftb_compile_report* rep);
/* A candidate table from caller arrays (build_programs on arbitrary UKernels,
 * combine.py:133). Metric pointers may be NULL; NaN = metric not cached. */
ftb_status ftb_cands_from_arrays(const ftb_instance* inst, int64_t n, const int64_t* reg,
                                 const int64_t* smem, const double* pad, const double* occ,
                                 const double* cmr, ftb_cands** out);
int64_t ftb_cands_size(const ftb_cands* c);
/* Row-major exports: reg[n][n_space], smem[n][n_space+n_reduce];
 * icol[n][7] = pad_num, pad_den, blocks, occ_den, regs_in_block, saturated,
 * retained_step; fcol[n][2] = cmr, kmem. Any pointer may be NULL. */
ftb_status ftb_cands_export(const ftb_cands* c, int64_t* reg, int64_t* smem, int64_t* icol,
                            double* fcol);
void ftb_cands_destroy(ftb_cands* c);

/* select_main_axis (combine.py:58-68). */
ftb_status ftb_select_main_axis(const ftb_instance* inst, int32_t* tau);
/* Size of the program pool build_programs would materialise (combine.py:133-194). */
ftb_status ftb_pool_count(const ftb_cands* c, int32_t tau, int64_t* n);
/* The pool in canonical plan-key order (combine.py:182): rows[i] =
 * {nparts, row_a, count_a, row_b, count_b} with rows into the candidate table. */
ftb_status ftb_pool_export(const ftb_cands* c, int32_t tau, int64_t cap, int64_t* rows,
                           int64_t* n);
/* rank_programs (scoring.py:83-126) over the implicit pool, streamed: the
 * pool is never materialised. rows as ftb_pool_export, scores[i] = sia. */
ftb_status ftb_rank_topk(const ftb_cands* c, int32_t tau, const ftb_coeffs* coeffs, int32_t k,
                         int32_t normalize, int64_t* rows, double* scores, int32_t* n_out);
/* compile_stage (filtering.py:376-405) + build/rank Top-1 for many shapes on
 * a host thread pool; out[i] is the Top-1 program of inst[i]. */
ftb_status ftb_plan_batch(const ftb_hw* hw, const ftb_instance* insts, int32_t n,
                          const ftb_params* p, const ftb_coeffs* coeffs, int32_t threads,
                          ftb_program* out, ftb_compile_report* reps, ftb_status* statuses);

/* ------------------------------------------------------------------------ */
/* Execution (the reference has none: SPEC.md:8 — this is the new L6)       */
/* ------------------------------------------------------------------------ */

enum { FTB_OP_DENSE = 0, FTB_OP_BMM = 1 };
enum { FTB_B_KN = 0, /* B stored [K,N], N contiguous (MN-major operand)  */
       FTB_B_NK = 1  /* B stored [N,K], K contiguous (K-major, nn.Linear) */ };
enum { FTB_DT_BF16 = 0, FTB_DT_F32 = 1 };
/* Fused epilogue (Dense only): C = act(A·B + bias), bias[N] in bias_dtype. */
enum { FTB_ACT_NONE = 0, FTB_ACT_GELU = 1 /* erf form, as torch.nn.functional.gelu */ };

/* One GEMM problem bound to device buffers. Strides are in elements.
 * Batch strides are ignored for dense (batch = 1). The tcgen05 path needs
 * bf16 A/B with 16-byte aligned row strides (lda, ldb multiples of 8). */
typedef struct {
  int32_t op;            /* FTB_OP_DENSE / FTB_OP_BMM                      */
  int32_t batch;         /* b (1 for dense)                                */
  int64_t M, N, K;
  const void* A; int64_t lda; int64_t a_batch_stride;   /* A[b][M][lda]    */
  const void* B; int64_t ldb; int64_t b_batch_stride;   /* see b_layout    */
  void* C;       int64_t ldc; int64_t c_batch_stride;   /* C[b][M][ldc]    */
  int32_t b_layout;      /* FTB_B_KN / FTB_B_NK                            */
  int32_t in_dtype;      /* FTB_DT_BF16 (tcgen05) / FTB_DT_F32 (FFMA mode) */
  int32_t out_dtype;     /* FTB_DT_BF16 / FTB_DT_F32                       */
  int32_t orientation;   /* -1 auto, 0 lanes=i (normal), 1 lanes=j (swap-AB) */
  const void* bias;      /* NULL or bias[N] added per output column (Dense) */
  int32_t bias_dtype;    /* FTB_DT_BF16 / FTB_DT_F32                       */
  int32_t activation;    /* FTB_ACT_NONE / FTB_ACT_GELU                    */
} ftb_gemm_desc;

typedef struct ftb_exec ftb_exec;   /* lowered tile-schedule table on device */

typedef struct {
  int64_t n_work;          /* work items in the table                       */
  int64_t n_ctas;          /* persistent CTAs launched                      */
  int64_t n_problems;
  int64_t mma_flops;       /* flops the tensor cores execute (incl. padding) */
  int64_t true_flops;      /* 2*b*M*N*K summed                              */
  int64_t covered_out;     /* output elements covered by the plans          */
  int64_t true_out;        /* true output elements                          */
  int32_t kernel;          /* 0 = tcgen05 bf16, 1 = FFMA fp32               */
} ftb_exec_info;

/* Lower n programs (one per problem) to a tile-schedule table and upload it:
 * replaces nothing in the reference. The programs must
 * cover each problem exactly as ProgramPlan.covered_extents (combine.py:44-55)
 * describes; the table is validated against that before upload. */
ftb_status ftb_exec_create(const ftb_gemm_desc* problems, const ftb_program* programs,
                           int32_t n, ftb_exec** out);
/* Launch the table as one persistent kernel on `stream` (cudaStream_t).
 * Launches of one executable must be stream-ordered (not concurrent on two
 * streams): a split-K table keeps its fp32 partials and arrival counters in
 * per-executable device memory. */
ftb_status ftb_exec_launch(ftb_exec* ex, void* stream);
ftb_status ftb_exec_get_info(const ftb_exec* ex, ftb_exec_info* info);
/* Host copy of the lowered table (int32 x 8 per work item), for tests. */
ftb_status ftb_exec_export_table(const ftb_exec* ex, int32_t* out, int64_t cap, int64_t* n_out);
void ftb_exec_destroy(ftb_exec* ex);
/* Debug: record per-CTA phase timestamps (%globaltimer, ns) for the first 16
 * items of every CTA on subsequent launches; read back per CTA as
 * [16 items][6 events] (producer pick, K0 issued, K0 landed, MMA commit,
 * epilogue start, epilogue release), [64 K blocks][2] (producer issued, MMA
 * saw data), then the CTA's start and end stamps (builds with FTB_TRACE_SPAN). */
ftb_status ftb_exec_set_trace(ftb_exec* ex, int32_t enable);
ftb_status ftb_exec_read_trace(const ftb_exec* ex, uint64_t* out, int64_t cap, int64_t* n_out);
/* Pipeline shapes chosen for the table, 12 ints: single-CTA kernel {stages,
 * col_stage_bytes, n_acc, acc_cols}, CTA-pair kernel {same}, n_singles, n_pairs,
 * on-chip split-K factor (0 or 1: none), global-workspace split-K (0/1). */
ftb_status ftb_exec_get_config(const ftb_exec* ex, int32_t* out4);
/* Host-only lowering (no device, no TMA descriptors): the same table
 * ftb_exec_create would upload, for inspection and CPU tests. */
ftb_status ftb_lower(const ftb_gemm_desc* problems, const ftb_program* programs, int32_t n,
                     int32_t* out, int64_t cap, int64_t* n_out, ftb_exec_info* info);

/* Number of SMs of the current device (0 if none). */
int32_t ftb_device_sm_count(void);

/* TEST HOOK (not on the hot path): launch n_ctas CTAs on `stream` that each
 * hold one SM (maximal dynamic shared memory) until ctl[0] != 0 or timeout_ns
 * elapses. ctl is mapped pinned host memory: ctl[1] counts CTAs that arrived,
 * ctl[2] CTAs that timed out. Lets tests run the executor while another
 * kernel occupies most SMs (split-K must not assume co-residency). */
ftb_status ftb_test_occupy_sms(int32_t n_ctas, int32_t* ctl, int64_t timeout_ns, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FTB_H_ */
