/*
 * stlg.h — C ABI of the B200 masked-STL robustness library (libstlg.so).
 *
 * The reference (/root/reference/pkg/src/stlmask) is pure Python and has no
 * FFI; these entry points replace its hot path at the call sites a binding
 * would patch (see INTEGRATION.md for the ctypes stub):
 *
 *   stlg_compile / stlg_free      <- the AST walk of masking.trace_var
 *                                    (masking.py:308-343), done once per
 *                                    formula instead of per call
 *   stlg_forward                  <- masking.trace_var forward
 *                                    (masking.py:308-343; robustness_trace
 *                                    masking.py:350-357)
 *   stlg_backward                 <- tape.backward(out, seed) over that graph
 *                                    (tape.py:114-134), including the
 *                                    smooth-interval (a, b, c) leaves of
 *                                    autodiff.value_and_grad (autodiff.py:88-106)
 *   stlg_workspace_bytes          <- (no reference equivalent: the tape
 *                                    allocates per node; here the caller owns
 *                                    all memory)
 *
 * Conventions
 *   - All data pointers are caller-owned DEVICE memory; the library never
 *     allocates or frees them.  Work is enqueued on `stream` (a cudaStream_t
 *     passed as void*), with no host synchronisation.
 *   - Signals are fp32, B rows x T samples; channel c is addressed as
 *     ptr[b * row_stride + t * elem_stride] (elements, not bytes), so
 *     [B, T] planes and interleaved [B, T, D] tensors both work.
 *   - Return value: STLG_OK or an error code.  ShapeError / EmptyWindowError
 *     / TypeError / RuntimeError in the Python shim map from these codes.
 *     ValidationError, InvalidIntervalError and binding ValueErrors are
 *     raised in Python before the call, at the reference's own sites.
 *   - Functions are reentrant; a plan is immutable after stlg_compile and may
 *     be used concurrently on different streams with different workspaces.
 *   - Plans whose root joins independent operands (no shared channel, slot or
 *     smooth binding) run one operand group on an internal side stream (one
 *     per host thread and device), forked from `stream` and joined back into
 *     it with events before the call returns: all work is ordered on `stream`
 *     as before, and under stream capture the two groups become parallel
 *     graph branches.  Their workspaces hold one more lane of scratch.
 */
#ifndef STLG_H
#define STLG_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define STLG_API __attribute__((visibility("default")))
#else
#define STLG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define STLG_ABI_VERSION 1

/* status codes */
#define STLG_OK 0
#define STLG_E_SHAPE 1        /* core.ShapeError            (core.py:58)  */
#define STLG_E_EMPTY_WINDOW 2 /* core.EmptyWindowError      (core.py:62)  */
#define STLG_E_UNSUPPORTED 3  /* TypeError (e.g. smooth Until, masking.py:239-240) */
#define STLG_E_CUDA 4         /* RuntimeError: a CUDA call failed          */
#define STLG_E_INVALID 5      /* malformed node program / argument         */

/* node opcodes: one per formula.py node class (formula.py:65-135) */
#define STLG_TRUE 0
#define STLG_PRED 1       /* chan cmp threshold                            */
#define STLG_NOT 2
#define STLG_AND 3
#define STLG_OR 4
#define STLG_EVENTUALLY 5
#define STLG_ALWAYS 6
#define STLG_UNTIL 7
#define STLG_NORM_PRED 8  /* extension: ||(chan, chan2) - center|| cmp threshold */

/* interval kinds for F / G / U */
#define STLG_ITV_NONE 0   /* untimed: whole remaining signal                */
#define STLG_ITV_STEP 1   /* core.StepInterval [a, b]                       */
#define STLG_ITV_SMOOTH 2 /* core.SmoothInterval, params passed at call time */

/* reduction modes (core.py:225-252) */
#define STLG_MODE_HARD 0
#define STLG_MODE_SOFTMAX 1
#define STLG_MODE_LSE 2

typedef struct stlg_node {
  int32_t op;          /* STLG_* opcode                                       */
  int32_t left;        /* child node index (NOT/F/G/AND/OR/UNTIL), else -1    */
  int32_t right;       /* second child (AND/OR/UNTIL), else -1                */
  int32_t chan;        /* PRED / NORM_PRED channel index                      */
  int32_t chan2;       /* NORM_PRED second channel                            */
  int32_t cmp;         /* 0: '>' or '>=' (x - c);  1: '<' or '<=' (c - x)     */
  double threshold;    /* PRED threshold / NORM_PRED radius                   */
  double center0;      /* NORM_PRED center                                    */
  double center1;
  int32_t itv_kind;    /* STLG_ITV_* for F/G/U                                */
  int32_t a, b;        /* STEP interval bounds                                */
  int32_t smooth_slot; /* SMOOTH: index into the per-call smooth_params table */
} stlg_node;

typedef struct stlg_cfg {
  int32_t mode;        /* STLG_MODE_*                                   */
  double temp;         /* temperature (softmax / lse)                   */
  int32_t pad_last;    /* 1: PaddingPolicy('last'), 0: const            */
  double pad_value;    /* const pad value                               */
  double top_value;    /* robustness of TRUE                            */
  double sentinel;     /* masked_fill sentinel                          */
  int32_t masked_fill; /* SemanticsConfig.masked_fill                   */
} stlg_cfg;

typedef struct stlg_channel {
  const float* ptr;
  int64_t row_stride;  /* elements between rows (b)                */
  int64_t elem_stride; /* elements between samples (t)             */
} stlg_channel;

typedef struct stlg_grad {
  float* ptr;
  int64_t row_stride;
  int64_t elem_stride;
  int32_t accumulate;  /* 1: add into the existing contents (+=);
                          0: overwrite — every element is written (zeros where the
                          formula does not depend on it); no zero-fill needed */
} stlg_grad;

/* per-call parameters of smooth-interval node slot s: a, b, c, eps (fp64) */
typedef struct stlg_smooth {
  double a, b, c, eps;
} stlg_smooth;

typedef struct stlg_plan stlg_plan;

/* Library / ABI version; lets a binding refuse a mismatched build. */
STLG_API int stlg_abi_version(void);

/* Human-readable text of the last error on the calling thread. */
STLG_API const char* stlg_last_error(void);

/* Compile a node program.  nodes[] is in topological order (children before
 * parents); nodes[n_nodes-1] is the root.  Children may be shared (a DAG). */
STLG_API int stlg_compile(const stlg_node* nodes, int32_t n_nodes, int32_t n_channels,
                 int32_t n_smooth, const stlg_cfg* cfg, stlg_plan** out_plan);

STLG_API void stlg_free(stlg_plan* plan);

/* Number of temporal-operator launches (diagnostics / launch counting). */
STLG_API int stlg_plan_info(const stlg_plan* plan, int32_t* n_temporal, int32_t* n_slots,
                   int32_t* root_is_temporal);

/* Device workspace needed for B x T.  `fwd_bytes` must stay alive (and
 * unmodified) from stlg_forward until the matching stlg_backward;
 * `bwd_bytes` is scratch for stlg_backward only. */
STLG_API int stlg_workspace_bytes(const stlg_plan* plan, int64_t B, int64_t T, size_t* fwd_bytes,
                         size_t* bwd_bytes);

/* Full robustness trace [B, T] (row stride T) of the root formula. */
STLG_API int stlg_forward(const stlg_plan* plan, const stlg_channel* channels, int64_t B, int64_t T,
                 const stlg_smooth* smooth_params, float* trace_out, void* fwd_ws,
                 size_t fwd_ws_bytes, void* stream);

/* VJP of the full trace with cotangent `cot` [B, T] (row stride T).
 * d_channels[c].ptr may be NULL for channels whose gradient is not needed.
 * d_smooth (device, fp64, 3 * n_smooth: d_a, d_b, d_c per slot) is
 * accumulated into when non-NULL.  `trace` is the forward output. */
STLG_API int stlg_backward(const stlg_plan* plan, const stlg_channel* channels, int64_t B, int64_t T,
                  const stlg_smooth* smooth_params, const float* trace, const float* cot,
                  const stlg_grad* d_channels, double* d_smooth, void* fwd_ws,
                  size_t fwd_ws_bytes, void* bwd_ws, size_t bwd_ws_bytes, void* stream);

/* Batched interval-mining objective (replaces the per-pair
 * loop of apps.grid_eval over apps.mining_objective, apps.py:272-335).
 * data: device fp32 [n, length] (row stride `row_stride`, unit element stride);
 * a, b: device fp64 [npairs] window bounds in (0, 1); sharp: sigmoid sharpness c;
 * mode: STLG_MODE_* with temperature `temp`.  loss_out (device fp64 [npairs]):
 *   mean_n relu(-rho0_n) + gamma (a - b),  rho0_n = smooth min of row n under
 *   w_i = relu(sigmoid(c (i - a L)) - sigmoid(c (i - b L)) - eps);
 * NaN where no weight is positive (the reference's EmptyWindowError).
 * dloss_out (device fp64 [2 npairs], optional): d loss / d a, d loss / d b. */
STLG_API int stlg_mining_grid(const float* data, int64_t n, int64_t length, int64_t row_stride,
                              const double* a, const double* b, int64_t npairs, double sharp,
                              double eps, int32_t mode, double temp, double gamma, double* loss_out,
                              double* dloss_out, void* stream);

/* Count of device kernel launches issued by the library (all threads) since the last reset. */
STLG_API int64_t stlg_launch_count(int reset);

#ifdef __cplusplus
}
#endif
#endif /* STLG_H */
