/*
 * syno.h -- C ABI of the B200 execution backend for synthesized operators.
 *
 * The reference (opsmith, pure Python) exposes the execution path as
 * Python functions; each entry point below replaces one of them and is
 * what a ctypes/cffi binding of the reference would call:
 *
 *   syno_compile         pgraph.parse_operator      pgraph.py:730-790
 *                        + codegen.build_loop_nest  codegen.py:297-362
 *                        + codegen.rfactor          codegen.py:490-508
 *   syno_forward         codegen.interpret          codegen.py:598-630
 *   syno_backward        codegen.weight_gradient    codegen.py:664-743
 *                        (+ the grad-input adjoint the reference lacks)
 *   syno_query           codegen.flops / param_count / input_shape /
 *                        output_shape / weight_shapes codegen.py:575-657
 *   syno_emit_loop_nest  codegen.emit_loop_nest     codegen.py:750-794
 *   syno_compile_nest    codegen.parse_loop_nest    codegen.py:846-943
 *   syno_print_operator  pgraph.print_operator      pgraph.py:712-727
 *   syno_index_map       codegen._eval_array        codegen.py:153-176
 *
 * Conventions: plain pointers and sizes only.  Tensor pointers are CUDA
 * device pointers to dense row-major buffers (x: batch + input dims,
 * y/dy: batch + output dims, w_j: weight dims) of the dtype named by the
 * `dtype` argument; `stream` is a cudaStream_t (NULL = legacy default).
 * Every call returns a status; on failure syno_last_error() (thread-local)
 * holds the message.  Handles are immutable after compile and may be used
 * from several threads and streams at once.
 */
#ifndef SYNO_H_
#define SYNO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct syno_op* syno_op_t;

/* status codes: one per reference exception family */
enum {
  SYNO_OK = 0,
  SYNO_E_PARSE = 1,        /* pgraph.OperatorParseError (pgraph.py:655) */
  SYNO_E_GRAPH = 2,        /* pgraph.GraphError and subclasses (pgraph.py:66-83) */
  SYNO_E_SHAPE = 3,        /* codegen.ShapeMismatch (codegen.py:68) */
  SYNO_E_NONINTEGRAL = 4,  /* symexpr.NonIntegralSize (symexpr.py:21) */
  SYNO_E_KEY = 5,          /* KeyError: unbound size variable (symexpr.py:112) */
  SYNO_E_VALUE = 6,        /* ValueError: bad size text / assignment < 1 */
  SYNO_E_CUDA = 7,         /* CUDA runtime failure */
  SYNO_E_INVALID = 8,      /* bad argument at this ABI */
  SYNO_E_UNSUPPORTED = 9   /* operator outside the device engine's limits */
};

/* dtypes: arithmetic type of x, w, y and the gradients */
enum { SYNO_F32 = 0, SYNO_BF16 = 1, SYNO_F64 = 2 };

/* compile flags */
enum {
  SYNO_STAGED = 1,      /* forward runs the rfactor-staged nest (interpret(..., staged=True)) */
  SYNO_REPLAY_ONLY = 2  /* parse + replay only (pgraph.parse_steps): no lowering, no execution */
};

#define SYNO_MAX_RANK 16
#define SYNO_MAX_WEIGHTS 16

typedef struct {
  int32_t n_weights;
  int32_t x_rank, y_rank, batch_rank;
  int64_t x_shape[SYNO_MAX_RANK]; /* batch + input dims */
  int64_t y_shape[SYNO_MAX_RANK]; /* batch + output dims */
  int32_t w_rank[SYNO_MAX_WEIGHTS];
  int64_t w_shape[SYNO_MAX_WEIGHTS][SYNO_MAX_RANK];
  int64_t flops_unstaged; /* codegen.flops(graph, assignment, staged=False) */
  int64_t flops_staged;   /* codegen.flops(graph, assignment, staged=True) */
  int64_t params;         /* codegen.param_count */
  int32_t n_forward_stages;
  int32_t grad_x_scatter; /* 1: grad-input uses the atomic scatter form */
  int32_t grad_w_scatter[SYNO_MAX_WEIGHTS];
  int64_t index_grid;     /* points of the unstaged batch-explicit loop grid */
  int32_t complete;       /* frontier matches the input (pgraph.match_input) */
  int32_t replay_only;    /* compiled with SYNO_REPLAY_ONLY: shapes/flops not filled */
  int32_t tc_path;        /* tcgen05 path for fp32 / bf16: 1 conv-shaped implicit GEMM, 2 gathered GEMM, 0 none */
} syno_info;

/* Parse an operator document (pgraph.print_operator format), replay its
 * steps, lower it under `assignment_kv` ("N=8,C_in=64,..."; NULL = the
 * document's reference values; when given it REPLACES them, as the
 * reference's `assignment` argument does) and build the execution plan. */
int syno_compile(const char* op_document, const char* assignment_kv, int flags, syno_op_t* out);

/* y = interpret(graph, x, w).  n_w must equal the operator's weight count. */
/* codegen.parse_loop_nest (codegen.py:846-943) + run_nest's operator:
 * parse loop-nest text (emit_loop_nest's grammar) under the spec of an
 * operator document (its operator/var/output/input/batch lines; a steps
 * line is optional and ignored) into a handle.  The handle runs the nest as
 * run_nest does: x without batch axes.  A single-stage nest is a complete
 * operator (forward, backward, tensor cores); a multi-stage (rfactored) nest
 * runs forward only.  Malformed text is SYNO_E_PARSE (LoopNestParseError). */
int syno_compile_nest(const char* spec_document, const char* nest_text, const char* assignment_kv, int flags,
                      syno_op_t* out);

int syno_forward(syno_op_t op, int dtype, const void* x, const void* const* w, int n_w, void* y, void* stream);

/* Gradients of <dy, interpret(graph, x, w)>.  dx may be NULL; dw may be
 * NULL or hold NULL entries for weights whose gradient is not wanted. */
int syno_backward(syno_op_t op, int dtype, const void* x, const void* const* w, int n_w, const void* dy,
                  void* dx, void* const* dw, void* stream);

/* syno_backward with flags.  SYNO_BWD_X_UNCHANGED / SYNO_BWD_W_UNCHANGED
 * promise that x / the weights hold the same values as in the most recent
 * syno_forward of this handle on this stream (the autograd contract for
 * saved inputs): operand layouts derived from them in that forward may be
 * reused.  The library still checks that the pointers match and recomputes
 * otherwise. */
enum { SYNO_BWD_X_UNCHANGED = 1, SYNO_BWD_W_UNCHANGED = 2 };
int syno_backward_ex(syno_op_t op, int dtype, const void* x, const void* const* w, int n_w, const void* dy,
                     void* dx, void* const* dw, int flags, void* stream);

int syno_query(syno_op_t op, syno_info* info);

/* Text forms; *len receives the full length (buffer may be too small). */
int syno_emit_loop_nest(syno_op_t op, int staged, char* buf, size_t cap, size_t* len);
int syno_print_operator(syno_op_t op, char* buf, size_t cap, size_t* len);
int syno_describe_plan(syno_op_t op, char* buf, size_t cap, size_t* len);

/* K1 parity hook: raw int64 value of coordinate `coord` of term `term`
 * (0 = x, 1.. = weights) of the unstaged, batch-explicit stage at every
 * point of its loop grid (row-major: batch, output axes, reduces).
 * out_dev must hold info.index_grid int64 values. */
int syno_index_map(syno_op_t op, int term, int coord, int64_t* out_dev, void* stream);

/* Search-side shape distance (shapedist.py).
 *
 * syno_shape_distance   shapedist.shape_distance / explain_distance  shapedist.py:377-412
 * syno_graph_distance   shapedist.graph_distance                     shapedist.py:415-420
 * syno_shape_distance_clear_cache  shapedist.clear_cache             shapedist.py:423-433
 *
 * Sizes are monomials: frontier dim k has dim_nterms[k] (variable id,
 * exponent) int32 pairs, consecutive in dim_terms (input dims likewise in
 * in_terms); variable ids are any non-negative ints the caller chooses (the
 * distance does not depend on the naming).  dim_flags[k]: bit 0 reduce_pure,
 * bit 1 strided.  *out receives the distance (+inf when no grouping is
 * valid).  When dim_group / in_group / n_groups are non-null they receive
 * one optimal grouping (explain_distance's witness): the group index of
 * every frontier dim and every input dim, and the group count.  The memo is
 * process-wide and thread-safe. */
int syno_shape_distance(int n_dims, const int32_t* dim_nterms, const int32_t* dim_terms, const uint8_t* dim_flags,
                        int n_inputs, const int32_t* in_nterms, const int32_t* in_terms, int may_reduce,
                        double* out, int32_t* dim_group, int32_t* in_group, int32_t* n_groups);
int syno_graph_distance(syno_op_t op, double* out);
void syno_shape_distance_clear_cache(void);

void syno_destroy(syno_op_t op);
const char* syno_last_error(void);
const char* syno_version(void);

/* The reference's tensor file format (codegen.save_tensor / load_tensor,
 * codegen.py:950-976): rank, then dims, as little-endian int64; float64
 * row-major payload.  syno_tensor_read fills dims (up to SYNO_MAX_RANK) and,
 * when data is non-null and cap >= the element count, the payload; a short
 * or inconsistent file is SYNO_E_SHAPE (ShapeMismatch in the reference). */
int syno_tensor_write(const char* path, int rank, const int64_t* dims, const double* data);
int syno_tensor_read(const char* path, int* rank, int64_t* dims, double* data, int64_t cap, int64_t* count);

/* Kernels this library has launched in this process (all handles, all
 * devices); bench.py reports the difference across its timed region. */
uint64_t syno_launch_count(void);

/* Per-kernel-class timing (measurement only; no reference counterpart).
 * Between syno_profile_begin() and syno_profile_end() every library launch
 * is bracketed by CUDA events on the stream it is issued to; end()
 * synchronises those events and returns one row per kernel class with the
 * launch count, summed device milliseconds and the summed ALGORITHMIC
 * FLOPs / bytes of the launches (codegen.flops per contraction GEMM).
 * While profiling is active the library serialises its launches on the
 * caller's stream (the concurrent grad-weight side stream is not used), so
 * per-launch durations never overlap and their sum is at most the step.
 * Must not be active during CUDA-graph capture. */
typedef struct {
  char name[48];
  int64_t launches;
  double ms;
  double flops;
  double bytes;
} syno_kernel_stat;

void syno_profile_begin(void);
int syno_profile_end(syno_kernel_stat* out, int cap, int* n);

#ifdef __cplusplus
}
#endif

#endif /* SYNO_H_ */
