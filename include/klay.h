/*
 * libklay — B200 (sm_100a) evaluator for layered arithmetic circuits.
 *
 * Plain C ABI: host pointers / device pointers / sizes only, no torch types.
 * Every entry point replaces one function of the reference evaluation engine
 * (/root/reference/pkg/src/laycirc/engine.py); the mapping is cited per call.
 * The reference is pure Python + numpy, so it has no FFI of its own; the
 * binding a maintainer would add is the ctypes stub in INTEGRATION.md, which
 * is exactly what paper_2410_11415_b200/_lib.py does.
 *
 * Value layout ("node-major"): one contiguous device buffer of rows, one row
 * per circuit node, `ld` elements per row (ld >= B, ld*sizeof(T) a multiple
 * of 16 bytes). Row order: the K input slots, then layer 1 .. layer L nodes
 * in the reference's within-layer order (indices are never permuted).
 *
 * Return codes: 0 = ok, otherwise a KLAY_E* code; klay_last_error() gives a
 * thread-local message. All device work is stream-ordered on `stream`
 * (a cudaStream_t; NULL = legacy default stream). No call allocates device
 * memory except klay_plan_create.
 */
#ifndef KLAY_H
#define KLAY_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define KLAY_API __attribute__((visibility("default")))
#else
#define KLAY_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define KLAY_OK 0
#define KLAY_EINVAL 1       /* bad argument / shape (maps to EvalError)       */
#define KLAY_EFORMAT 2      /* circuit invariant violated (KlayFormatError)   */
#define KLAY_ECUDA 3        /* CUDA runtime / launch failure                  */
#define KLAY_EUNSUPPORTED 4 /* semiring/domain combination not defined        */

/* semirings (engine.py:158-193, forward_log 247-282) */
#define KLAY_REAL 0
#define KLAY_LOG 1
#define KLAY_BOOL 2
#define KLAY_MAXPROD 3

/* element types */
#define KLAY_F32 0
#define KLAY_F64 1
#define KLAY_U1 2  /* bit-packed Boolean rows (32 batch rows per 32-bit word);
                      KLAY_BOOL forward only, weights exactly 0/1, `ld` in words,
                      outputs [B, R] 0.0/1.0 in the weights' element type */

typedef struct KlayPlan KlayPlan;

/* Library version string. */
KLAY_API const char* klay_version(void);

/* Thread-local message for the last nonzero return code of this thread. */
KLAY_API const char* klay_last_error(void);

/*
 * Build the immutable device plan of a tensorized circuit and upload it to
 * `device`. Replaces engine._plans (engine.py:138-155): per layer the CSR
 * offsets of the parent segments and the stable, ascending-edge-order
 * transposed CSR (child -> parents) used by the atomic-free backward.
 *
 *   widths[L], edge_counts[L]        per gate layer (TensorLayer.width / num_edges)
 *   sources, segments                concatenation over layers of
 *                                    TensorLayer.sources / .segments (int64,
 *                                    tensorize.py:47-48)
 *   root_nodes[R]                    final-layer index per root position, or -1
 *                                    for a constant root (root_indices +
 *                                    constant_roots, tensorize.py:65-76)
 *   const_vals[R]                    1/0 value of constant roots (ignored else)
 * The structural invariants of tensorize.py:94-132 are re-checked on the
 * host; a violation returns KLAY_EFORMAT.
 */
KLAY_API int klay_plan_create(int64_t num_inputs, int32_t num_layers, const int64_t* widths,
                     const int64_t* edge_counts, const int64_t* sources,
                     const int64_t* segments, int32_t num_roots, const int64_t* root_nodes,
                     const int8_t* const_vals, int32_t device, KlayPlan** out);

KLAY_API int klay_plan_destroy(KlayPlan* plan);

/* Sum of all layer widths including the K input rows (= trace rows). */
KLAY_API int64_t klay_plan_num_nodes(const KlayPlan* plan);
/* Largest row count of any single layer (inputs included). */
KLAY_API int64_t klay_plan_max_width(const KlayPlan* plan);
/* Row offset of layer l (0 = inputs) inside the trace buffer. */
KLAY_API int64_t klay_plan_layer_offset(const KlayPlan* plan, int32_t layer);
/* The plan's schedule (out[8]): out[0] first layer of the persistent
 * (cluster) tail, out[1] / out[2] first layer of the forward / backward (log
 * semiring) micro tail (0-based gate layers; L = none), out[3] number of
 * aliased (never written) rows of a backward-only trace, out[4] / out[5]
 * layers in the forward / backward micro head (0 = none), out[6] rows of the
 * backward's adjoint buffer (node layers with disjoint lifetimes share
 * rows), out[7] rows of the trace. Returns 0, or EINVAL for a null
 * argument. */
KLAY_API int klay_plan_schedule(const KlayPlan* plan, int64_t* out);

/* Smallest legal row stride (elements) for batch B and element type. */
KLAY_API int64_t klay_row_stride(int64_t batch, int32_t dtype);

/*
 * Forward pass. Replaces forward_real / forward_log / evaluate_semiring
 * (engine.py:226-304) including _run_layers (215-223) and _assemble_outputs
 * (203-212).
 *   weights      device [B, K] row-major, element type `weights_dtype`
 *                (values in the semiring's domain: log values for KLAY_LOG)
 *   values       retain != 0: trace buffer [num_nodes, ld] (every layer kept,
 *                EvalTrace.node_values); retain == 0: scratch of
 *                2 * max_width rows (ping-pong, only the last layer survives)
 *   retain       0: no trace; 1: full trace; 2 (KLAY_RETAIN_BACKWARD): the
 *                trace klay_backward needs. With KLAY_LOG and epsilon 0 the
 *                rows of unary gate nodes below the tail (each a copy of its
 *                only child, +inf -> NaN through a sum) are then left
 *                unwritten: readers use the first non-unary row below.
 *                klay_fill_trace() writes them on demand.
 *   outputs      device [B, R] row-major, element type `dtype` (may be NULL)
 *   epsilon      log semiring only, added inside the log (must be >= 0)
 *   workspace    device scratch of klay_forward_workspace() bytes (may be
 *                NULL when that is 0: no segment needs a split reduction)
 */
KLAY_API int klay_forward(const KlayPlan* plan, int32_t semiring, int32_t dtype,
                 const void* weights, int32_t weights_dtype, void* values, int64_t ld,
                 int32_t retain, void* outputs, int64_t batch, double epsilon,
                 void* workspace, void* stream);

#define KLAY_RETAIN_BACKWARD 2

/* Completes a retain = 2 trace of klay_forward(semiring, epsilon): writes the
 * rows of unary nodes from their chains' sources (through a unary sum, a
 * logsumexp of one element: +inf becomes NaN). No-op for traces that left
 * nothing out (any semiring but KLAY_LOG, epsilon != 0). */
KLAY_API int klay_fill_trace(const KlayPlan* plan, int32_t semiring, int32_t dtype, void* values,
                    int64_t ld, int64_t batch, double epsilon, void* stream);

/* Scratch bytes klay_forward needs for row stride `ld` (leaf partials of
 * segments longer than 129 edges, split in numpy pairwise-tree order). */
KLAY_API size_t klay_forward_workspace(const KlayPlan* plan, int32_t dtype, int64_t ld);

/*
 * Backward pass over a retained trace. Replaces engine.backward
 * (engine.py:307-355) with _product_adjoint (358-369): gradient of
 * sum_r seed[:, r] * root_r w.r.t. the K input slots.
 *   domain       KLAY_REAL or KLAY_LOG (the trace's domain)
 *   seed         device [B, R] row-major in `dtype`, or NULL for all-ones
 *   grads        device [B, K] row-major in `dtype`
 *   workspace    device scratch of klay_backward_workspace() bytes
 *   epsilon      the epsilon the (log-domain) trace was computed with
 *                (the reference keeps it in trace.epsilon). Exactly 0 lets
 *                unary sum parents skip their value reads (their weight
 *                exp(child - parent) is then exactly 1, or 0 at -inf); any
 *                other value, e.g. -1 when unknown, reads every parent.
 *   retain       the retain mode klay_forward wrote the trace with (1 full,
 *                2 backward-only). A backward-only log trace with epsilon 0
 *                carries, in unwritten rows, the finiteness masks this
 *                backward uses to send adjoints down chains of unary nodes
 *                in one step; pass 1 for any other (e.g. uploaded) trace.
 */
KLAY_API int klay_backward(const KlayPlan* plan, int32_t domain, int32_t dtype, const void* trace,
                  int64_t ld, const void* seed, void* grads, void* workspace,
                  int64_t batch, double epsilon, int32_t retain, void* stream);

KLAY_API size_t klay_backward_workspace(const KlayPlan* plan, int32_t dtype, int64_t ld);

/* ---- .klay reader ---------------------------------- */

/*
 * Parse and validate `.klay` text (tensorize.py:197-313; the structural rules
 * of tensorize.py:94-132). Rejects, never repairs: KLAY_EFORMAT with the
 * reason in klay_read_klay_error(). Host only (no CUDA).
 *   sizes[7] from klay_file_info: num_inputs, num_vars, num_layers,
 *   num_edges, num_roots, num_constant_roots, inputmap entries.
 * Layer ops alternate product (layer 1) / sum, as validated.
 */
typedef struct KlayFile KlayFile;
KLAY_API int klay_read_klay(const char* text, int64_t len, KlayFile** out);
KLAY_API const char* klay_read_klay_error(void);
KLAY_API int klay_file_info(const KlayFile* file, int64_t* sizes);
KLAY_API int klay_file_export(const KlayFile* file, int64_t* widths, int64_t* counts,
                     int64_t* sources, int64_t* segments, int64_t* roots,
                     int64_t* const_pos, int64_t* const_val, int64_t* lit_codes,
                     int64_t* lit_slots);
KLAY_API void klay_file_destroy(KlayFile* file);

/* ---- host-side layerization ----------------------- */

/*
 * layerize() + tensorize() of one or more constant-folded circuits
 * (laycirc/layerize.py:158-271, tensorize.py:135-194), bit-identical index
 * vectors. Circuits are given as flat arrays (circuit c owns nodes
 * [node_offsets[c], node_offsets[c+1]), ids local to the circuit):
 *   kinds[n]        0 leaf, 1 and, 2 or, 3 true, 4 false
 *   literals[n]     DIMACS literal of a leaf (0 otherwise)
 *   child_offsets   CSR over all nodes (global), children[] = local child ids
 *   roots           root_offsets[c]..[c+1] (local ids); num_vars[c]
 * Read the result with klay_layered_info / _export, free with _destroy.
 * Errors: KLAY_EFORMAT (CircuitError cases) with klay_layerize_error().
 */
typedef struct KlayLayered KlayLayered;
KLAY_API int klay_layerize(int32_t num_circuits, const int64_t* node_offsets, const int8_t* kinds,
                  const int32_t* literals, const int64_t* child_offsets, const int32_t* children,
                  const int64_t* root_offsets, const int32_t* roots, const int32_t* num_vars,
                  KlayLayered** out);
/* 0 num_inputs, 1 num_vars, 2 gate layers, 3 total edges, 4 non-constant
 * roots, 5 constant roots */
KLAY_API int64_t klay_layered_info(const KlayLayered* layered, int32_t what);
KLAY_API int klay_layered_export(const KlayLayered* layered, int64_t* widths, int64_t* edge_counts,
                        int64_t* sources, int64_t* segments, int32_t* input_lits,
                        int64_t* root_indices, int64_t* const_pos, int8_t* const_val);
KLAY_API void klay_layered_destroy(KlayLayered* layered);
KLAY_API const char* klay_layerize_error(void);

/* ---- instrumentation (no counterpart in the reference) ---------------- */

/* Number of kernels this library has launched so far (process-wide). */
KLAY_API int64_t klay_launch_count(void);

/* Time every subsequent launch of this thread with CUDA events on its
 * stream until klay_profiler_end (which synchronizes). Record kinds:
 * 0 = forward layer kernel, 1 = backward layer kernel, 2 = forward
 * boundary (inputs / outputs), 3 = backward boundary (seeds / grads),
 * 4 / 5 = forward / backward persistent tail (layers >= `layers`),
 * 6 / 7 = forward / backward micro tail (the thinnest layers, all >= `layers`);
 * `layers` holds the 1-based gate layer (0 / L+1 for boundary kernels). */
KLAY_API int klay_profiler_begin(void);
KLAY_API int klay_profiler_end(int32_t max_records, int32_t* kinds, int32_t* layers, float* ms,
                      int32_t* n_records);

/* Launch classes (per-template roofline accounting in bench.py). */
#define KLAY_CLASS_FWD_PROD 0     /* forward layer kernel, product layer        */
#define KLAY_CLASS_FWD_SUM 1      /* forward layer kernel, sum layer            */
#define KLAY_CLASS_BWD_PASS 2     /* backward pass-through (incl. route masks)  */
#define KLAY_CLASS_BWD_LOGSUM 3   /* backward log-sum (softmax edge weights)    */
#define KLAY_CLASS_BWD_REALPROD 4 /* backward real product (zero-safe adjoint)  */
#define KLAY_CLASS_FWD_MICRO 5    /* forward micro tail / micro head            */
#define KLAY_CLASS_BWD_MICRO 6    /* backward micro tail / micro head           */
#define KLAY_CLASS_TAIL 7         /* persistent cluster tail (either direction) */
#define KLAY_CLASS_BOUNDARY 8     /* inputs, outputs, seeds, grads              */
/* Profiling hook: launch only the kernels whose class bit is set in
 * `class_mask` on this thread (default all); returns the previous mask.
 * A pass captured with a filter holds just those launches, so it times one
 * template inside a CUDA graph. Results of a filtered pass are garbage. */
KLAY_API uint32_t klay_set_launch_filter(uint32_t class_mask);

#ifdef __cplusplus
}
#endif

#endif /* KLAY_H */
