// Host-visible interface between the C-ABI layer (klay.cu) and the kernel
// translation units (fwd_*.cu, bwd_*.cu, boundary.cu).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace klay {

template <typename T>
struct LayerArgs {
  const int4* items;  // work items of this layer/direction
  const unsigned* masks;  // per item: stage-batch start nodes (short tasks)
  int n_items;
  const int4* heavy;  // {node, first leaf slot, #leaves, 0}
  int n_heavy;
  const int* off;     // segment offsets [nodes+1]
  const int* idx;     // edge -> operand row
  T* out;             // output rows
  T* scratch;         // leaf partials [slots, ld] (+ [slots, ld] t-part for LSE)
  long long tpart;    // element offset of the LSE t-part inside scratch
  int V;              // 16-byte vectors per row
  long long ld;
  T eps;
  // forward operand
  const T* prev;
  // backward operands
  const T* gcur;      // adjoint rows of the layer above (parents)
  const T* ncur;      // forward values of the parents
  const T* nprev;     // forward values of the children (own value x)
  const int* foff;    // forward CSR (real-product zero path)
  const int* fsrc;
  int prod;           // product layer (selects the reduction in the tail kernel)
  int unary_ok;       // backward: edges flagged as unary parents need no parent value
  int* hcount;        // per (heavy segment, chunk) leaf counters: the last leaf combines
                      // (null: a separate combine pass / the tail's own barrier)
  // unary-node aliases (klay.cu build_aliases); all null when off
  //   forward:  omap[j] = row of item node j (compacted sets); xmap[j] = row
  //             of mbase where node j stores its value's finiteness mask, or
  //             -1 (mbase null: no masks)
  //   backward: omap[j] = output row (absolute; bit 31: weight the adjoint by
  //             the value's finiteness), xmap[j] = own-value row (absolute):
  //             the child's value (log-sum layers) or the row holding its
  //             mask (pass-through layers)
  const int* omap;
  const int* xmap;
  T* mbase;
  // padded per-item index data (klay.cu pad_items; PADW ints per item):
  // edge indices, raw segment offsets, and for alias sets omap / xmap entries
  const int* pidx;
  const int* poff;
  const int* pmap;
  const int* pxmap;
  int rev;            // visit the column chunks last to first (L2 reuse across launches)
  // streaming path (stream_kernels.cuh): node ranges of the CTAs (n_scta + 1
  // entries over this set's nodes); spv / sring are set at launch
  const int* scta;
  int n_scta;
  int spv, sring;
  unsigned long long* trace;  // KLAY_STREAM_TRACE builds: per-CTA timing records (debug)
  ChkRanges chk;              // KLAY_CHECKS builds: valid byte ranges + violation record
};

// The persistent tail kernel (thin upper layers in one launch) takes its
// per-layer arguments by value as a __grid_constant__ kernel parameter.
constexpr int TAIL_MAX_LAYERS = 96;
template <typename T>
struct TailArgs {
  LayerArgs<T> layer[TAIL_MAX_LAYERS];
  int n;
  // plan-data ranges of all tail layers (indices, offsets, items, masks), pulled
  // into L2 at kernel start so no layer waits on DRAM for its structure
  const void* pf_ptr[4];
  long long pf_bytes[4];
  int debug_skip;  // KLAY_TAIL_DEBUG=1: barriers only (timing experiments; wrong results)
  unsigned long long* trace_ts;  // KLAY_TAIL_TRACE=1: per-layer globaltimer stamps (debug)
};

// The micro tails: the thin top layers (widths <= MICRO_WF / MICRO_WB, fan-in
// / fan-out <= MICRO_FAN, one layer's CSR <= MICRO_CSRF / MICRO_CSRB ints) evaluated by one
// CTA per column chunk with the layer values held in shared memory. Each
// layer's CSR (offsets local from 0, then indices) is packed at a 16-byte
// aligned offset of one plan int array and staged per layer.
constexpr int MICRO_MAX_LAYERS = 64;
constexpr int MICRO_P = 2;        // 16-byte pieces per CTA column chunk (32 bytes)
#ifndef KLAY_MICRO_WF
#define KLAY_MICRO_WF 1280
#endif
constexpr int MICRO_WF = KLAY_MICRO_WF;  // forward: two row sets of 32-byte chunks
#ifndef KLAY_MICRO_WB
#define KLAY_MICRO_WB 1280
#endif
constexpr int MICRO_WB = KLAY_MICRO_WB;  // backward: four row sets of 32-byte chunks
constexpr int MICRO_FAN = 129;
constexpr int MICRO_HEAD_W = 256;  // widths of micro-head layers (the thin bottom)
constexpr int MICRO_CSRF = 8192;  // ints per staged layer CSR
constexpr int MICRO_CSRB = 8192;
template <typename T>
struct MicroArgs {
  const T* in;                    // rows of the layer below the first micro layer
  T* out[MICRO_MAX_LAYERS];       // output rows per layer (null: not stored)
  int w[MICRO_MAX_LAYERS];        // widths
  int csr_at[MICRO_MAX_LAYERS];   // offset of the layer's [W+1 offsets, E indices] in csr
  int csr_n[MICRO_MAX_LAYERS];    // its length (ints)
  int prod[MICRO_MAX_LAYERS];
  const int* csr;
  int n, w_in, V;
  long long ld;
  T eps;
  ChkRanges chk;
};
// backward micro tail: steps i = 0.. walk the micro layers top down; step i
// computes the children's adjoints of one layer
template <typename T>
struct MicroBwdArgs {
  const T* gin;                     // adjoint rows of the top layer (seeded)
  T* gout[MICRO_MAX_LAYERS];        // children's adjoint rows per step (null: not stored)
  const T* vpar[MICRO_MAX_LAYERS];  // forward values of the parents / children
  const T* vchild[MICRO_MAX_LAYERS];
  int wp[MICRO_MAX_LAYERS];         // parents (layer width) / children (width below)
  int wc[MICRO_MAX_LAYERS];
  int csr_at[MICRO_MAX_LAYERS];     // [wc+1 transposed offsets, E parent indices] in csr
  int csr_n[MICRO_MAX_LAYERS];
  int logsum[MICRO_MAX_LAYERS];     // weighted edges (log sum / real product) or pass-through
  const int* csr;
  int n, w_top, V, unary_ok;
  long long ld;
  ChkRanges chk;
};
int launch_backward_micro(int domain, const MicroBwdArgs<float>& m, cudaStream_t s);
int launch_backward_micro(int domain, const MicroBwdArgs<double>& m, cudaStream_t s);
int launch_forward_micro(int sr, const MicroArgs<float>& m, cudaStream_t s);
int launch_forward_micro(int sr, const MicroArgs<double>& m, cudaStream_t s);
int launch_forward_micro_u1(const MicroArgs<unsigned>& m, cudaStream_t s);

// forward layer: semiring x layer op -> reduction kind (RK_*)
int launch_forward_layer(int sr, bool prod, bool alias, const LayerArgs<float>& a, cudaStream_t s);
int launch_forward_layer(int sr, bool prod, bool alias, const LayerArgs<double>& a, cudaStream_t s);
// backward layer (BW_* mode): always a pairwise sum over each child's out-edges
int launch_backward_layer(int mode, const LayerArgs<float>& a, cudaStream_t s);
int launch_backward_layer(int mode, const LayerArgs<double>& a, cudaStream_t s);
// the same layers on the bulk-copy streaming kernel (a.scta / a.n_scta set;
// every segment of the set <= MICRO_FAN edges)
int launch_forward_stream(int sr, bool prod, bool alias, const LayerArgs<float>& a, cudaStream_t s);
int launch_forward_stream(int sr, bool prod, bool alias, const LayerArgs<double>& a, cudaStream_t s);
int launch_backward_stream(int mode, const LayerArgs<float>& a, cudaStream_t s);
int launch_backward_stream(int mode, const LayerArgs<double>& a, cudaStream_t s);

// persistent tail: layers t.layer[0..n) in order, one cluster per column
// chunk; returns the number of kernels launched (0 on a launch failure)
int launch_forward_tail(int sr, const TailArgs<float>& t, int cluster, cudaStream_t s);
int launch_forward_tail(int sr, const TailArgs<double>& t, int cluster, cudaStream_t s);
int launch_backward_tail(int domain, const TailArgs<float>& t, int cluster, cudaStream_t s);
int launch_backward_tail(int domain, const TailArgs<double>& t, int cluster, cudaStream_t s);

// bit-packed Boolean forward (dtype KLAY_U1): AND products, OR sums
int launch_forward_layer_u1(bool prod, const LayerArgs<unsigned>& a, cudaStream_t s);
int launch_forward_tail_u1(const TailArgs<unsigned>& t, int cluster, cudaStream_t s);
// 0/1 weights [B, K] (f64 or f32) -> packed node-major rows [K, ldw words];
// sets *bad (device int) when a weight is not exactly 0 or 1
void launch_pack_inputs(const void* w, bool w_f64, unsigned* n0, int K, long long B, long long ldw,
                        int* bad, cudaStream_t s);
// packed root rows -> [B, R] 0.0/1.0 (f64 or f32), constants as given
void launch_unpack_outputs(const unsigned* last, const int* root_node, const signed char* const_val,
                           void* out, bool out_f64, int R, long long B, long long ldw,
                           cudaStream_t s);

// boundary kernels
template <typename T>
void launch_load_inputs(const void* w, bool w_f64, T* n0, int K, long long B, long long ld, T pad,
                        cudaStream_t s);
template <typename T>
void launch_store_rows(const T* rows, T* out, int Q, long long B, long long ld, cudaStream_t s);
template <typename T>
void launch_assemble_outputs(const T* last, const int* root_node, const signed char* const_val,
                             T* out, int R, long long B, long long ld, T zero, T one,
                             cudaStream_t s);
template <typename T>
void launch_seed(const T* seed, const int* top_off, const int* top_pos, T* g, int WL, int R,
                 long long B, long long ld, cudaStream_t s);
template <typename T>
void launch_fill_aliases(const int2* pairs, long long n, T* values, long long ld, cudaStream_t s);

}  // namespace klay
