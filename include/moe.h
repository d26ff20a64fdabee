/*
 * moe.h -- C ABI of libmoe_b200.so: the HetuMoE (arXiv 2203.14685) token-
 * routing hot path, hand-written for B200 (sm_100a).
 *
 * The calls follow Algorithm 1, "General MoE Training Process"
 * (PAPER.md:41-68):
 *
 *   W_(S,E), id_S = Gate(x_S)                    step 1  -> moe_gate
 *   x'_S = Layout_Transform(x_S, id_S)           step 2  -> moe_layout
 *   x'_S = AllToAll(x'_S)                        step 3  -> moe_alltoall
 *   y_i += w_(i,idx) * e_idx(x_i)                step 4  (experts: out of scope;
 *                                                         bench stand-in moe_expert_scale)
 *   y_S = AllToAll(y_S)                          step 5  -> moe_alltoall
 *   y_S = Reverse_Layout_Transform(y_S, id_S)    step 6  -> moe_reverse_layout
 *
 * Conventions (apply to every call unless stated otherwise):
 *  - Pointers named as tensors are DEVICE pointers (cudaMalloc / torch CUDA
 *    memory of the current device).  Host-only calls say "host".
 *  - Every device call is asynchronous on `stream` (a cudaStream_t; NULL =
 *    legacy default stream) and enqueues no host synchronisation.
 *  - All memory is caller-owned.  The library allocates nothing on the hot
 *    path; it only owns moe_comm_t (the NCCL communicator) and the symmetric
 *    peer-mapped buffers of the one-sided NVLink path (moe_comm_symm_alloc).
 *  - Arguments are validated on the host BEFORE anything is enqueued: on any
 *    error nothing was launched, the status says which class of error, and
 *    moe_last_error() (thread-local) names the argument and the values.
 *  - Index arrays are int32, row-major, item index i = t*k + j for token t
 *    and slot j (j = 0 is the best-scoring choice).
 *  - Readings of points the paper leaves open are DESIGN.md §3 "R<n>".
 */
#ifndef MOE_B200_H
#define MOE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Binary compatible with cudaStream_t (driver_types.h declares the same). */
typedef struct CUstream_st* moe_stream_t;

typedef enum {
  MOE_OK = 0,
  MOE_ERR_INVALID_ARG = 1, /* bad size, enum, NULL pointer, shape mismatch   */
  MOE_ERR_UNSUPPORTED = 2, /* valid but outside this build's limits          */
  MOE_ERR_ALIGNMENT = 3,   /* pointer or row size not 16-byte aligned        */
  MOE_ERR_WORKSPACE = 4,   /* workspace NULL or smaller than *_workspace_bytes */
  MOE_ERR_CUDA = 5,        /* a CUDA launch / runtime call failed            */
  MOE_ERR_NCCL = 6,        /* an NCCL call failed                            */
  MOE_ERR_TIMEOUT = 7      /* a device barrier gave up waiting for a peer    */
} moe_status_t;

typedef enum { MOE_F32 = 0, MOE_BF16 = 1 } moe_dtype_t;

/* Gate kinds (§3.1):
 *   TOPK  : Eq. 1 top-k; k=1 is Switch, k=2 is GShard
 *   KTOP1 : M6-T k-top-1, k prototypes of E/k contiguous experts each, top-1
 *           inside every prototype, outputs summed (R11)
 *   HASH  : Hash layer, expert = table[token_id], k = 1 */
typedef enum {
  MOE_GATE_TOPK = 0,
  MOE_GATE_KTOP1 = 1,
  MOE_GATE_HASH = 2,
  MOE_GATE_SAM = 3, /* hierarchical top-k (SAM): moe_gate_ex  */
  MOE_GATE_D2S = 4  /* Dense-to-Sparse, k == E: moe_gate_ex    */
} moe_gate_kind_t;

/* Combine weights (R1):
 *   RENORM  : Eq. 1 literally, g = softmax over the k selected logits
 *             (k-top-1: softmax of one logit = 1; hash: 1)
 *   SOFTMAX : full-row (k-top-1: prototype-slice) softmax evaluated at the
 *             selected experts, not renormalised (Switch-paper convention) */
typedef enum { MOE_W_RENORM = 0, MOE_W_SOFTMAX = 1 } moe_weight_mode_t;

/* Capacity admission order (R5): TOKEN = items (t,j) t-major;
 * SLOT = j-major, all first choices before any second choice (GShard). */
typedef enum { MOE_PRIO_TOKEN = 0, MOE_PRIO_SLOT = 1 } moe_priority_t;

/* AllToAll algorithms:
 *   FLAT        : one grouped send/recv to every peer (Fig. 5)
 *   HIER_LEADER : the paper's hierarchical scheme mimicked with groups of
 *                 `group_size` consecutive ranks on one box (Fig. 6, R13)
 *   P2P         : one-sided: SM stores straight into the peers' receive
 *                 buffers over NVLink (recv must be a symmetric buffer,
 *                 moe_comm_symm_alloc), between two device-side barriers
 *   HIER_2D     : two-level decoupled form: an exchange inside
 *                 each group of `group_size` ranks, then one aggregated
 *                 message per group pair between ranks of equal local index
 *                 (every rank works; no leader), R21.
 * (SURVEY §8(b) numbered HIER_2D 2; P2P took slot 2 first.) */
typedef enum {
  MOE_A2A_FLAT = 0,
  MOE_A2A_HIER_LEADER = 1,
  MOE_A2A_P2P = 2,
  MOE_A2A_HIER_2D = 3
} moe_a2a_algo_t;

/* Gate problem description.  Enums are carried as int32 for a fixed ABI. */
typedef struct {
  int32_t S;           /* tokens on this rank (x_S of Alg. 1), >= 1          */
  int32_t E;           /* number of experts, 1..256                          */
  int32_t k;           /* slots per token: top-k k; k-top-1 prototypes; hash 1 */
  int32_t capacity;    /* per-expert capacity cap >= 1 (see moe_capacity)    */
  int32_t kind;        /* moe_gate_kind_t                                    */
  int32_t weight_mode; /* moe_weight_mode_t                                  */
  int32_t priority;    /* moe_priority_t                                     */
} moe_gate_desc_t;

/* Routing decision W_(S,E), id_S of Alg. 1, stored sparsely.
 * All arrays are caller-allocated device memory. */
typedef struct {
  int32_t* expert_idx; /* [S*k] chosen expert, descending logit order
                          (ties -> lower index, R3); -1 only for an invalid
                          hash id                                            */
  int32_t* slot_idx;   /* [S*k] row inside the expert's buffer, in [0,cap),
                          or -1 = dropped by capacity                        */
  float* weight;       /* [S*k] combine weight w_(t,idx); 0 where dropped,
                          survivors NOT renormalised (R6)                    */
  int32_t* load;       /* [E]   requests per expert before capacity          */
  int32_t* slot_src;   /* [E*cap] inverse map t*k+j, -1 for an empty slot;
                          may be NULL (not produced)                         */
} moe_routing_t;

/* ---------------------------------------------------------------- gate */

/* host.  cap = ceil(C*S*k/E) evaluated in double ("capacity
 * factor C to force the max received tokens by each expert"; formula
 * SPEC.md:138; R4).  S is this rank's token count.  Returns -1 if S, E, k < 1,
 * C <= 0 or the result does not fit in int32. */
int32_t moe_capacity(int32_t S, int32_t E, int32_t k, double C);

/* host.  Device workspace moe_gate needs for `desc` (0 if desc is invalid):
 * per-tile, per-expert counts and the invalid-hash-id counter.  Zero-fill it
 * once before first use (the counter); it may then be reused by any number of
 * calls and CUDA-graph replays on one stream.  Do not use one workspace from
 * two streams concurrently. */
size_t moe_gate_workspace_bytes(const moe_gate_desc_t* desc);

/* host.  How many kernels one moe_gate / moe_gate_ex call enqueues for
 * `desc` with the default tuning (2 or 3; -1 if desc is invalid or the
 * count is decided at launch).  For launch accounting (bench.py). */
int32_t moe_gate_kernel_count(const moe_gate_desc_t* desc, int32_t n_groups);

/* Step 1 of Algorithm 1 plus capacity:
 * selection (TOPK: Eq. 1 TopK on raw fp32 logits, R2; KTOP1: per-prototype
 * argmax; HASH: table lookup), weights (Eq. 1 softmax, R1) and capacity
 * slots (per-expert prefix sum in admission order, slot >= cap -> dropped).
 *   logits    [S,E] fp32 row-major, 16-byte aligned (TOPK, KTOP1; ignored
 *             for HASH)
 *   token_ids [S] int32, table [vocab] int32 (HASH only; else may be NULL)
 *   out       routing arrays (see moe_routing_t); all written
 *   ws        workspace of >= moe_gate_workspace_bytes(desc) bytes
 * Device-side preconditions (not checked synchronously): logits finite;
 * for HASH 0 <= token_ids[t] < vocab and 0 <= table[v] < E -- a violating
 * token is routed as dropped (expert_idx = slot_idx = -1, weight 0) and
 * counted in ws (read it with moe_gate_check).
 * Errors: INVALID_ARG (S<1, E<1, k<1 or k>E, cap<1, KTOP1 with E%k != 0,
 * HASH with k != 1 or missing ids/table/vocab, bad enum, NULL output),
 * UNSUPPORTED (E > 256; SLOT priority with k*E > 2048), WORKSPACE. */
moe_status_t moe_gate(const moe_gate_desc_t* desc, const float* logits,
                      const int32_t* token_ids, const int32_t* table, int32_t vocab,
                      const moe_routing_t* out, void* ws, size_t ws_bytes,
                      moe_stream_t stream);

/* Inputs of every gate kind, for moe_gate_ex. */
typedef struct {
  const float* logits;       /* [S,E] fp32, 16-byte aligned (all but HASH)         */
  const int32_t* token_ids;  /* [S] (HASH)                                          */
  const int32_t* table;      /* [vocab] (HASH)                                      */
  int32_t vocab;             /* (HASH)                                              */
  const float* group_logits; /* [S,n_groups] fp32 (SAM): the Switch Router's scores */
  int32_t n_groups;          /* SAM: experts in n_groups contiguous groups of E/n   */
  const float* uniforms;     /* [S,E] fp32 in (0,1) (D2S train: Gumbel draws); NULL
                                = eval (no noise).  Random numbers are inputs: the
                                caller owns the generator.                          */
  double tau;                /* D2S temperature > 0                                 */
  double eps;                /* D2S prune threshold >= 0 (SPEC: 1e-3)               */
} moe_gate_inputs_t;

/* moe_gate for every gate kind (the same routing outputs and workspace).
 * SAM (R17): group g = argmax of group_logits[t] (lowest index on ties),
 *   then the top-k (k <= E/n_groups, k <= 8) of the logits of experts
 *   [g*E/n, (g+1)*E/n); weights: RENORM = softmax over the k selected;
 *   SOFTMAX = P(g) * P(e | g) (group softmax x within-group softmax).
 * D2S (R18): desc->k must equal E.  z_e = (l_e + G_e)/tau, G_e =
 *   -log(-log(u_e)) (0 without uniforms), p = softmax(z) over all E; experts
 *   with p_e < eps are pruned; survivors fill slots 0..k'-1 in descending z
 *   (ties: lower index) with weight p_e / sum_survivors p (RENORM) or p_e
 *   (SOFTMAX); pruned slots get expert_idx = slot_idx = -1, weight 0.  All in
 *   fp64, one rounding; then capacity over the survivors as for every gate.
 * Errors: as moe_gate; INVALID_ARG for SAM without group_logits or with
 *   E % n_groups != 0 or k > E/n_groups, D2S with k != E, tau <= 0, eps < 0;
 *   UNSUPPORTED for SAM with k > 8. */
moe_status_t moe_gate_ex(const moe_gate_desc_t* desc, const moe_gate_inputs_t* in,
                         const moe_routing_t* out, void* ws, size_t ws_bytes,
                         moe_stream_t stream);

/* Steps 1 + 2 fused: exactly moe_gate_ex followed by
 * moe_layout (same routing outputs, same dispatch buffer, bit for bit), as
 * ONE persistent kernel: tiles of tokens are gated in order of a device-side
 * counter, each resolves its per-expert slot offsets by a decoupled
 * look-back over earlier tiles and scatters its rows at once, so the gate's
 * latency hides behind the row traffic.  TOKEN priority,
 * TOPK / KTOP1 with k <= 8 and HASH, rows a multiple of 32 bytes; other
 * shapes run moe_gate_ex then moe_layout.  Uses the same workspace as
 * moe_gate.  Errors: as moe_gate_ex and moe_layout. */
moe_status_t moe_gate_layout(const moe_gate_desc_t* desc, const moe_gate_inputs_t* in,
                             const moe_routing_t* out, void* ws, size_t ws_bytes, const void* x,
                             int32_t d, int32_t dtype, void* dispatch, moe_stream_t stream);

/* host, SYNCHRONISES `stream`.  Number of invalid hash tokens seen since the
 * last check (the counter is reset to 0). */
moe_status_t moe_gate_check(void* ws, moe_stream_t stream, int32_t* bad_count);

/* ---------------------------------------------------------------- layout */

/* Step 2, Layout_Transform (§3.2 "tokens assigned to the same
 * expert need to be put in physically continuous memory locations",
 * PAPER.md:175-177), padded form (R9):
 *   dispatch[e][s][:] = x[t][:]  for every admitted item (t,j) with
 *                                e = expert_idx[t*k+j], s = slot_idx[t*k+j];
 *   dispatch[e][s][:] = 0        for s in [min(load[e],cap), cap).
 * x [S,d] and dispatch [E,cap,d] have element type `dtype`; the copy is
 * bit-exact.  Uses expert_idx, slot_idx, load of `routing`.
 * Errors: INVALID_ARG, ALIGNMENT (x/dispatch not 16-byte aligned or d*size
 * not a multiple of 16 bytes). */
moe_status_t moe_layout(const moe_gate_desc_t* desc, const moe_routing_t* routing,
                        const void* x, int32_t d, int32_t dtype, void* dispatch,
                        moe_stream_t stream);

/* Step 6 with the weighted combine of step 4, Reverse_Layout_Transform
 * (PAPER.md:56-59, 64-65):
 *   y[t][:] = sum_{j = 0..k-1, slot_idx >= 0} weight[t*k+j] * back[e][s][:]
 * accumulated in fp32 in ascending j from 0, rounded once to dtype (RNE);
 * a token with every slot dropped gets y[t] = 0 (R7).
 * back [E,cap,d], y [S,d] of `dtype`.  Uses expert_idx, slot_idx, weight.
 * Errors: as moe_layout. */
moe_status_t moe_reverse_layout(const moe_gate_desc_t* desc, const moe_routing_t* routing,
                                const void* back, int32_t d, int32_t dtype, void* y,
                                moe_stream_t stream);

/* Bench stand-in for the expert (step 4; R16), NOT part of the method:
 *   out[src][le][s][:] = s_e * in[src][le][s][:],  e = e_base + le,
 *   s_e = 1 + (e mod 8)/8  (bit-reproducible: one rounding of an exact product)
 * in/out [nsrc][E_local][cap][d] of dtype; in == out is allowed. */
moe_status_t moe_expert_scale(const void* in, void* out, int32_t nsrc, int32_t E_local,
                              int32_t e_base, int32_t cap, int32_t d, int32_t dtype,
                              moe_stream_t stream);

/* ---------------------------------------------------------------- dropless packed form
 * SURVEY §8(f) NEXT-4.  SPEC's Permutation: the admitted
 * rows grouped by expert ascending, within an expert in admission order
 * (slot), no padding.  With capacity >= every load (e.g. S*k) nothing is
 * dropped: exact hash-gate semantics without a padding tax. */

/* offsets[e] = sum_{e' < e} min(load[e'], capacity), e = 0..E; offsets[E]
 * = R, the admitted rows.  One tiny kernel (E <= 256).  offsets: [E+1]
 * int32 device. */
moe_status_t moe_expert_offsets(const moe_gate_desc_t* desc, const moe_routing_t* routing,
                                int32_t* offsets, moe_stream_t stream);

/* packed[offsets[e] + s][:] = x[t][:] for every admitted (t,j) at (e,s).
 * packed: [>= offsets[E], d] of dtype (size it for the worst case S*k rows
 * to avoid reading offsets[E] on the host).  Errors: as moe_layout. */
moe_status_t moe_layout_packed(const moe_gate_desc_t* desc, const moe_routing_t* routing,
                               const int32_t* offsets, const void* x, int32_t d, int32_t dtype,
                               void* packed, moe_stream_t stream);

/* y[t] = sum_{j ascending, admitted} weight[t*k+j] * back[offsets[e] + s]
 * (fp32 accumulate, one RNE store; 0 if every slot was dropped). */
moe_status_t moe_reverse_layout_packed(const moe_gate_desc_t* desc,
                                       const moe_routing_t* routing, const int32_t* offsets,
                                       const void* back, int32_t d, int32_t dtype, void* y,
                                       moe_stream_t stream);

/* ---------------------------------------------------------------- backward
 * SURVEY §8(f) NEXT-1.  Algorithm 1 is a training process (PAPER.md:26-28,
 * 41-68); these are the adjoints of its routing steps, with the routing of
 * the forward (expert_idx, slot_idx, weight, load) held fixed.  The AllToAll
 * steps are their own adjoints with the direction swapped (moe_alltoall with
 * the roles of send/recv exchanged), so a backward pass is
 *   moe_reverse_layout_backward -> moe_alltoall -> (expert backward) ->
 *   moe_alltoall -> moe_layout_backward, plus moe_gate_backward. */

/* Adjoint of step 6 + the combine, given dy [S,d]
 * and the expert outputs back [E,cap,d] of the forward:
 *   d_back[e][s][:] = weight[t*k+j] * dy[t][:]   for the admitted (t,j) at
 *                     (e,s): the product rounded once to dtype (RNE) --
 *                     bit-identical to an exact product rounded once;
 *   d_back[e][s][:] = 0                          for s in [min(load,cap), cap);
 *   d_weight[t*k+j] = sum_c dy[t][c] * back[e][s][c]  (fp32 accumulate; 0 for
 *                     a dropped slot, whose weight is the constant 0, R6).
 * dy, back, d_back of `dtype`; d_weight [S*k] fp32.  Uses expert_idx,
 * slot_idx, weight, load.  Errors: as moe_layout. */
moe_status_t moe_reverse_layout_backward(const moe_gate_desc_t* desc,
                                         const moe_routing_t* routing, const void* dy,
                                         const void* back, int32_t d, int32_t dtype,
                                         void* d_back, float* d_weight, moe_stream_t stream);

/* Adjoint of step 2, Layout_Transform:
 *   dx[t][:] = sum_{j ascending, slot_idx >= 0} d_dispatch[e][s][:]
 * fp32 accumulate from 0, one RNE store; 0 for a fully dropped token.
 * d_dispatch [E,cap,d], dx [S,d] of dtype.  Errors: as moe_layout. */
moe_status_t moe_layout_backward(const moe_gate_desc_t* desc, const moe_routing_t* routing,
                                 const void* d_dispatch, int32_t d, int32_t dtype, void* dx,
                                 moe_stream_t stream);

/* Adjoint of the gate weights (Eq. 1; R1, R6, R11) w.r.t. the
 * logits [S,E] fp32, selection fixed: with p the Eq. 1 probabilities over the
 * softmax's domain (RENORM top-k: the k selected; SOFTMAX top-k: the row;
 * SOFTMAX k-top-1: the prototype slice) and g_j = d_weight[t*k+j] for an
 * admitted slot, 0 for a dropped one:
 *   d_logits[t][e] = sum_j g_j p_j (delta(e, e_j) - p_e)  on the domain, 0
 *   elsewhere; k-top-1 RENORM weights are constant: d_logits = 0.
 * Evaluated in fp64, rounded once to fp32.  Errors: INVALID_ARG (HASH has no
 * logits; NULL pointers), as moe_gate's description checks. */
moe_status_t moe_gate_backward(const moe_gate_desc_t* desc, const float* logits,
                               const moe_routing_t* routing, const float* d_weight,
                               float* d_logits, moe_stream_t stream);

/* moe_gate_backward for every gate with logits, the NEXT-3 gates included
 * (R17-R19), selection fixed; inputs as given to moe_gate_ex:
 *  SAM RENORM : as top-k RENORM; d_group_logits = 0.
 *  SAM SOFTMAX: w_j = P(g) q(e_j), q = softmax over group g:
 *               d_logits[e] = sum_j g_j w_j (delta(e, e_j) - q_e) on group g,
 *               d_group_logits[h] = sum_j g_j w_j (delta(h, g) - P(h)).
 *  D2S        : z = (l + G)/tau; q = softmax of z over the survivors (RENORM)
 *               or the row (SOFTMAX): d_logits[e] = (1/tau) sum_j g_j w_j
 *               (delta(e, e_j) - q_e) on that domain, 0 for pruned experts.
 * g_j = d_weight for an admitted slot, 0 otherwise.  fp64, one rounding.
 * d_group_logits [S, n_groups] fp32 (SAM only; else ignored). */
moe_status_t moe_gate_backward_ex(const moe_gate_desc_t* desc, const moe_gate_inputs_t* in,
                                  const moe_routing_t* routing, const float* d_weight,
                                  float* d_logits, float* d_group_logits, moe_stream_t stream);

/* Adjoints of the dropless packed form (NEXT-4): as moe_reverse_layout_backward
 * / moe_layout_backward with row (e, s) at offsets[e] + s and no padding
 * rows (d_back rows >= offsets[E] are not written). */
moe_status_t moe_reverse_layout_packed_backward(const moe_gate_desc_t* desc,
                                                const moe_routing_t* routing,
                                                const int32_t* offsets, const void* dy,
                                                const void* back, int32_t d, int32_t dtype,
                                                void* d_back, float* d_weight,
                                                moe_stream_t stream);
moe_status_t moe_layout_packed_backward(const moe_gate_desc_t* desc,
                                        const moe_routing_t* routing, const int32_t* offsets,
                                        const void* d_packed, int32_t d, int32_t dtype, void* dx,
                                        moe_stream_t stream);

/* ---------------------------------------------------------------- AllToAll */

typedef struct moe_comm moe_comm_t;

/* host.  A fresh NCCL unique id (128 bytes) on rank 0, to be broadcast to the
 * other ranks by the caller (e.g. torch.distributed over gloo). */
moe_status_t moe_comm_unique_id(uint8_t id[128]);

/* host, collective over all ranks, blocking.  Creates the library-owned NCCL
 * communicator on the CURRENT CUDA device.  *out is owned by the caller until
 * moe_comm_destroy. */
moe_status_t moe_comm_init(const uint8_t id[128], int32_t nranks, int32_t rank,
                           moe_comm_t** out);
moe_status_t moe_comm_destroy(moe_comm_t* comm);
moe_status_t moe_comm_size(const moe_comm_t* comm, int32_t* nranks, int32_t* rank);

/* host, SYNCHRONISES `stream` (the stream the communicator's calls use).
 * Failure detection: MOE_OK, or
 *   MOE_ERR_TIMEOUT -- a device barrier of this rank waited longer than the
 *     tuning's barrier_timeout_ms for a peer (a rank died, hung, or skipped
 *     a matching call) and gave up; the stream went on with incomplete
 *     data and the ranks' barrier epochs are out of step: the communicator
 *     is unusable (moe_comm_abort).  The condition is sticky.
 *   MOE_ERR_NCCL -- ncclCommGetAsyncError reports an error.
 * A bounded barrier cannot hang the stream; an NCCL collective waiting on
 * a dead peer can: call moe_comm_abort from another host thread. */
moe_status_t moe_comm_check(moe_comm_t* comm, moe_stream_t stream);

/* host.  ncclCommAbort (unblocks this rank's NCCL kernels), then releases
 * the symmetric buffers and frees comm, without waiting for the peers. */
moe_status_t moe_comm_abort(moe_comm_t* comm);

/* host.  Device memory from ncclMemAlloc, registered with the communicator
 * (ncclCommRegister) so NCCL's send/recv move it without staging through its
 * own buffers (zero-copy over NVLink).  For moe_alltoall / moe_alltoallv
 * send and receive buffers.  Freed by moe_comm_mem_free or destroy. */
moe_status_t moe_comm_mem_alloc(moe_comm_t* comm, size_t bytes, void** ptr);
moe_status_t moe_comm_mem_free(moe_comm_t* comm, void* ptr);

/* host.  Device workspace moe_alltoall needs (0 for FLAT and P2P; for
 * HIER_LEADER the leader's staging, 2 * group_size * nranks * bytes_per_peer
 * (members need none); for HIER_2D 2 * nranks * bytes_per_peer on every
 * rank).  (SURVEY §8(b) took the communicator; this takes its size.) */
size_t moe_alltoall_workspace_bytes(int32_t nranks, int32_t algo, int32_t group_size,
                                    size_t bytes_per_peer);

/* Steps 3 and 5 (§3.2 "each GPU sends its data to all
 * GPUs ... where each data will be divided equally into n parts",
 * PAPER.md:179).  send and recv are [P][bytes_per_peer]:
 *   recv[q] (on rank r) = send[r] (on rank q)   for all q
 * i.e. chunks arrive in ascending source rank.  With the padded
 * layout [E][cap][d] = [P][E/P][cap][d] and experts in contiguous blocks of
 * E/P per rank (R10), dispatch and combine are this same call.
 * FLAT: one NCCL group of send/recv pairs with every peer (self included).
 * HIER_LEADER: groups of group_size consecutive ranks; (1) members send to
 * their leader (local rank 0) sub-messages addressed by destination group,
 * (3) leaders exchange one aggregated message per group pair (B*G/N bytes,
 * PAPER.md:213), (4) the leader permutes chunks by destination device, (5)
 * scatters.  HIER_2D: (0) local transpose [dst group][dst local] ->
 * [dst local][dst group], (1) exchange inside the group, (2) local
 * transpose, (3) one message of group_size chunks (B*G/P bytes) to the rank
 * of equal local index in every group.  Results byte-identical to FLAT (R13).
 * Collective: every rank must call it with the same algo, group_size and
 * bytes_per_peer, in the same order relative to its other NCCL calls.
 * send != recv when nranks > 1 (nranks == 1: a device copy, or nothing if
 * send == recv).  Errors: INVALID_ARG (nranks % group_size, in-place),
 * WORKSPACE (HIER_LEADER on a leader, HIER_2D), NCCL. */
moe_status_t moe_alltoall(moe_comm_t* comm, int32_t algo, int32_t group_size,
                          const void* send, void* recv, size_t bytes_per_peer,
                          void* ws, size_t ws_bytes, moe_stream_t stream);

/* ---------------------------------------------------------------- one-sided NVLink path
 * the layout transform fused with the dispatch AllToAll,
 * with rows stored by the SMs straight into the owner rank's memory over
 * NVLink peer mappings.  Needs GPUs that can map each other's memory (all
 * GPUs of an NVSwitch box); otherwise these calls return UNSUPPORTED. */

/* host, collective, blocking.  Allocates `bytes` of device memory on every
 * rank, zero-filled, mapped into every peer (CUDA IPC).  The library owns it;
 * free it with moe_comm_symm_free (collective) or moe_comm_destroy. */
moe_status_t moe_comm_symm_alloc(moe_comm_t* comm, size_t bytes, void** local);
moe_status_t moe_comm_symm_free(moe_comm_t* comm, void* local);

/* Device-side barrier of all ranks, enqueued on `stream`: returns (in stream
 * order) once every rank's stream has reached its matching barrier; all
 * memory writes made before it (including stores into peers' symmetric
 * buffers) are visible to every rank after it. */
moe_status_t moe_comm_barrier(moe_comm_t* comm, moe_stream_t stream);

/* Flags of the one-sided calls (default 0: both barriers, no assumption).
 * MOE_P2P_NO_ENTRY_BARRIER / MOE_P2P_NO_EXIT_BARRIER skip the entry / exit
 * device barrier.  The entry barrier guarantees no rank writes into
 * (dispatch) or reads from (combine) a peer's buffer before that peer's
 * stream reached the call, and (combine) that every rank's writes into the
 * buffer -- its expert's, and the library's own duplicate-row copies after a
 * deduped moe_dispatch_p2p -- are complete; the exit barrier that every
 * store landed (dispatch) / every read finished (combine).  A caller that
 * orders its steps itself (e.g. moe_comm_barrier after its expert) may skip
 * redundant ones, e.g. dispatch(NO_ENTRY) after a combine with its exit
 * barrier.  The tables the senders write into an owner during a dispatch
 * (padding counts, duplicate rows) belong to its receive buffer (allocated
 * collectively on the first dispatch into that buffer outside stream capture;
 * released with it), so a caller that ALTERNATES two receive buffers A, B --
 * dispatch(A) combine(A) dispatch(B) combine(B) dispatch(A) ... on every
 * rank -- may give every combine NO_EXIT_BARRIER and every dispatch after the
 * first into its buffer NO_ENTRY_BARRIER: a rank that dispatches into A again
 * has passed the exit barrier of the dispatch into B, which no rank reaches
 * before its combine of A has finished reading.  Exception: a combine of a buffer whose last moe_dispatch_p2p
 * sent some token rows once for two slots (k >= 2, two experts of the token
 * on one remote owner, tuning p2p_dedupe) keeps its entry barrier under
 * NO_ENTRY_BARRIER, because the owners' duplicate-row copies run after the
 * dispatch's exit barrier -- unless MOE_P2P_RECV_UNMODIFIED is also given.
 * MOE_P2P_RECV_UNMODIFIED (combine only): the caller asserts that nothing
 * wrote expert_out since the moe_dispatch_p2p that filled it (an identity
 * expert); the combine then reads such a slot from the row that was sent
 * (one read for both slots, no wait for the copies).  Passing it after an
 * expert wrote the buffer gives wrong results (undefined). */
enum {
  MOE_P2P_NO_ENTRY_BARRIER = 1,
  MOE_P2P_NO_EXIT_BARRIER = 2,
  MOE_P2P_RECV_UNMODIFIED = 4
};

/* Steps 2+3 fused: for every admitted item (t,j) with
 * expert e and slot s, the row x[t] is stored into rank q = e/(E/P)'s
 * `recv` at [r][e mod E/P][s] (r = this rank); padding rows
 * [min(load[e],cap), cap) are zeroed there; bracketed by moe_comm_barrier
 * (see flags).  The resulting recv buffers are byte-identical to moe_layout
 * followed by moe_alltoall(FLAT).  recv: symmetric, [P][E/P][cap][d]. */
moe_status_t moe_dispatch_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                              const moe_routing_t* routing, const void* x, int32_t d,
                              int32_t dtype, void* recv, int32_t flags, moe_stream_t stream);

/* Steps 5+6 fused: moe_comm_barrier (every rank's experts
 * are done; see flags), then y[t] = sum_j w[t,j] * expert_out_q[r][e mod E/P][s] with
 * every admitted row read straight from its owner rank q's `expert_out` over
 * NVLink (fp32 accumulate in ascending j, one RNE store, 0 if all slots
 * dropped), then moe_comm_barrier (the buffers may be reused).  Same result
 * as moe_alltoall(FLAT) back + moe_reverse_layout.  With k = 2 after a
 * deduped moe_dispatch_p2p into expert_out (and no RECV_UNMODIFIED), every
 * rank first combines, on its own rows, the token pairs that dispatch sent
 * it once (both slots of a token on this owner; tuning p2p_precombine), and
 * such a token's y row is then read as that one pre-combined row: the same
 * fp32 FMA order and rounding, byte-identical y, half the NVLink reads for
 * those tokens (a symmetric pre-row buffer the size of expert_out is
 * allocated collectively on first use outside stream capture).  Flags: see
 * above (NO_ENTRY_BARRIER, NO_EXIT_BARRIER, RECV_UNMODIFIED).  expert_out:
 * symmetric, [P][E/P][cap][d] of dtype (e.g. the recv of moe_dispatch_p2p). */
moe_status_t moe_combine_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                             const moe_routing_t* routing, const void* expert_out, int32_t d,
                             int32_t dtype, void* y, int32_t flags, moe_stream_t stream);

/* Steps 1 + 2 + 3 fused: moe_gate_ex + moe_dispatch_p2p
 * with the gate and the NVLink row scatter as one persistent kernel (as
 * moe_gate_layout; same dedupe and local padding as moe_dispatch_p2p); same
 * routing and receive buffers, bit for bit.  Shapes without a fused kernel
 * run moe_gate_ex then moe_dispatch_p2p. */
moe_status_t moe_gate_dispatch_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                   const moe_gate_inputs_t* in, const moe_routing_t* out,
                                   void* ws, size_t ws_bytes, const void* x, int32_t d,
                                   int32_t dtype, void* recv, int32_t flags, moe_stream_t stream);

/* Backward of the fused steps over NVLink (adjoints of moe_combine_p2p and
 * moe_dispatch_p2p, same barrier flags).
 * moe_combine_backward_p2p: entry barrier; for every admitted item (t,j) at
 * expert e (owner q) and slot s, reads expert_out_q[r][e mod E/P][s] for
 * d_weight and stores weight * dy[t] into d_expert_out_q[r][e mod E/P][s],
 * zero-fills the padding rows there; exit barrier.  Equals
 * moe_alltoall(FLAT) of expert_out + moe_reverse_layout_backward +
 * moe_alltoall(FLAT) of d_back.  expert_out, d_expert_out: symmetric
 * [P][E/P][cap][d]; d_weight [S*k] fp32 local. */
moe_status_t moe_combine_backward_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                      const moe_routing_t* routing, const void* dy,
                                      const void* expert_out, int32_t d, int32_t dtype,
                                      void* d_expert_out, float* d_weight, int32_t flags,
                                      moe_stream_t stream);

/* moe_combine_backward_push_p2p: the same outputs as moe_combine_backward_p2p
 * with half the NVLink bytes: dy rows (the dispatch kernel) and the slot
 * weights are pushed to the experts' owners, each owner scales the rows in
 * place into d_expert_out (same exact rounding) and dots them with its
 * LOCAL expert_out rows, writing the results into the token owner's dw
 * table, from which d_weight is read.  wtab, dwtab: symmetric fp32
 * [E*cap] scratch.  Ends with barriers; d_expert_out is final on return
 * (in stream order). */
moe_status_t moe_combine_backward_push_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                           const moe_routing_t* routing, const void* dy,
                                           const void* expert_out, int32_t d, int32_t dtype,
                                           void* d_expert_out, float* wtab, float* dwtab,
                                           float* d_weight, int32_t flags, moe_stream_t stream);

/* Adjoints of the dropless NVLink exchange (NEXT-1 x NEXT-4): as
 * moe_combine_backward_p2p / moe_dispatch_backward_p2p with rows at
 * peer_base[q] + offsets[e] - offsets[q*E/P] + s of the owner's buffer
 * (the layout moe_dispatch_packed_p2p produced; pass its peer_base), no
 * padding rows.  rows: the symmetric buffers' row count (>= nranks*S*k). */
moe_status_t moe_combine_packed_backward_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                            const moe_routing_t* routing, const int32_t* offsets,
                                            const int32_t* peer_base, const void* dy,
                                            const void* expert_out, int32_t d, int32_t dtype,
                                            int64_t rows, void* d_expert_out, float* d_weight,
                                            int32_t flags, moe_stream_t stream);
moe_status_t moe_dispatch_packed_backward_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                             const moe_routing_t* routing, const int32_t* offsets,
                                             const int32_t* peer_base, const void* d_recv,
                                             int32_t d, int32_t dtype, int64_t rows, void* dx,
                                             int32_t flags, moe_stream_t stream);

/* moe_dispatch_backward_p2p: entry barrier; dx[t] = sum_j d_recv_q[r][e mod
 * E/P][s] read from each owner q over NVLink (fp32 accumulate, one RNE
 * store); exit barrier.  Equals moe_alltoall(FLAT) + moe_layout_backward.
 * d_recv: symmetric [P][E/P][cap][d]. */
moe_status_t moe_dispatch_backward_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                       const moe_routing_t* routing, const void* d_recv,
                                       int32_t d, int32_t dtype, void* dx, int32_t flags,
                                       moe_stream_t stream);

/* host.  The plan of the NCCL dropless exchange from this rank's expert
 * offsets [E+1] (moe_expert_offsets, copied to the host) and the per-expert
 * row counts it receives, recv_counts[src*E/P + le] (an AllToAll of the
 * [P][E/P] count tables): send_rows[q] = rows for rank q's experts,
 * recv_rows[q] = rows from rank q, recv_offsets[E+1] = where (src, le)
 * starts in the receive buffer (source-rank major, R20).  Experts are
 * contiguous blocks of E/P per rank (R10).  All arrays host memory. */
moe_status_t moe_alltoallv_plan(int32_t nranks, int32_t E, const int32_t* offsets,
                                const int32_t* recv_counts, int64_t* send_rows,
                                int64_t* recv_rows, int32_t* recv_offsets);

/* Variable-size AllToAll (the NCCL dropless exchange): rank r sends
 * send_rows[q] rows of row_bytes to every rank q, taken consecutively from
 * `send` in ascending q, and receives recv_rows[q] rows from every q into
 * `recv`, consecutively in ascending q (SPEC's alltoallv).  send_rows /
 * recv_rows are HOST arrays [nranks] (exchange the per-expert counts first,
 * e.g. moe_alltoall(FLAT) of an int32 [P][E/P] count table, and read them on
 * the host).  Collective.  Errors: INVALID_ARG, NCCL. */
moe_status_t moe_alltoallv(moe_comm_t* comm, const void* send, const int64_t* send_rows,
                           void* recv, const int64_t* recv_rows, size_t row_bytes,
                           moe_stream_t stream);

/* Dropless dispatch over NVLink, no host synchronisation: the count
 * exchange and the offsets are computed on the device.
 *  1. (entry barrier) rank r stores its per-expert admitted counts for rank
 *     q's experts into q's symmetric `counts` [P][E/P] int32 at row r;
 *     barrier;
 *  2. peer_base[q] = rows earlier ranks put into q's recv (read from q's
 *     counts); recv_offsets[src*E/P + le] = where rank src's rows of local
 *     expert le start in this rank's recv (prefix over `counts`), [E+1];
 *  3. every admitted row x[t] of (e,s) is stored into q = e/(E/P)'s `recv`
 *     at row peer_base[q] + offsets[e] - offsets[q*E/P] + s; (exit barrier).
 * recv layout: source-rank major, then local expert, then slot -- equal to
 * moe_alltoallv of moe_layout_packed.  recv: symmetric, recv_cap_rows rows,
 * which must be >= nranks*S*k (the worst case: everything to one rank).
 * offsets: this rank's moe_expert_offsets; peer_base [P], recv_offsets
 * [E+1] int32 device outputs (keep them for the combine). */
moe_status_t moe_dispatch_packed_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                     const moe_routing_t* routing, const int32_t* offsets,
                                     int32_t* counts, int32_t* peer_base, int32_t* recv_offsets,
                                     const void* x, int32_t d, int32_t dtype, void* recv,
                                     int64_t recv_cap_rows, int32_t flags, moe_stream_t stream);

/* Dropless combine over NVLink: (entry barrier) y[t] = sum_j w[t,j] *
 * expert_out_q[peer_base[q] + offsets[e] - offsets[q*E/P] + s] read from
 * each owner q (fp32 accumulate, one RNE store); (exit barrier).
 * expert_out: symmetric, recv layout of moe_dispatch_packed_p2p. */
moe_status_t moe_combine_packed_p2p(moe_comm_t* comm, const moe_gate_desc_t* desc,
                                    const moe_routing_t* routing, const int32_t* offsets,
                                    const int32_t* peer_base, const void* expert_out, int32_t d,
                                    int32_t dtype, int64_t expert_out_rows, void* y,
                                    int32_t flags, moe_stream_t stream);

/* One step of an AllToAll schedule, as executed by moe_alltoall.  Exported
 * (host) so the schedule can be checked without GPUs.  Buffers: 0 = send,
 * 1 = recv, 2 = ws staging A, 3 = ws staging B (each half of the
 * workspace).  Offsets/bytes are in units of bytes_per_peer chunks. */
typedef struct {
  int32_t phase; /* ops of one phase: the SEND/RECVs as one NCCL group, then
                    the local ops in order; phases in order                 */
  int32_t op;    /* 0 = SEND, 1 = RECV, 2 = COPY (local), 3 = PERMUTE
                    (dst (n,g,m) <- src (g,m,n)), 4 = TRANSPOSE (dst [y][x]
                    <- src [x][y])                                         */
  int32_t peer;  /* SEND/RECV: peer rank; PERMUTE: N (groups); TRANSPOSE: X */
  int32_t src_buf, dst_buf;
  int64_t src_off, dst_off, chunks; /* PERMUTE: G (group size); TRANSPOSE: Y */
} moe_a2a_op_t;

/* host.  Fills ops[0..*n_ops) with rank `rank`'s schedule; returns
 * INVALID_ARG if capacity is too small (*n_ops then holds the count needed). */
moe_status_t moe_alltoall_plan(int32_t nranks, int32_t rank, int32_t algo, int32_t group_size,
                               moe_a2a_op_t* ops, int32_t capacity, int32_t* n_ops);

/* ---------------------------------------------------------------- simulated ranks
 * TEST INFRASTRUCTURE: P ranks of the multi-GPU path simulated on ONE GPU,
 * so every exchange step (Alg. 1 steps 3 and 5) is
 * parity-testable without NVLink.  A world owns P simulated communicators
 * (each a moe_comm_t* usable with every call above that takes one).  Their
 * symmetric buffers are P ordinary allocations on the current device, each
 * mapped to its "peers" directly.  Calls on a simulated rank validate their
 * arguments and then do NOT launch: they append their steps to the rank's
 * program.  moe_sim_world_run executes every rank's program on `stream`:
 * kernels of a rank in its call order; a device barrier waits until every
 * rank reached its matching barrier (a step boundary, no spinning kernel);
 * NCCL send/recv groups are matched across the ranks in issue order per
 * (source, destination) and executed as device copies.  The kernels are the
 * ones the real path launches (same peer-pointer tables, same flags).
 * No NCCL communicator exists; moe_comm_check of a simulated rank reads its
 * device error word.  Not for production use. */
typedef struct moe_sim_world moe_sim_world_t;

/* host.  nranks in 1..32.  Allocates the signal buffers on the current
 * device. */
moe_status_t moe_sim_world_create(int32_t nranks, moe_sim_world_t** out);
/* host.  The simulated communicator of `rank` (owned by the world). */
moe_status_t moe_sim_world_comm(moe_sim_world_t* w, int32_t rank, moe_comm_t** out);
/* Execute (enqueue on `stream`) every rank's queued steps, then clear them.
 * INVALID_ARG if the programs do not match (a rank reaches a barrier or a
 * send that no other rank matches); what ran before stays enqueued. */
moe_status_t moe_sim_world_run(moe_sim_world_t* w, moe_stream_t stream);
/* host.  Enqueue ONE rank's real barrier kernel (k_barrier on the world's
 * signal words, bounded by the tuning's barrier_timeout_ms), for testing the
 * timeout: with no other rank arriving it gives up and sets the rank's error
 * word (moe_comm_check -> MOE_ERR_TIMEOUT).  Only one spinning kernel runs. */
moe_status_t moe_sim_live_barrier(moe_sim_world_t* w, int32_t rank, moe_stream_t stream);
/* host.  Synchronises the device and frees everything the world owns. */
moe_status_t moe_sim_world_destroy(moe_sim_world_t* w);

/* ---------------------------------------------------------------- tuning
 * Kernel-variant choices of the row movers and the gate.  Every default is
 * the measured-best one; the other values select variants
 * that compute the SAME bits (the parity tests run each).  One process-wide
 * table: it is filled once, at the first call into the library, from the
 * MOE_<FIELD> environment variables (upper case, e.g. MOE_GATE_TILES) when
 * set; moe_set_tuning replaces it.  No call reads the environment after
 * that.  "auto" = decided per call from the shapes, as documented. */
typedef struct {
  int32_t gate_tiles;        /* gate: aim for >= this many tiles (256)             */
  int32_t gate_max_tile;     /* gate (and the fused gate + layout): largest tile in
                                tokens; 0 = auto (128 for logit gates, 256 for
                                hash)                                              */
  int32_t gate_two_maxw;     /* gate: tiles x columns <= this -> select + slots2,
                                else select + scan + slots (4096)                  */
  int32_t layout_u;          /* layout: 32-byte vectors per lane per segment;
                                0 = auto (2 for rows <= 2 KiB, else 4); 1, 2, 4    */
  int32_t layout_pads_first; /* layout + combine adjoint: zero the padding rows
                                before the token rows; -1 = auto (local buffers
                                with >= 5% padding by construction), 0, 1          */
  int32_t reverse_ku;        /* combine (k <= 2): vectors in flight per lane;
                                0 = auto (2 for local k = 2, else 4); 2, 4         */
  int32_t reverse_tpw;       /* combine (k = 1): two tokens per warp round on
                                rows <= 2 KiB; -1 = auto (on), 0, 1                */
  int32_t reverse_kspec;     /* combine: 1 = the k <= 2 specialised kernel, 0 =
                                the generic one (1)                                */
  int32_t reverse_backwards; /* combine: walk tokens last to first; -1 = auto
                                (local buffers), 0, 1                              */
  int32_t reverse_y_ef;      /* combine: evict-first y stores; -1 = auto (local), 0, 1 */
  int32_t row_ctas_per_sm;   /* row movers: CTAs per SM; 0 = occupancy limit       */
  int32_t reverse_ctas_per_sm; /* local combine (moe_reverse_layout): CTAs per SM;
                                0 = row_ctas_per_sm                                */
  int32_t combine_ctas_per_sm; /* NVLink combine (moe_combine_p2p and the packed and
                                adjoint peer reads): CTAs per SM; 0 = row_ctas_per_sm
                                (8: measured 5% faster than the occupancy limit)  */
  int32_t combine_bwd_kspec; /* combine adjoint: k <= 2 specialised kernel (1)      */
  int32_t gate_bwd_lanes;    /* gate adjoint: lanes per token; 0 = auto (~8 experts
                                per lane)                                          */
  int32_t p2p_dedupe;        /* one-sided dispatch: a token's row crosses once per
                                owner (1)                                          */
  int32_t p2p_local_pad;     /* one-sided dispatch: owners zero their own padding
                                rows; -1 = auto (>= 5% padding by construction)    */
  int32_t a2a_ctas_per_sm;   /* moe_alltoall(P2P): CTAs per SM (4)                 */
  int32_t barrier_timeout_ms;/* device barriers give up after this long and
                                report MOE_ERR_TIMEOUT (moe_comm_check); 0 = wait
                                forever (60000)                                    */
  int32_t barrier_pdl;       /* device barrier launched with programmatic dependent
                                launch (1)                                         */
  int32_t disable_p2p;       /* moe_comm_init: do not map peer memory (0)          */
  int32_t nccl_alltoall;     /* moe_alltoall(FLAT): 1 = ncclAlltoAll, 0 = one group
                                of ncclSend/ncclRecv pairs (0)                     */
  int32_t nccl_max_ctas;     /* moe_comm_init: ncclConfig_t maxCTAs; 0 = NCCL's    */
  int32_t nccl_min_ctas;     /* moe_comm_init: ncclConfig_t minCTAs; 0 = NCCL's    */
  int32_t nccl_cta_policy;   /* moe_comm_init: ncclConfig_t CTAPolicy (0 default, 1
                                efficiency, 2 zero); -1 = NCCL's                   */
  int32_t layout_tokens_per_warp; /* local layout: grid of ceil(S / (8 warps x this))
                                CTAs (at least the persistent grid), which the
                                block scheduler balances over the SMs; 0 = the
                                persistent grid (row_ctas_per_sm) (2)              */
  int32_t p2p_precombine;    /* NVLink combine, k = 2 after a deduped dispatch: each
                                owner first combines the token pairs it received
                                once (one rounding, the same result), and the
                                token's owner reads one row instead of two (1)    */
} moe_tuning_t;

/* host.  Copy of the current table (after the one-time environment read). */
moe_status_t moe_get_tuning(moe_tuning_t* out);
/* host.  Replace the table.  INVALID_ARG (and no change) if a field is out of
 * its range.  Affects calls made after it returns; not synchronised with
 * calls running on other host threads. */
moe_status_t moe_set_tuning(const moe_tuning_t* t);

/* host.  PROFILING: a device buffer of `bytes` that the fused gate + layout
 * kernel (moe_gate_layout, moe_gate_dispatch_p2p) fills with %globaltimer
 * stamps (ns, uint64) on every launch made while it is set: words 0..2 =
 * n_tiles, n_chunks, CTAs; from word 4: per tile of the gate [claim,
 * aggregate published, prefix published, ready] at 4*tile, per 32-token
 * scatter chunk [claim, its tile seen ready] at 4*n_tiles + 2*chunk, per CTA
 * [start, end] after those; stamps beyond `bytes` are dropped.  The separate
 * gate (moe_gate, select -> slots2) fills the same buffer with words 0..3 =
 * n_tiles, 16, 0, 2 and, per tile, 16 words from 4 + 16*tile: k_gate_select
 * [entry, after its grid-dependency wait, logits staged, selection done,
 * in-tile ranks, tile aggregate, end] at 0..6, k_gate_slots2 [entry, after
 * its wait, prefixes reduced, end] at 8..11 (select -> scan -> slots:
 * k_gate_slots [entry, after its wait, end] at 8, 9, 11 and k_gate_scan's
 * CTA b [entry, after its wait, its warp 0 done] at 12..14 of tile b's
 * words).  The row kernels of moe_layout / the one-sided
 * dispatch and of moe_reverse_layout / the one-sided combine stamp [entry,
 * after the grid-dependency wait, end] per CTA at word 4*cta of the buffer's
 * second half (layout) and last quarter (reverse).
 * NULL (or 0 bytes) turns it off.  Affects launches made after it returns
 * (a captured graph keeps the buffer it was captured with). */
moe_status_t moe_set_trace(void* buf, size_t bytes);

/* ---------------------------------------------------------------- misc */

const char* moe_status_str(moe_status_t s);
const char* moe_last_error(void);   /* thread-local detail of the last error */
const char* moe_version(void);      /* build string: arch, NCCL version      */

#ifdef __cplusplus
}
#endif
#endif /* MOE_B200_H */
