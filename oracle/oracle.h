/*
 * oracle.h -- plain, slow, single-threaded CPU oracle of the HetuMoE
 * (arXiv 2203.14685) token-routing path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load liboracle.so.
 * The product path (paper_2203_14685_b200/) never links, loads or calls it,
 * and this file shares no code, header, table or helper with the CUDA path.
 *
 * Every function follows the paper's definition written out literally, in
 * double precision, in the paper's order (Algorithm 1):
 *   Gate (step 1) -> Layout_Transform (step 2) -> AllToAll (step 3)
 *   -> expert (step 4; here the fixed per-expert scale stand-in)
 *   -> AllToAll (step 5) -> Reverse_Layout_Transform (step 6).
 * Readings of points the paper leaves open are listed in DESIGN.md §3 and
 * cited below as "R<n>".
 *
 * Parity pins: every function here is pinned by tests/test_oracle_*.py
 * against closed forms, brute force, hand-worked golden examples
 * (tests/golden/) and library routines.  See DESIGN.md §4 for the pin map.
 */
#ifndef MOE_ORACLE_H
#define MOE_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* gate kinds / modes: same numbering as the public header by convention, but
 * defined independently here (the oracle includes nothing from include/). */
enum { ORC_TOPK = 0, ORC_KTOP1 = 1, ORC_HASH = 2 };
enum { ORC_RENORM = 0, ORC_SOFTMAX = 1 };
enum { ORC_PRIO_TOKEN = 0, ORC_PRIO_SLOT = 1 };
enum { ORC_F32 = 0, ORC_BF16 = 1 };

/* capacity = ceil(C*S*k/E), evaluated in double left to right (R4;
 * PAPER.md:97 "capacity factor C to force the max received tokens";
 * formula SPEC.md:138).  Returns -1 for invalid arguments. */
int32_t orc_capacity(int32_t S, int32_t E, int32_t k, double C);

/* Step 1 of Algorithm 1: W_(S,E), id_S = Gate(x_S), on
 * given logits (x.W is out of scope), followed by the
 * capacity replay.  Outputs are indexed t*k+j.
 *   expert_idx: chosen expert, -1 only for an invalid hash id
 *   slot_idx  : position inside the expert's buffer, -1 = dropped
 *   weight    : combine weight, 0 where dropped (no renormalisation, R6)
 *   load      : [E] requests per expert before capacity
 *   slot_src  : [E*cap] t*k+j or -1 for an empty slot (may be NULL)
 * Returns the number of invalid hash ids (0 for the other gates), or -1
 * for invalid arguments. */
int64_t orc_gate(int kind, int weight_mode, int priority,
                 int32_t S, int32_t E, int32_t k, int32_t cap,
                 const float* logits, const int32_t* token_ids,
                 const int32_t* table, int32_t vocab,
                 int32_t* expert_idx, int32_t* slot_idx, float* weight,
                 int32_t* load, int32_t* slot_src);

/* Hierarchical top-k / SAM (R17): experts in n_groups
 * contiguous groups of n = E/n_groups; group g = argmax of the group logits
 * [S,n_groups] (the Switch Router), then the top-k (k <= n) of the expert
 * logits inside group g (the Mixture Router).  Weights: RENORM = softmax
 * over the k selected logits; SOFTMAX = P(g) * P(e | g) (group softmax times
 * the within-group softmax, not renormalised).  Capacity as orc_gate.
 * Returns 0, or -1 for invalid arguments. */
int64_t orc_gate_sam(int weight_mode, int priority, int32_t S, int32_t E, int32_t k,
                     int32_t cap, int32_t n_groups, const float* group_logits,
                     const float* logits, int32_t* expert_idx, int32_t* slot_idx,
                     float* weight, int32_t* load, int32_t* slot_src);

/* Dense-to-Sparse (R18): k = E candidate slots per token.
 * z_e = (l_e + G_e)/tau with G_e = -log(-log(u_e)) (train: uniforms [S,E]
 * in (0,1)) or 0 (eval: uniforms NULL); p = softmax(z) over all E; experts
 * with p_e < eps are pruned; survivors fill slots 0..k'-1 in descending z
 * (ties: lower index), weight p_e / sum_survivors p (RENORM) or p_e
 * (SOFTMAX); pruned slots j >= k' get expert -1, slot -1, weight 0.
 * Capacity as orc_gate over the survivors.  Returns 0, or -1 for invalid
 * arguments. */
int64_t orc_gate_d2s(int weight_mode, int priority, int32_t S, int32_t E, int32_t cap,
                     double tau, double eps, const float* logits, const float* uniforms,
                     int32_t* expert_idx, int32_t* slot_idx, float* weight, int32_t* load,
                     int32_t* slot_src);

/* Step 2: dispatch[e][s][:] = x[t][:] for every
 * admitted (t,j), padded layout [E][cap][row] with zeroed padding (R9).
 * Byte copy: dtype agnostic. */
void orc_layout(int32_t S, int32_t E, int32_t k, int32_t cap, int64_t row_bytes,
                const int32_t* expert_idx, const int32_t* slot_idx,
                const void* x, void* dispatch);

/* Step 6 + the combine loop of step 4:
 * y[t] = sum_{j ascending, slot>=0} w[t,j] * back[idx][slot], accumulated in
 * double, rounded once to dtype (RNE).  Fully dropped tokens give 0 (R7). */
void orc_reverse_layout(int dtype, int32_t S, int32_t E, int32_t k, int32_t cap,
                        int32_t d, const int32_t* expert_idx,
                        const int32_t* slot_idx, const float* weight,
                        const void* back, void* y);

/* Bench stand-in for step 4 (R16): out[src][le][s][:] = s_e * in, with
 * e = e_base + le and s_e = 1 + (e mod 8)/8.  Buffer layout
 * [nsrc][E_local][cap][d]. */
void orc_expert_scale(int dtype, int32_t nsrc, int32_t E_local, int32_t e_base,
                      int32_t cap, int32_t d, const void* in, void* out);

/* Steps 3/5, flat (Fig. 5): recv_r[q] = send_q[r]: chunk q of
 * rank r's receive buffer is chunk r of rank q's send buffer (ascending
 * source rank).  send[p], recv[p] are P host buffers of
 * P*bytes_per_peer bytes each. */
void orc_alltoall_flat(int32_t P, int64_t bytes_per_peer,
                       const void* const* send, void* const* recv);

/* Message statistics of one simulated collective. */
typedef struct {
  int64_t intra_msgs;       /* messages between ranks of one group (incl. self) */
  int64_t inter_msgs;       /* messages crossing groups                         */
  int64_t inter_msg_bytes;  /* bytes of one cross-group message (uniform)       */
  int64_t intra_bytes;      /* total bytes moved inside groups                  */
  int64_t inter_bytes;      /* total bytes moved across groups                  */
} orc_a2a_stats_t;

/* Steps 3/5, hierarchical (Fig. 6), simulated as the five
 * explicit phases of SPEC.md:324 with groups of G consecutive ranks and the
 * leader = local rank 0 (R13): (1) gather into the leader, (2) reorder by
 * destination group, (3) leader-to-leader exchange, (4) reorder by
 * destination device, (5) scatter.  Returns 0, or -1 if P % G != 0. */
int orc_alltoall_hier(int32_t P, int32_t G, int64_t bytes_per_peer,
                      const void* const* send, void* const* recv,
                      orc_a2a_stats_t* stats);

/* Flat message statistics for the same P, G split (for the G^2 pin). */
void orc_alltoall_flat_stats(int32_t P, int32_t G, int64_t bytes_per_peer,
                             orc_a2a_stats_t* stats);

/* ---- Dropless packed layout (SPEC.md:241-256
 * "Permutation": rows grouped by expert ascending, within an expert in
 * admission order -- a stable counting sort; no padding rows). */

/* offsets[e] = sum_{e' < e} min(load[e'], cap), e = 0..E (offsets[E] = R,
 * the number of admitted slots). */
void orc_expert_offsets(int32_t E, int32_t cap, const int32_t* load, int32_t* offsets);

/* packed[offsets[e] + s][:] = x[t][:] for every admitted (t,j) at (e,s);
 * [offsets[E]][row] bytes.  Byte copy. */
void orc_layout_packed(int32_t S, int32_t E, int32_t k, int64_t row_bytes,
                       const int32_t* expert_idx, const int32_t* slot_idx,
                       const int32_t* offsets, const void* x, void* packed);

/* y[t] = sum_{j ascending, admitted} w[t,j] * back[offsets[e] + s] (double,
 * one rounding); 0 for a fully dropped token. */
void orc_reverse_layout_packed(int dtype, int32_t S, int32_t E, int32_t k, int32_t d,
                               const int32_t* expert_idx, const int32_t* slot_idx,
                               const float* weight, const int32_t* offsets,
                               const void* back, void* y);

/* Variable-size AllToAll (the dropless exchange): rank q sends rows
 * counts[q*P + r] to rank r, taken consecutively from send[q] in ascending
 * r; recv[r] = the segments of every q in ascending q.  Rows of row_bytes. */
void orc_alltoallv(int32_t P, int64_t row_bytes, const int64_t* counts,
                   const void* const* send, void* const* recv);

/* ---- Backward of the routing path: Algorithm 1 is a
 * training process, so each forward step has an
 * adjoint.  Routing (expert_idx, slot_idx, weight) is the forward's output and
 * is held fixed (selection and capacity are piecewise constant in the
 * inputs). */

/* Adjoint of step 6 + the combine, y[t] =
 * sum_j w[t,j] * back[e_j][s_j]:
 *   d_back[e][s]  = w[t,j] * dy[t]             for the admitted (t,j) at (e,s),
 *                   0 for every empty slot      (double product, one rounding)
 *   d_weight[t,j] = sum_c dy[t][c] * back[e_j][s_j][c]   (double, one rounding;
 *                   0 for a dropped slot: its weight is the constant 0, R6) */
void orc_reverse_layout_bwd(int dtype, int32_t S, int32_t E, int32_t k, int32_t cap,
                            int32_t d, const int32_t* expert_idx,
                            const int32_t* slot_idx, const float* weight,
                            const void* dy, const void* back, void* d_back,
                            float* d_weight);

/* Adjoint of step 2, dispatch[e_j][s_j] = x[t]:
 *   dx[t] = sum_{j ascending, admitted} d_dispatch[e_j][s_j]  (double, one
 *   rounding); 0 for a fully dropped token. */
void orc_layout_bwd(int dtype, int32_t S, int32_t E, int32_t k, int32_t cap, int32_t d,
                    const int32_t* expert_idx, const int32_t* slot_idx,
                    const void* d_dispatch, void* dx);

/* Adjoint of the gate weights (Eq. 1; R1, R6, R11) w.r.t. the
 * logits, selection fixed.  The combine uses w'_j = m_j * p_j with m_j = 1
 * for an admitted slot, 0 for a dropped one, and p_j the Eq. 1 probability;
 * so with g_j = d_weight[t,j]:
 *   d_logits[t][e] = sum_j m_j * g_j * dp_j/dl_e
 * where dp_j/dl_e = p_j * (delta(e, e_j) - p_e) over the softmax's domain
 * (RENORM: the k selected logits; SOFTMAX: the row; k-top-1 SOFTMAX: the
 * prototype slice) and 0 outside it.  k-top-1 RENORM weights are the constant
 * 1: zero gradient.  Written out as the Jacobian sum, in double, one
 * rounding.  Returns 0, or -1 for invalid arguments (HASH has no logits). */
int orc_gate_bwd(int kind, int weight_mode, int32_t S, int32_t E, int32_t k,
                 const float* logits, const int32_t* expert_idx, const int32_t* slot_idx,
                 const float* d_weight, float* d_logits);

/* orc_gate_bwd for the NEXT-3 gates (R17, R18, R19), selection fixed:
 *  SAM RENORM : the top-k RENORM adjoint on the expert logits (the k
 *               selected are the domain); no group-logit gradient.
 *  SAM SOFTMAX: w_j = P(g) P(e_j | g):
 *               d_logits[e]       = sum_j m_j g_j w_j (delta(e, e_j) - P(e | g)),
 *                                   e in group g (0 elsewhere);
 *               d_group_logits[h] = sum_j m_j g_j w_j (delta(h, g) - P(h)).
 *  D2S        : over the survivors (RENORM: w = softmax of z over the
 *               survivors) or the row (SOFTMAX: w = softmax of z), z = (l+G)/tau:
 *               d_logits[e] = (1/tau) sum_j m_j g_j w_j (delta(e, e_j) - q_e), q
 *               the same softmax; pruned experts (RENORM) get 0.
 * Jacobian sums in double, one rounding.  group_logits / d_group_logits are
 * used for SAM only, uniforms / tau for D2S only (uniforms NULL = eval).
 * Returns 0, or -1 for invalid arguments. */
int orc_gate_bwd_ex(int kind, int weight_mode, int32_t S, int32_t E, int32_t k,
                    const float* logits, const float* group_logits, int32_t n_groups,
                    const float* uniforms, double tau, const int32_t* expert_idx,
                    const int32_t* slot_idx, const float* d_weight, float* d_logits,
                    float* d_group_logits);

/* bf16 helpers of the oracle's own (R14): exact widening, and a single
 * round-to-nearest-even narrowing from double. */
double   orc_bf16_to_f64(uint16_t h);
uint16_t orc_f64_to_bf16(double v);

#ifdef __cplusplus
}
#endif
#endif
