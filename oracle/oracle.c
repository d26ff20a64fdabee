/*
 * oracle.c -- plain, slow, single-threaded CPU oracle of the HetuMoE
 * (arXiv 2203.14685) token-routing path.  See oracle.h.
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
 * bench.py (cpu_baseline / --impl reference).  Never by the product path.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared (no fast-math), so
 * every double operation below rounds exactly as written.
 *
 * Citations: PAPER.md:<line> [section / equation / algorithm];
 * "R<n>" = reading n of DESIGN.md §3 (where the paper is silent).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* bf16 (R14): bf16 is the top 16 bits of an IEEE binary32.                  */
/* ------------------------------------------------------------------------ */
double orc_bf16_to_f64(uint16_t h) {
  uint32_t bits = (uint32_t)h << 16;
  float f;
  memcpy(&f, &bits, sizeof f);
  return (double)f;
}

/* One rounding, to nearest with ties to even, straight from double: find the
 * spacing of bf16 values (7 fraction bits) around |v|, divide (exact: a power
 * of two), round to an integer with rint() (default mode = nearest-even), and
 * scale back. */
uint16_t orc_f64_to_bf16(double v) {
  if (isnan(v)) return 0x7FC0;
  uint16_t sign = signbit(v) ? 0x8000u : 0u;
  double a = fabs(v);
  if (a == 0.0) return sign;
  int e2;
  (void)frexp(a, &e2);          /* a in [2^(e2-1), 2^e2) */
  int ex = e2 - 1;
  if (ex < -126) ex = -126;      /* subnormal bf16: fixed spacing 2^-133 */
  double ulp = ldexp(1.0, ex - 7);
  double q = rint(a / ulp);
  double r = q * ulp;
  if (r >= ldexp(1.0, 128)) return (uint16_t)(sign | 0x7F80u); /* -> inf */
  float f = (float)r;            /* exact: r has <= 8 significant bits */
  uint32_t bits;
  memcpy(&bits, &f, sizeof bits);
  return (uint16_t)(sign | (uint16_t)(bits >> 16));
}

static double load_elem(int dtype, const void* p, int64_t i) {
  if (dtype == ORC_F32) return (double)((const float*)p)[i];
  return orc_bf16_to_f64(((const uint16_t*)p)[i]);
}

static void store_elem(int dtype, void* p, int64_t i, double v) {
  if (dtype == ORC_F32) ((float*)p)[i] = (float)v;  /* C cast: nearest-even */
  else ((uint16_t*)p)[i] = orc_f64_to_bf16(v);
}

/* ------------------------------------------------------------------------ */
/* Capacity (R4): ceil(C*S*k/E), in double, left to right.                  */
/* ------------------------------------------------------------------------ */
int32_t orc_capacity(int32_t S, int32_t E, int32_t k, double C) {
  if (S < 1 || E < 1 || k < 1 || !(C > 0.0)) return -1;
  double c = ceil(C * (double)S * (double)k / (double)E);
  if (c < 1.0 || c > 2147483647.0) return -1;
  return (int32_t)c;
}

/* ------------------------------------------------------------------------ */
/* Gate selection (Eq. 1; 123-124 kTop1; 144-145 Hash).    */
/* ------------------------------------------------------------------------ */

/* "a beats b": larger raw logit, ties to the lower expert index (R2, R3).
 * Float comparison, so -0.0 and +0.0 tie. */
static int beats(float va, int32_t ia, float vb, int32_t ib) {
  return va > vb || (va == vb && ia < ib);
}

/* Top-k of one row: stable insertion sort of all E indices by `beats`, then
 * the first k (R2).  Slot j = position in that order. */
static void topk_row(const float* row, int32_t E, int32_t k, int32_t* order,
                     int32_t* out) {
  for (int32_t e = 0; e < E; ++e) order[e] = e;
  for (int32_t i = 1; i < E; ++i) {
    int32_t cur = order[i];
    int32_t p = i - 1;
    while (p >= 0 && beats(row[cur], cur, row[order[p]], order[p])) {
      order[p + 1] = order[p];
      --p;
    }
    order[p + 1] = cur;
  }
  for (int32_t j = 0; j < k; ++j) out[j] = order[j];
}

/* Eq. 1 weights, in double, rounded once to float (R1):
 *   RENORM : g = softmax over the k selected logits (Eq. 1 literally);
 *   SOFTMAX: g_j = exp(l_j - m) / sum_{e<E} exp(l_e - m), m = row max. */
static void topk_weights(const float* row, int32_t E, int32_t k, int mode,
                         const int32_t* sel, float* w) {
  double m = (double)row[sel[0]];  /* slot 0 holds the row maximum */
  double den = 0.0;
  if (mode == ORC_RENORM) {
    for (int32_t j = 0; j < k; ++j) den += exp((double)row[sel[j]] - m);
  } else {
    for (int32_t e = 0; e < E; ++e) den += exp((double)row[e] - m);
  }
  for (int32_t j = 0; j < k; ++j)
    w[j] = (float)(exp((double)row[sel[j]] - m) / den);
}

/* kTop1 (R11): prototype p owns experts
 * [p*E/k, (p+1)*E/k); slot j = p is the argmax of that slice, strict '>'
 * scanning upward so the lowest index wins ties.  Weight: RENORM = softmax
 * over the single selected logit = 1; SOFTMAX = the slice-softmax
 * probability of the argmax. */
static void ktop1_row(const float* row, int32_t E, int32_t k, int mode,
                      int32_t* sel, float* w) {
  int32_t n = E / k;
  for (int32_t p = 0; p < k; ++p) {
    int32_t lo = p * n, best = lo;
    for (int32_t e = lo + 1; e < lo + n; ++e)
      if (row[e] > row[best]) best = e;
    sel[p] = best;
    if (mode == ORC_RENORM) {
      w[p] = 1.0f;
    } else {
      double m = (double)row[best], den = 0.0;
      for (int32_t e = lo; e < lo + n; ++e) den += exp((double)row[e] - m);
      w[p] = (float)(1.0 / den);
    }
  }
}

static void capacity_replay(int priority, int32_t S, int32_t E, int32_t k, int32_t cap,
                            const int32_t* expert_idx, int32_t* slot_idx, float* weight,
                            int32_t* load, int32_t* slot_src);

int64_t orc_gate(int kind, int weight_mode, int priority,
                 int32_t S, int32_t E, int32_t k, int32_t cap,
                 const float* logits, const int32_t* token_ids,
                 const int32_t* table, int32_t vocab,
                 int32_t* expert_idx, int32_t* slot_idx, float* weight,
                 int32_t* load, int32_t* slot_src) {
  if (S < 1 || E < 1 || k < 1 || k > E || cap < 1) return -1;
  if (kind == ORC_KTOP1 && E % k != 0) return -1;
  if (kind == ORC_HASH && (k != 1 || !token_ids || !table || vocab < 1)) return -1;
  if (kind != ORC_HASH && !logits) return -1;
  int64_t bad = 0;

  /* 1. selection + weights, token by token */
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
  for (int32_t t = 0; t < S; ++t) {
    int32_t* sel = expert_idx + (int64_t)t * k;
    float* w = weight + (int64_t)t * k;
    if (kind == ORC_TOPK) {
      const float* row = logits + (int64_t)t * E;
      topk_row(row, E, k, order, sel);
      topk_weights(row, E, k, weight_mode, sel, w);
    } else if (kind == ORC_KTOP1) {
      ktop1_row(logits + (int64_t)t * E, E, k, weight_mode, sel, w);
    } else {
      /* Hash layer: expert = table[token_id], weight 1.
       * Out-of-range ids / table entries are routed as dropped (R12). */
      int32_t id = token_ids[t];
      int32_t e = (id >= 0 && id < vocab) ? table[id] : -1;
      if (e < 0 || e >= E) { e = -1; ++bad; }
      sel[0] = e;
      w[0] = (e < 0) ? 0.0f : 1.0f;
    }
  }
  free(order);

  capacity_replay(priority, S, E, k, cap, expert_idx, slot_idx, weight, load, slot_src);
  return bad;
}

/* Capacity (R4, R5, R6): walk the items in admission order;
 * slot = number of earlier items with the same expert; slot >= cap ->
 * dropped, weight 0.  Items with expert -1 (an invalid hash id, a pruned
 * Dense-to-Sparse slot) are not admitted and not counted. */
static void capacity_replay(int priority, int32_t S, int32_t E, int32_t k, int32_t cap,
                            const int32_t* expert_idx, int32_t* slot_idx, float* weight,
                            int32_t* load, int32_t* slot_src) {
  /* 2. capacity replay */
  int32_t* cnt = (int32_t*)calloc((size_t)E, sizeof(int32_t));
  int64_t n_items = (int64_t)S * k;
  for (int64_t it = 0; it < n_items; ++it) {
    int64_t t, j;
    if (priority == ORC_PRIO_TOKEN) { t = it / k; j = it % k; }
    else                            { j = it / S; t = it % S; }
    int64_t i = t * k + j;
    int32_t e = expert_idx[i];
    if (e < 0) { slot_idx[i] = -1; weight[i] = 0.0f; continue; }
    if (cnt[e] < cap) {
      slot_idx[i] = cnt[e];
    } else {
      slot_idx[i] = -1;
      weight[i] = 0.0f;
    }
    cnt[e] += 1;
  }
  for (int32_t e = 0; e < E; ++e) load[e] = cnt[e];
  free(cnt);

  /* 3. inverse map: slot_src[e*cap+s] = t*k+j, -1 for empty slots */
  if (slot_src) {
    for (int64_t i = 0; i < (int64_t)E * cap; ++i) slot_src[i] = -1;
    for (int64_t i = 0; i < n_items; ++i)
      if (slot_idx[i] >= 0)
        slot_src[(int64_t)expert_idx[i] * cap + slot_idx[i]] = (int32_t)i;
  }
}

/* ------------------------------------------------------------------------ */
/* Layout_Transform (R8, R9).                      */
/* ------------------------------------------------------------------------ */
void orc_layout(int32_t S, int32_t E, int32_t k, int32_t cap, int64_t row_bytes,
                const int32_t* expert_idx, const int32_t* slot_idx,
                const void* x, void* dispatch) {
  memset(dispatch, 0, (size_t)((int64_t)E * cap * row_bytes));
  for (int32_t t = 0; t < S; ++t)
    for (int32_t j = 0; j < k; ++j) {
      int64_t i = (int64_t)t * k + j;
      if (slot_idx[i] < 0) continue;
      int64_t dst = ((int64_t)expert_idx[i] * cap + slot_idx[i]) * row_bytes;
      memcpy((char*)dispatch + dst, (const char*)x + (int64_t)t * row_bytes,
             (size_t)row_bytes);
    }
}

/* ------------------------------------------------------------------------ */
/* Reverse_Layout_Transform with the weighted combine (PAPER.md:56-59,      */
/* 64-65; R7).  y_i = 0; for idx in id_i: y_i += w_(i,idx) * e_idx(x_i).     */
/* ------------------------------------------------------------------------ */
void orc_reverse_layout(int dtype, int32_t S, int32_t E, int32_t k, int32_t cap,
                        int32_t d, const int32_t* expert_idx,
                        const int32_t* slot_idx, const float* weight,
                        const void* back, void* y) {
  (void)E;
  for (int32_t t = 0; t < S; ++t)
    for (int32_t c = 0; c < d; ++c) {
      double acc = 0.0;
      for (int32_t j = 0; j < k; ++j) {
        int64_t i = (int64_t)t * k + j;
        if (slot_idx[i] < 0) continue;
        int64_t row = (int64_t)expert_idx[i] * cap + slot_idx[i];
        acc += (double)weight[i] * load_elem(dtype, back, row * d + c);
      }
      store_elem(dtype, y, (int64_t)t * d + c, acc);
    }
}

/* ------------------------------------------------------------------------ */
/* Expert stand-in (R16): s_e = 1 + (e mod 8)/8.                             */
/* ------------------------------------------------------------------------ */
void orc_expert_scale(int dtype, int32_t nsrc, int32_t E_local, int32_t e_base,
                      int32_t cap, int32_t d, const void* in, void* out) {
  for (int32_t src = 0; src < nsrc; ++src)
    for (int32_t le = 0; le < E_local; ++le) {
      int32_t e = e_base + le;
      double s = 1.0 + (double)(e % 8) / 8.0;
      int64_t base = (((int64_t)src * E_local + le) * cap) * d;
      for (int64_t i = 0; i < (int64_t)cap * d; ++i)
        store_elem(dtype, out, base + i, s * load_elem(dtype, in, base + i));
    }
}

/* ------------------------------------------------------------------------ */
/* AllToAll, flat (Fig. 5).                                    */
/* ------------------------------------------------------------------------ */
void orc_alltoall_flat(int32_t P, int64_t bytes_per_peer,
                       const void* const* send, void* const* recv) {
  for (int32_t r = 0; r < P; ++r)
    for (int32_t q = 0; q < P; ++q)
      memcpy((char*)recv[r] + (int64_t)q * bytes_per_peer,
             (const char*)send[q] + (int64_t)r * bytes_per_peer,
             (size_t)bytes_per_peer);
}

void orc_alltoall_flat_stats(int32_t P, int32_t G, int64_t bytes_per_peer,
                             orc_a2a_stats_t* st) {
  memset(st, 0, sizeof *st);
  for (int32_t s = 0; s < P; ++s)
    for (int32_t d = 0; d < P; ++d) {
      if (s / G == d / G) { st->intra_msgs++; st->intra_bytes += bytes_per_peer; }
      else { st->inter_msgs++; st->inter_bytes += bytes_per_peer; }
    }
  st->inter_msg_bytes = (P / G > 1) ? bytes_per_peer : 0;
}

/* ------------------------------------------------------------------------ */
/* AllToAll, hierarchical (Fig. 6), five explicit phases   */
/* (R13).  N = P/G groups of G consecutive ranks; leader = local rank 0.     */
/* ------------------------------------------------------------------------ */
int orc_alltoall_hier(int32_t P, int32_t G, int64_t bytes_per_peer,
                      const void* const* send, void* const* recv,
                      orc_a2a_stats_t* st) {
  if (G < 1 || P % G != 0) return -1;
  const int32_t N = P / G;
  const int64_t B = bytes_per_peer;
  const int64_t leader_bytes = (int64_t)G * P * B;  /* G ranks x P chunks */
  char** g1 = (char**)malloc(sizeof(char*) * (size_t)N);  /* phase 1 */
  char** g2 = (char**)malloc(sizeof(char*) * (size_t)N);  /* phase 2 */
  char** r3 = (char**)malloc(sizeof(char*) * (size_t)N);  /* phase 3 */
  char** r4 = (char**)malloc(sizeof(char*) * (size_t)N);  /* phase 4 */
  for (int32_t g = 0; g < N; ++g) {
    g1[g] = (char*)malloc((size_t)leader_bytes);
    g2[g] = (char*)malloc((size_t)leader_bytes);
    r3[g] = (char*)malloc((size_t)leader_bytes);
    r4[g] = (char*)malloc((size_t)leader_bytes);
  }
  orc_a2a_stats_t s;
  memset(&s, 0, sizeof s);

  /* (1) "gathers the data of all GPUs inside one node into one GPU":
   *     g1_g[m][q] = send_{gG+m}[q]                                         */
  for (int32_t g = 0; g < N; ++g)
    for (int32_t m = 0; m < G; ++m) {
      memcpy(g1[g] + (int64_t)m * P * B, send[g * G + m], (size_t)(P * B));
      s.intra_msgs += 1;
      s.intra_bytes += P * B;
    }
  /* (2) "place the token assigned to the same node in physically continuous
   *     memory": g2_g[h][m][n] = g1_g[m][hG+n]                              */
  for (int32_t g = 0; g < N; ++g)
    for (int32_t h = 0; h < N; ++h)
      for (int32_t m = 0; m < G; ++m)
        for (int32_t n = 0; n < G; ++n)
          memcpy(g2[g] + (((int64_t)h * G + m) * G + n) * B,
                 g1[g] + ((int64_t)m * P + h * G + n) * B, (size_t)B);
  /* (3) "launches All2All communication between nodes": leader h receives
   *     from leader g the block g2_g[h], G*G chunks = B_paper*G/N bytes with
   *     B_paper = P*B the per-GPU data size:
   *     r3_h[g][m][n] = g2_g[h][m][n]                                       */
  for (int32_t h = 0; h < N; ++h)
    for (int32_t g = 0; g < N; ++g) {
      memcpy(r3[h] + (int64_t)g * G * G * B, g2[g] + (int64_t)h * G * G * B,
             (size_t)(G * G * B));
      if (g != h) { s.inter_msgs += 1; s.inter_bytes += G * G * B; }
    }
  s.inter_msg_bytes = (N > 1) ? (int64_t)G * G * B : 0;
  /* (4) "the corresponding data layout transformation":
   *     r4_h[n][g][m] = r3_h[g][m][n]                                       */
  for (int32_t h = 0; h < N; ++h)
    for (int32_t n = 0; n < G; ++n)
      for (int32_t g = 0; g < N; ++g)
        for (int32_t m = 0; m < G; ++m)
          memcpy(r4[h] + (((int64_t)n * N + g) * G + m) * B,
                 r3[h] + (((int64_t)g * G + m) * G + n) * B, (size_t)B);
  /* (5) "scatter operation to put each token to its corresponding expert":
   *     recv_{hG+n} = r4_h[n], i.e. chunks in ascending source rank gG+m    */
  for (int32_t h = 0; h < N; ++h)
    for (int32_t n = 0; n < G; ++n) {
      memcpy(recv[h * G + n], r4[h] + (int64_t)n * P * B, (size_t)(P * B));
      s.intra_msgs += 1;
      s.intra_bytes += P * B;
    }
  for (int32_t g = 0; g < N; ++g) { free(g1[g]); free(g2[g]); free(r3[g]); free(r4[g]); }
  free(g1); free(g2); free(r3); free(r4);
  if (st) *st = s;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Backward of the routing path.       */
/* ------------------------------------------------------------------------ */

/* Adjoint of the combine y_i += w_(i,idx) * e_idx(x_i). */
void orc_reverse_layout_bwd(int dtype, int32_t S, int32_t E, int32_t k, int32_t cap,
                            int32_t d, const int32_t* expert_idx,
                            const int32_t* slot_idx, const float* weight,
                            const void* dy, const void* back, void* d_back,
                            float* d_weight) {
  /* every slot starts at 0: empty slots and padding get no gradient */
  for (int64_t i = 0; i < (int64_t)E * cap * d; ++i) store_elem(dtype, d_back, i, 0.0);
  for (int32_t t = 0; t < S; ++t)
    for (int32_t j = 0; j < k; ++j) {
      int64_t i = (int64_t)t * k + j;
      if (slot_idx[i] < 0) { d_weight[i] = 0.0f; continue; }
      int64_t row = (int64_t)expert_idx[i] * cap + slot_idx[i];
      double dot = 0.0;
      for (int32_t c = 0; c < d; ++c) {
        double g = load_elem(dtype, dy, (int64_t)t * d + c);
        /* dy/d(back[row][c]) = w_(t,j)                                   */
        store_elem(dtype, d_back, row * d + c, (double)weight[i] * g);
        /* dy/d(w_(t,j)) = back[row][c]                                   */
        dot += g * load_elem(dtype, back, row * d + c);
      }
      d_weight[i] = (float)dot;
    }
}

/* Adjoint of Layout_Transform: a gather-sum. */
void orc_layout_bwd(int dtype, int32_t S, int32_t E, int32_t k, int32_t cap, int32_t d,
                    const int32_t* expert_idx, const int32_t* slot_idx,
                    const void* d_dispatch, void* dx) {
  (void)E;
  for (int32_t t = 0; t < S; ++t)
    for (int32_t c = 0; c < d; ++c) {
      double acc = 0.0;
      for (int32_t j = 0; j < k; ++j) {
        int64_t i = (int64_t)t * k + j;
        if (slot_idx[i] < 0) continue;
        int64_t row = (int64_t)expert_idx[i] * cap + slot_idx[i];
        acc += load_elem(dtype, d_dispatch, row * d + c);
      }
      store_elem(dtype, dx, (int64_t)t * d + c, acc);
    }
}

/* Softmax probabilities over the domain dom[0..n) of one row, in double:
 * p[q] = exp(l_dom[q] - m) / sum exp(l - m), m = max over the domain. */
static void softmax_dom(const float* row, const int32_t* dom, int32_t n, double* p) {
  double m = (double)row[dom[0]];
  for (int32_t q = 1; q < n; ++q)
    if ((double)row[dom[q]] > m) m = (double)row[dom[q]];
  double den = 0.0;
  for (int32_t q = 0; q < n; ++q) den += exp((double)row[dom[q]] - m);
  for (int32_t q = 0; q < n; ++q) p[q] = exp((double)row[dom[q]] - m) / den;
}

/* Adjoint of Eq. 1's softmax w.r.t. the logits. */
int orc_gate_bwd(int kind, int weight_mode, int32_t S, int32_t E, int32_t k,
                 const float* logits, const int32_t* expert_idx, const int32_t* slot_idx,
                 const float* d_weight, float* d_logits) {
  if (S < 1 || E < 1 || k < 1 || k > E || !logits) return -1;
  if (kind != ORC_TOPK && kind != ORC_KTOP1) return -1;
  if (kind == ORC_KTOP1 && E % k != 0) return -1;
  int32_t* dom = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
  double* p = (double*)malloc(sizeof(double) * (size_t)E);
  double* grad = (double*)malloc(sizeof(double) * (size_t)E);
  for (int32_t t = 0; t < S; ++t) {
    const float* row = logits + (int64_t)t * E;
    const int32_t* sel = expert_idx + (int64_t)t * k;
    for (int32_t e = 0; e < E; ++e) grad[e] = 0.0;
    for (int32_t j = 0; j < k; ++j) {
      int64_t i = (int64_t)t * k + j;
      double gj = slot_idx[i] >= 0 ? (double)d_weight[i] : 0.0;  /* m_j * g_j */
      int32_t n;
      if (kind == ORC_TOPK && weight_mode == ORC_RENORM) {        /* the k selected */
        n = k;
        for (int32_t q = 0; q < k; ++q) dom[q] = sel[q];
      } else if (kind == ORC_TOPK) {                              /* the whole row */
        n = E;
        for (int32_t q = 0; q < E; ++q) dom[q] = q;
      } else if (weight_mode == ORC_SOFTMAX) {                    /* prototype slice j */
        n = E / k;
        for (int32_t q = 0; q < n; ++q) dom[q] = j * n + q;
      } else {
        continue;                                                 /* w = 1: constant */
      }
      softmax_dom(row, dom, n, p);
      double pj = 0.0;
      for (int32_t q = 0; q < n; ++q)
        if (dom[q] == sel[j]) pj = p[q];
      /* dp_j/dl_e = p_j * (delta(e, e_j) - p_e) for e in the domain */
      for (int32_t q = 0; q < n; ++q) {
        double delta = (dom[q] == sel[j]) ? 1.0 : 0.0;
        grad[dom[q]] += gj * pj * (delta - p[q]);
      }
    }
    for (int32_t e = 0; e < E; ++e) d_logits[(int64_t)t * E + e] = (float)grad[e];
  }
  free(dom);
  free(p);
  free(grad);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Hierarchical top-k, SAM ("the Switch Router first        */
/* selects one group and then the Mixture Router selects multiple experts in */
/* the same group"; R17).                                                    */
/* ------------------------------------------------------------------------ */
int64_t orc_gate_sam(int weight_mode, int priority, int32_t S, int32_t E, int32_t k,
                     int32_t cap, int32_t n_groups, const float* group_logits,
                     const float* logits, int32_t* expert_idx, int32_t* slot_idx,
                     float* weight, int32_t* load, int32_t* slot_src) {
  if (S < 1 || E < 1 || k < 1 || cap < 1 || n_groups < 1 || E % n_groups != 0) return -1;
  const int32_t n = E / n_groups;  /* experts per group, contiguous (R10, R17) */
  if (k > n || !group_logits || !logits) return -1;
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  for (int32_t t = 0; t < S; ++t) {
    const float* gl = group_logits + (int64_t)t * n_groups;
    const float* row = logits + (int64_t)t * E;
    /* Switch Router: the group of largest logit (= largest softmax
     * probability), strict '>' scanning upward: lowest index on ties (R3) */
    int32_t g = 0;
    for (int32_t h = 1; h < n_groups; ++h)
      if (gl[h] > gl[g]) g = h;
    /* Mixture Router: top-k of the expert logits inside group g (R2, R3) */
    int32_t* sel = expert_idx + (int64_t)t * k;
    topk_row(row + (int64_t)g * n, n, k, order, sel);
    for (int32_t j = 0; j < k; ++j) sel[j] += g * n;
    /* weights, in double, rounded once (R17):
     *   RENORM : softmax over the k selected logits (group probability x
     *            within-group softmax, renormalised to sum 1);
     *   SOFTMAX: P(g) * P(e | g), P(g) = softmax over the group logits,
     *            P(e | g) = softmax over the n logits of group g. */
    double m = (double)row[sel[0]], den = 0.0, pg = 1.0;
    if (weight_mode == ORC_RENORM) {
      for (int32_t j = 0; j < k; ++j) den += exp((double)row[sel[j]] - m);
    } else {
      for (int32_t e = g * n; e < (g + 1) * n; ++e) den += exp((double)row[e] - m);
      double gden = 0.0;
      for (int32_t h = 0; h < n_groups; ++h) gden += exp((double)gl[h] - (double)gl[g]);
      pg = 1.0 / gden;
    }
    for (int32_t j = 0; j < k; ++j)
      weight[(int64_t)t * k + j] = (float)(pg * (exp((double)row[sel[j]] - m) / den));
  }
  free(order);
  capacity_replay(priority, S, E, k, cap, expert_idx, slot_idx, weight, load, slot_src);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Dense-to-Sparse ("utilizes the Gumbel Softmax and decreases  */
/* the temperature during training"; R18).                                  */
/* ------------------------------------------------------------------------ */
int64_t orc_gate_d2s(int weight_mode, int priority, int32_t S, int32_t E, int32_t cap,
                     double tau, double eps, const float* logits, const float* uniforms,
                     int32_t* expert_idx, int32_t* slot_idx, float* weight, int32_t* load,
                     int32_t* slot_src) {
  if (S < 1 || E < 1 || cap < 1 || !(tau > 0.0) || !(eps >= 0.0) || !logits) return -1;
  const int32_t k = E;  /* every expert is a candidate slot */
  double* z = (double*)malloc(sizeof(double) * (size_t)E);
  double* p = (double*)malloc(sizeof(double) * (size_t)E);
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
  for (int32_t t = 0; t < S; ++t) {
    const float* row = logits + (int64_t)t * E;
    /* z_e = (l_e + G_e) / tau, G_e = -log(-log(u_e)) a Gumbel(0,1) draw
     * (train), 0 (eval) */
    for (int32_t e = 0; e < E; ++e) {
      double g = 0.0;
      if (uniforms) g = -log(-log((double)uniforms[(int64_t)t * E + e]));
      z[e] = ((double)row[e] + g) / tau;
    }
    /* p = softmax(z) over all E experts (the dense gate) */
    double m = z[0];
    for (int32_t e = 1; e < E; ++e)
      if (z[e] > m) m = z[e];
    double den = 0.0;
    for (int32_t e = 0; e < E; ++e) den += exp(z[e] - m);
    for (int32_t e = 0; e < E; ++e) p[e] = exp(z[e] - m) / den;
    /* survivors p_e >= eps, in descending z (ties: lower index): insertion
     * sort of the survivors */
    int32_t ns = 0;
    double psum = 0.0;
    for (int32_t e = 0; e < E; ++e) {
      if (!(p[e] >= eps)) continue;
      psum += p[e];
      int32_t q = ns++;
      while (q > 0 && (z[e] > z[order[q - 1]] || (z[e] == z[order[q - 1]] && e < order[q - 1]))) {
        order[q] = order[q - 1];
        --q;
      }
      order[q] = e;
    }
    for (int32_t j = 0; j < k; ++j) {
      int64_t i = (int64_t)t * k + j;
      if (j < ns) {
        expert_idx[i] = order[j];
        /* RENORM: survivors renormalised to sum 1; SOFTMAX: p unchanged */
        weight[i] = (float)(weight_mode == ORC_RENORM ? p[order[j]] / psum : p[order[j]]);
      } else {
        expert_idx[i] = -1;  /* pruned */
        weight[i] = 0.0f;
      }
    }
  }
  free(z);
  free(p);
  free(order);
  capacity_replay(priority, S, E, k, cap, expert_idx, slot_idx, weight, load, slot_src);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Dropless packed layout.            */
/* ------------------------------------------------------------------------ */
void orc_expert_offsets(int32_t E, int32_t cap, const int32_t* load, int32_t* offsets) {
  offsets[0] = 0;
  for (int32_t e = 0; e < E; ++e)
    offsets[e + 1] = offsets[e] + (load[e] < cap ? load[e] : cap);
}

void orc_layout_packed(int32_t S, int32_t E, int32_t k, int64_t row_bytes,
                       const int32_t* expert_idx, const int32_t* slot_idx,
                       const int32_t* offsets, const void* x, void* packed) {
  (void)E;
  for (int32_t t = 0; t < S; ++t)
    for (int32_t j = 0; j < k; ++j) {
      int64_t i = (int64_t)t * k + j;
      if (slot_idx[i] < 0) continue;
      int64_t row = (int64_t)offsets[expert_idx[i]] + slot_idx[i];
      memcpy((char*)packed + row * row_bytes, (const char*)x + (int64_t)t * row_bytes,
             (size_t)row_bytes);
    }
}

void orc_reverse_layout_packed(int dtype, int32_t S, int32_t E, int32_t k, int32_t d,
                               const int32_t* expert_idx, const int32_t* slot_idx,
                               const float* weight, const int32_t* offsets,
                               const void* back, void* y) {
  (void)E;
  for (int32_t t = 0; t < S; ++t)
    for (int32_t c = 0; c < d; ++c) {
      double acc = 0.0;
      for (int32_t j = 0; j < k; ++j) {
        int64_t i = (int64_t)t * k + j;
        if (slot_idx[i] < 0) continue;
        int64_t row = (int64_t)offsets[expert_idx[i]] + slot_idx[i];
        acc += (double)weight[i] * load_elem(dtype, back, row * d + c);
      }
      store_elem(dtype, y, (int64_t)t * d + c, acc);
    }
}

void orc_alltoallv(int32_t P, int64_t row_bytes, const int64_t* counts,
                   const void* const* send, void* const* recv) {
  for (int32_t r = 0; r < P; ++r) {
    int64_t at = 0;  /* rows already placed in recv[r] */
    for (int32_t q = 0; q < P; ++q) {
      int64_t from = 0;  /* rows of send[q] before its segment for r */
      for (int32_t rr = 0; rr < r; ++rr) from += counts[(int64_t)q * P + rr];
      int64_t n = counts[(int64_t)q * P + r];
      memcpy((char*)recv[r] + at * row_bytes, (const char*)send[q] + from * row_bytes,
             (size_t)(n * row_bytes));
      at += n;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Adjoints of the SAM and Dense-to-Sparse weights (R17, R18, R19).          */
/* ------------------------------------------------------------------------ */
int orc_gate_bwd_ex(int kind, int weight_mode, int32_t S, int32_t E, int32_t k,
                    const float* logits, const float* group_logits, int32_t n_groups,
                    const float* uniforms, double tau, const int32_t* expert_idx,
                    const int32_t* slot_idx, const float* d_weight, float* d_logits,
                    float* d_group_logits) {
  enum { SAM = 3, D2S = 4 };
  if (kind != SAM && kind != D2S)
    return orc_gate_bwd(kind, weight_mode, S, E, k, logits, expert_idx, slot_idx, d_weight,
                        d_logits);
  if (S < 1 || E < 1 || k < 1 || !logits) return -1;
  if (kind == SAM && (n_groups < 1 || E % n_groups != 0 || !group_logits)) return -1;
  if (kind == D2S && (k != E || !(tau > 0.0))) return -1;
  if (kind == SAM && weight_mode == ORC_RENORM) {
    /* RENORM SAM weights are Eq. 1 on the k selected expert logits */
    int rc = orc_gate_bwd(ORC_TOPK, ORC_RENORM, S, E, k, logits, expert_idx, slot_idx,
                          d_weight, d_logits);
    if (rc == 0 && d_group_logits)
      for (int64_t i = 0; i < (int64_t)S * n_groups; ++i) d_group_logits[i] = 0.0f;
    return rc;
  }
  double* grad = (double*)malloc(sizeof(double) * (size_t)E);
  double* q = (double*)malloc(sizeof(double) * (size_t)E);    /* softmax over the domain */
  double* z = (double*)malloc(sizeof(double) * (size_t)E);
  int32_t* in_dom = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
  double* gg = kind == SAM ? (double*)malloc(sizeof(double) * (size_t)n_groups) : NULL;
  for (int32_t t = 0; t < S; ++t) {
    const float* row = logits + (int64_t)t * E;
    const int32_t* sel = expert_idx + (int64_t)t * k;
    for (int32_t e = 0; e < E; ++e) grad[e] = 0.0;
    double scale = 1.0;
    int32_t g = 0;
    if (kind == SAM) {
      /* domain = the group of the selected experts; z = the raw logits */
      const int32_t n = E / n_groups;
      g = sel[0] / n;
      for (int32_t e = 0; e < E; ++e) { in_dom[e] = (e / n == g); z[e] = (double)row[e]; }
    } else {
      /* z = (l + G)/tau; domain = the survivors (RENORM) or the row (SOFTMAX) */
      for (int32_t e = 0; e < E; ++e) {
        double gn = uniforms ? -log(-log((double)uniforms[(int64_t)t * E + e])) : 0.0;
        z[e] = ((double)row[e] + gn) / tau;
        in_dom[e] = (weight_mode == ORC_SOFTMAX);
      }
      if (weight_mode == ORC_RENORM)
        for (int32_t j = 0; j < k; ++j)
          if (sel[j] >= 0) in_dom[sel[j]] = 1;
      scale = 1.0 / tau;
    }
    double m = -INFINITY, den = 0.0;
    for (int32_t e = 0; e < E; ++e)
      if (in_dom[e] && z[e] > m) m = z[e];
    for (int32_t e = 0; e < E; ++e) den += in_dom[e] ? exp(z[e] - m) : 0.0;
    for (int32_t e = 0; e < E; ++e) q[e] = in_dom[e] ? exp(z[e] - m) / den : 0.0;
    double pg = 1.0;
    if (kind == SAM) {
      const float* gl = group_logits + (int64_t)t * n_groups;
      double gden = 0.0;
      for (int32_t h = 0; h < n_groups; ++h) gden += exp((double)gl[h] - (double)gl[g]);
      pg = 1.0 / gden;
      for (int32_t h = 0; h < n_groups; ++h) gg[h] = 0.0;
    }
    for (int32_t j = 0; j < k; ++j) {
      int64_t i = (int64_t)t * k + j;
      if (sel[j] < 0 || slot_idx[i] < 0) continue;               /* m_j = 0 */
      double gj = (double)d_weight[i];
      double wj = pg * q[sel[j]];                                 /* the weight */
      /* dw_j/dz_e = w_j (delta(e, e_j) - q_e) on the domain; dz/dl = scale */
      for (int32_t e = 0; e < E; ++e)
        if (in_dom[e]) grad[e] += gj * scale * wj * ((e == sel[j] ? 1.0 : 0.0) - q[e]);
      if (kind == SAM) {
        /* dw_j/dgl_h = w_j (delta(h, g) - P(h)) */
        const float* gl = group_logits + (int64_t)t * n_groups;
        for (int32_t h = 0; h < n_groups; ++h) {
          double ph = exp((double)gl[h] - (double)gl[g]) * pg;
          gg[h] += gj * wj * ((h == g ? 1.0 : 0.0) - ph);
        }
      }
    }
    for (int32_t e = 0; e < E; ++e) d_logits[(int64_t)t * E + e] = (float)grad[e];
    if (kind == SAM && d_group_logits)
      for (int32_t h = 0; h < n_groups; ++h)
        d_group_logits[(int64_t)t * n_groups + h] = (float)gg[h];
  }
  free(grad); free(q); free(z); free(in_dom);
  if (gg) free(gg);
  return 0;
}
