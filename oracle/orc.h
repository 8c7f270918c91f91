/* oracle/orc.h — fp64 CPU oracle of the ASR-KF-EGR generation step (arXiv 2512.11221).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code with the
 * CUDA path (paper_2512_11221_b200/, include/asr.h); the only common module is the seeded
 * input generator gen/, which holds none of the method's arithmetic.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (see SURVEY.md legend); the readings of
 * ambiguous passages are the ones listed in DESIGN.md §"Readings" (R-tick, R-W, ...).
 *
 * Every function is a plain transcription of the paper's definitions in its own order:
 *   Eq. 1  attention over the active set, two-pass max-subtracted softmax
 *   Eq. 2  s_j = (1/H) sum_h |Q_i^(h) . K_j^(h)|, H = L*Hq (R-layer, R-gqa), raw
 *   Eq. 3  d_j = floor(sqrt(c_j)/k) = max m >= 0 with (m*k)^2 <= c_j
 *   Alg. 1 attention -> score -> flag/count/freeze -> tick/restore, literal order
 *   Sec 3.6 entropy-guided recovery SR -> WR -> FR -> RR (detector/ladder: R-det, R-ladder)
 * Parity status: every function here is pinned by tests/test_oracle_*.py.
 */
#ifndef ORC_H
#define ORC_H
#include <stdint.h>

typedef struct {
  int L, Hq, Hkv, d;       /* model shape; Hq % Hkv == 0, head h uses KV head h/(Hq/Hkv) (R-gqa) */
  int window;              /* K: positions >= n-K are protected (R-win) */
  double tau;              /* strict s_j < tau */
  double softness;         /* k of Eq. 3 */
  int history_window;      /* W; 0 = infinite (R-W) */
  int pinned_prefix;       /* positions < pinned are never frozen (R-sink) */
  int score_scaled;        /* 0 = raw Eq. 2 (default), 1 = x 1/sqrt(d) */
  int tick_skip_new;       /* 0 = R0 literal Alg. 1 order (default), 1 = R1 */
  int vocab;               /* logits row length (0 = entropy off) */
  double ent_temp;         /* entropy temperature (R-ent) */
  int det_enable, det_baseline, det_cooldown, wr_window;
  double det_z, det_sigma_floor;
  int fr_clear_counts;     /* FR also clears detection counts (SPEC reading; default 0) */
} orc_cfg;

typedef struct {
  int step;                /* i of this step (0-based) */
  int n;                   /* total tokens after the append */
  int attended;            /* |A_i| */
  int active_post;         /* #Active after the tick (Table 1/3 convention) */
  int frozen_post;
  int frozen_this_step;    /* tokens given d>0 in the freeze loop (incl. d=1 ones the tick restores) */
  int restored_this_step;  /* tick restores + recovery restores + explicit restores since last step */
  int recovery_action;     /* 0 none, 1 SR, 2 WR, 3 FR, 4 RR */
  int rewalk_requested;
  int entropy_valid;
  double entropy;          /* H of logits_prev (nats) */
} orc_out;

typedef struct orc_seq orc_seq;

orc_seq* orc_seq_new(const orc_cfg* cfg, int capacity, int prompt_len);
void orc_seq_free(orc_seq* s);

/* One full generation step (Alg. 1 lines 1-15).  The caller has already written the new
 * token's K/V at position n_before (= current total) of K/V.
 *   q       [L][Hq][d]        dtype 0 = bf16 bits, 1 = f32 (values taken exactly)
 *   K, V    [capacity][L][Hkv][d]
 *   logits_prev [vocab] or NULL (entropy of the previous step's output row)
 *   O       out [L][Hq][d] fp64
 *   act     out [capacity] attended positions (sorted), scores out [capacity] s_j per attended index
 * Returns 0, or -1 on a bad argument (capacity exceeded). */
int orc_step(orc_seq* s, const void* q, int q_dtype, const void* K, const void* V, int kv_dtype,
             const void* logits_prev, int logits_dtype, double* O, int* act, double* scores,
             orc_out* out);

/* Policy-only step (SPEC trace_sim replay): identical to orc_step except that attention is
 * skipped and "s_j < tau" is read from below[pos] (1 = scores below tau).  H_valid=0 skips
 * the entropy/detector stage, else H is the entropy of logits_prev. */
int orc_step_policy(orc_seq* s, const unsigned char* below, double H, int H_valid, int* act,
                    orc_out* out);

/* Explicit recovery (asr_restore analogue) at the boundary before the next step:
 * level 1 SR, 2 WR, 3 FR.  Returns the number of tokens restored. */
int orc_restore(orc_seq* s, int level);

/* Ledger: res 1 = Active, 0 = Frozen; timer d_j; count c_j (lifetime, or within W);
 * freeze_step = step of the last freeze (-1 never).  Arrays of length >= n. */
int orc_n(const orc_seq* s);
void orc_ledger(const orc_seq* s, unsigned char* res, int* timer, uint32_t* count, int* fstep);

/* Building blocks, exposed for the pin tests. */
int orc_duration(uint32_t c, double k);                                       /* Eq. 3 */
double orc_entropy(const void* logits, int dtype, int vocab, double temp);     /* -sum p ln p */

/* Single outputs, for sampled parity checks at full size (where a whole orc_step is too slow):
 * Eq. 1 for one (layer, head): out[d] = softmax(q K^T / sqrt(d)) V over n rows K, V [n][d] (the
 * head's KV rows of the attended tokens, in attended order); q [d]. */
void orc_attend_head(const void* q, int q_dtype, const void* K, const void* V, int kv_dtype, int n, int d,
                     double* out);
/* Eq. 2 for one token: s_j = (1/(L*Hq)) sum over (layer, head) of |q_{l,h} . k_{j,l,h/(Hq/Hkv)}|,
 * q [L][Hq][d], k_j [L][Hkv][d]; x 1/sqrt(d) when scaled (R-scale). */
double orc_score_token(const void* q, int q_dtype, const void* k, int kv_dtype, int L, int Hq, int Hkv, int d,
                       int scaled);

#endif
