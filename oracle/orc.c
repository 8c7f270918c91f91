/* oracle/orc.c — fp64 CPU oracle of the ASR-KF-EGR generation step.  TEST INFRASTRUCTURE.
 *
 * A plain, slow, step-by-step transcription of the paper (arXiv 2512.11221) in its own order;
 * see orc.h for the passage each function follows and DESIGN.md §"Readings" for every reading
 * of an ambiguous passage.  No blocking, no fusion, no reordering: a reader can check each
 * loop against Alg. 1 by eye.  Shares no code with the CUDA path.
 */
#include "orc.h"

#include <float.h>
#include <limits.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { ACTIVE = 1, FROZEN = 0 };
enum { LV_NONE = 0, LV_SR = 1, LV_WR = 2, LV_FR = 3, LV_RR = 4 };

struct orc_seq {
  orc_cfg cfg;
  int cap;        /* maximum positions */
  int n;          /* tokens currently held (total) */
  int step;       /* index i of the next step */
  unsigned char* res;
  int* timer;
  uint32_t* count;   /* lifetime detections (W = infinity) */
  int* fstep;
  int** dlog;        /* finite W: detection steps per position (ring of length W) */
  int* dlog_len;
  double* hist;      /* previous entropies (ring of det_baseline) */
  int hist_len, hist_head;
  int ladder_level;
  int last_action_step;
  int has_last_action;
  int pending_restored;  /* explicit restores since the last step */
};

/* ---------------------------------------------------------------- value access */

static double bf16_to_double(uint16_t b) {
  uint32_t u = ((uint32_t)b) << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

static double val(const void* base, long idx, int dtype) {
  if (dtype == 0) return bf16_to_double(((const uint16_t*)base)[idx]);
  return (double)((const float*)base)[idx];
}

/* ---------------------------------------------------------------- Eq. 3 */

/* d = floor(sqrt(c) / k): the largest m >= 0 with m*k <= sqrt(c), i.e. (m*k)^2 <= c
 * (floor-of-quotient order fixed by the worked values c=9 -> 1 at k=2). */
int orc_duration(uint32_t c, double k) {
  int m = 0;
  while (((double)(m + 1) * k) * ((double)(m + 1) * k) <= (double)c) m++;
  return m;
}

/* ---------------------------------------------------------------- entropy (Sec. 3.6, R-ent) */

/* H = -sum_v p_v ln p_v with p = softmax(x / T), 0 ln 0 = 0. */
double orc_entropy(const void* logits, int dtype, int vocab, double temp) {
  double m = -DBL_MAX;
  for (int v = 0; v < vocab; ++v) {
    double x = val(logits, v, dtype) / temp;
    if (x > m) m = x;
  }
  double Z = 0.0;
  for (int v = 0; v < vocab; ++v) Z += exp(val(logits, v, dtype) / temp - m);
  double H = 0.0;
  for (int v = 0; v < vocab; ++v) {
    double p = exp(val(logits, v, dtype) / temp - m) / Z;
    if (p > 0.0) H -= p * log(p);
  }
  return H;
}

/* ---------------------------------------------------------------- lifecycle */

orc_seq* orc_seq_new(const orc_cfg* cfg, int capacity, int prompt_len) {
  if (capacity <= 0 || prompt_len < 0 || prompt_len > capacity) return NULL;
  orc_seq* s = (orc_seq*)calloc(1, sizeof(orc_seq));
  s->cfg = *cfg;
  s->cap = capacity;
  s->res = (unsigned char*)calloc((size_t)capacity, 1);
  s->timer = (int*)calloc((size_t)capacity, sizeof(int));
  s->count = (uint32_t*)calloc((size_t)capacity, sizeof(uint32_t));
  s->fstep = (int*)malloc(sizeof(int) * (size_t)capacity);
  s->dlog = (int**)calloc((size_t)capacity, sizeof(int*));
  s->dlog_len = (int*)calloc((size_t)capacity, sizeof(int));
  int hb = cfg->det_baseline > 0 ? cfg->det_baseline : 1;
  s->hist = (double*)calloc((size_t)hb, sizeof(double));
  for (int j = 0; j < capacity; ++j) s->fstep[j] = -1;
  /* prefill: every prompt token Active, c = 0, d = 0; no decisions at prefill (R-prefill) */
  for (int j = 0; j < prompt_len; ++j) s->res[j] = ACTIVE;
  s->n = prompt_len;
  s->step = 0;
  return s;
}

void orc_seq_free(orc_seq* s) {
  if (!s) return;
  for (int j = 0; j < s->cap; ++j) free(s->dlog[j]);
  free(s->dlog);
  free(s->dlog_len);
  free(s->res);
  free(s->timer);
  free(s->count);
  free(s->fstep);
  free(s->hist);
  free(s);
}

int orc_n(const orc_seq* s) { return s->n; }

void orc_ledger(const orc_seq* s, unsigned char* res, int* timer, uint32_t* count, int* fstep) {
  for (int j = 0; j < s->n; ++j) {
    if (res) res[j] = s->res[j];
    if (timer) timer[j] = s->timer[j];
    if (fstep) fstep[j] = s->fstep[j];
    if (count) {
      if (s->cfg.history_window <= 0) {
        count[j] = s->count[j];
      } else { /* detections within the window ending at the last completed step */
        int last = s->step - 1, c = 0;
        for (int t = 0; t < s->dlog_len[j]; ++t)
          if (s->dlog[j][t] > last - s->cfg.history_window) c++;
        count[j] = (uint32_t)c;
      }
    }
  }
}

/* ---------------------------------------------------------------- recovery levels */

static int apply_level(orc_seq* s, int level, int i) {
  int restored = 0;
  for (int j = 0; j < s->n; ++j) {
    if (s->res[j] != FROZEN) continue;
    int go = 0;
    if (level == LV_SR) go = s->timer[j] > 1;                          /* "Unfreeze tokens with d > 1" */
    else if (level == LV_WR) go = s->fstep[j] >= i - s->cfg.wr_window; /* "all tokens in the last N steps" */
    else if (level >= LV_FR) go = 1;                                   /* "Clear all freeze durations" */
    if (go) {
      s->res[j] = ACTIVE;
      s->timer[j] = 0;
      restored++;
    }
  }
  if (level >= LV_FR && s->cfg.fr_clear_counts) {
    for (int j = 0; j < s->n; ++j) {
      s->count[j] = 0;
      s->dlog_len[j] = 0;
    }
  }
  return restored;
}

int orc_restore(orc_seq* s, int level) {
  int r = apply_level(s, level, s->step);
  s->pending_restored += r;
  return r;
}

/* Detector (R-det): trigger iff H > mean + z * max(sigma, sigma_floor) over the previous
 * <= det_baseline values (current excluded), with >= 2 observations.  Population sigma. */
static int detect(orc_seq* s, double H) {
  const orc_cfg* c = &s->cfg;
  int trig = 0;
  if (c->det_enable && s->hist_len >= 2) {
    double mu = 0.0;
    for (int t = 0; t < s->hist_len; ++t) mu += s->hist[t];
    mu /= s->hist_len;
    double var = 0.0;
    for (int t = 0; t < s->hist_len; ++t) var += (s->hist[t] - mu) * (s->hist[t] - mu);
    var /= s->hist_len;
    double sigma = sqrt(var);
    double sd = sigma > c->det_sigma_floor ? sigma : c->det_sigma_floor;
    trig = H > mu + c->det_z * sd;
  }
  /* push the current value */
  int hb = c->det_baseline > 0 ? c->det_baseline : 1;
  if (s->hist_len < hb) {
    s->hist[s->hist_len++] = H;
  } else {
    s->hist[s->hist_head] = H;
    s->hist_head = (s->hist_head + 1) % hb;
  }
  return trig;
}

/* Ladder (R-ladder): absorbed if dt < cooldown, escalate one level if cooldown <= dt <
 * 2*cooldown, else restart at SR.  RR = FR + rewalk flag. */
static int ladder(orc_seq* s, int i) {
  int dt = i - s->last_action_step;
  int level;
  if (s->has_last_action && dt < s->cfg.det_cooldown) return LV_NONE;
  if (s->has_last_action && dt < 2 * s->cfg.det_cooldown)
    level = s->ladder_level < LV_RR ? s->ladder_level + 1 : LV_RR;
  else
    level = LV_SR;
  s->ladder_level = level;
  s->last_action_step = i;
  s->has_last_action = 1;
  return level;
}

/* ---------------------------------------------------------------- the step */

static int count_in_window(orc_seq* s, int j, int i) {
  /* record detection at step i, return detections within (i - W, i] */
  int W = s->cfg.history_window;
  if (!s->dlog[j]) s->dlog[j] = (int*)malloc(sizeof(int) * (size_t)(W + 1));
  /* drop entries that left the window */
  int k = 0;
  for (int t = 0; t < s->dlog_len[j]; ++t)
    if (s->dlog[j][t] > i - W) s->dlog[j][k++] = s->dlog[j][t];
  s->dlog[j][k++] = i;
  s->dlog_len[j] = k;
  return k;
}

/* Shared by the full and the policy-only step: Alg. 1 lines 3-15 given s_j < tau flags. */
static void freeze_and_tick(orc_seq* s, int i, const int* act, int A, const unsigned char* below_a,
                            orc_out* out) {
  const orc_cfg* c = &s->cfg;
  const int n = s->n;
  unsigned char* newly = (unsigned char*)calloc((size_t)n, 1);
  int frozen_now = 0;
  /* lines 3-9: for j outside the sliding window with s_j < tau (ascending j) */
  for (int a = 0; a < A; ++a) {
    int j = act[a];
    int eligible = (j < n - c->window) && (j >= c->pinned_prefix);
    if (!eligible || !below_a[a]) continue;
    int cj;
    if (c->history_window <= 0) cj = (int)(++s->count[j]);   /* line 4: c_j <- c_j + 1 */
    else cj = count_in_window(s, j, i);
    int dj = orc_duration((uint32_t)cj, c->softness);        /* line 5: d_j <- floor(sqrt(c_j)/k) */
    if (dj > 0) {                                            /* line 6 */
      s->res[j] = FROZEN;                                    /* line 7: move A -> F */
      s->timer[j] = dj;
      s->fstep[j] = i;
      newly[j] = 1;
      frozen_now++;
    }
  }
  /* lines 10-15: for j in F: d_j <- d_j - 1; if d_j <= 0 restore (R-tick: R0 includes newly frozen) */
  int restored = 0;
  for (int j = 0; j < n; ++j) {
    if (s->res[j] != FROZEN) continue;
    if (c->tick_skip_new && newly[j]) continue;
    s->timer[j] -= 1;
    if (s->timer[j] <= 0) {
      s->timer[j] = 0;
      s->res[j] = ACTIVE;
      restored++;
    }
  }
  free(newly);
  int act_post = 0;
  for (int j = 0; j < n; ++j) act_post += s->res[j] == ACTIVE;
  out->frozen_this_step = frozen_now;
  out->restored_this_step += restored;
  out->active_post = act_post;
  out->frozen_post = n - act_post;
}

/* Steps 1-3 of DESIGN.md §"Oracle step": append, recovery at the boundary, build A_i. */
static int begin_step(orc_seq* s, double H, int H_valid, int* act, orc_out* out) {
  if (s->n >= s->cap) return -1;
  memset(out, 0, sizeof(*out));
  const int i = s->step;
  /* append the token generated by the previous step (Alg. 1 line 16 of step i-1) */
  int j = s->n++;
  s->res[j] = ACTIVE;
  s->timer[j] = 0;
  s->count[j] = 0;
  s->dlog_len[j] = 0;
  s->fstep[j] = -1;
  out->restored_this_step = s->pending_restored;
  s->pending_restored = 0;
  /* recovery on logits_{i-1} */
  if (H_valid) {
    out->entropy_valid = 1;
    out->entropy = H;
    if (detect(s, H)) {
      int level = ladder(s, i);
      if (level != LV_NONE) {
        out->recovery_action = level;
        out->rewalk_requested = level == LV_RR;
        out->restored_this_step += apply_level(s, level, i);
      }
    }
  }
  /* A_i = sorted active positions */
  int A = 0;
  for (int p = 0; p < s->n; ++p)
    if (s->res[p] == ACTIVE) act[A++] = p;
  out->step = i;
  out->n = s->n;
  out->attended = A;
  return A;
}

int orc_step(orc_seq* s, const void* q, int q_dtype, const void* K, const void* V, int kv_dtype,
             const void* logits_prev, int logits_dtype, double* O, int* act, double* scores,
             orc_out* out) {
  const orc_cfg* c = &s->cfg;
  const int L = c->L, Hq = c->Hq, Hkv = c->Hkv, d = c->d;
  const int group = Hq / Hkv;
  double H = 0.0;
  int H_valid = 0;
  if (logits_prev && c->vocab > 0) {
    H = orc_entropy(logits_prev, logits_dtype, c->vocab, c->ent_temp);
    H_valid = 1;
  }
  int A = begin_step(s, H, H_valid, act, out);
  if (A < 0) return -1;
  const int i = s->step;

  /* Alg. 1 line 1 / Eq. 1: O = softmax(q K_A^T / sqrt(d)) V_A for every (layer, head) */
  double* logit = (double*)malloc(sizeof(double) * (size_t)(A > 0 ? A : 1));
  for (int l = 0; l < L; ++l)
    for (int h = 0; h < Hq; ++h) {
      int g = h / group;
      const long qo = ((long)l * Hq + h) * d;
      double mx = -DBL_MAX;
      for (int a = 0; a < A; ++a) {
        const long ko = (((long)act[a] * L + l) * Hkv + g) * d;
        double dot = 0.0;
        for (int e = 0; e < d; ++e) dot += val(q, qo + e, q_dtype) * val(K, ko + e, kv_dtype);
        logit[a] = dot / sqrt((double)d);
        if (logit[a] > mx) mx = logit[a];
      }
      double Z = 0.0;
      for (int a = 0; a < A; ++a) Z += exp(logit[a] - mx);
      for (int e = 0; e < d; ++e) {
        double acc = 0.0;
        for (int a = 0; a < A; ++a) {
          const long vo = (((long)act[a] * L + l) * Hkv + g) * d;
          acc += exp(logit[a] - mx) / Z * val(V, vo + e, kv_dtype);
        }
        O[qo + e] = acc;
      }
    }
  free(logit);

  /* Alg. 1 line 2 / Eq. 2: s_j = (1/H) sum over all L*Hq (layer, head) of |q . k_j| */
  unsigned char* below = (unsigned char*)malloc((size_t)(A > 0 ? A : 1));
  for (int a = 0; a < A; ++a) {
    double sum = 0.0;
    for (int l = 0; l < L; ++l)
      for (int h = 0; h < Hq; ++h) {
        int g = h / group;
        const long qo = ((long)l * Hq + h) * d;
        const long ko = (((long)act[a] * L + l) * Hkv + g) * d;
        double dot = 0.0;
        for (int e = 0; e < d; ++e) dot += val(q, qo + e, q_dtype) * val(K, ko + e, kv_dtype);
        sum += fabs(dot);
      }
    double sj = sum / (double)(L * Hq);
    if (c->score_scaled) sj = sj / sqrt((double)d);
    if (scores) scores[a] = sj;
    below[a] = sj < c->tau; /* strict */
  }
  freeze_and_tick(s, i, act, A, below, out);
  free(below);
  s->step++;
  return 0;
}

int orc_step_policy(orc_seq* s, const unsigned char* below_pos, double H, int H_valid, int* act,
                    orc_out* out) {
  int A = begin_step(s, H, H_valid, act, out);
  if (A < 0) return -1;
  unsigned char* below = (unsigned char*)malloc((size_t)(A > 0 ? A : 1));
  for (int a = 0; a < A; ++a) below[a] = below_pos[act[a]];
  freeze_and_tick(s, s->step, act, A, below, out);
  free(below);
  s->step++;
  return 0;
}

/* ---------------------------------------------------------------- single outputs */

/* Eq. 1 for one (layer, head), in the same order as orc_step: logits q.k_a / sqrt(d),
 * their maximum, Z = sum exp(logit - max), out[e] = sum_a exp(logit_a - max) / Z * v_a[e]. */
void orc_attend_head(const void* q, int q_dtype, const void* K, const void* V, int kv_dtype, int n, int d,
                     double* out) {
  double* logit = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double mx = -DBL_MAX;
  for (int a = 0; a < n; ++a) {
    double dot = 0.0;
    for (int e = 0; e < d; ++e) dot += val(q, e, q_dtype) * val(K, (long)a * d + e, kv_dtype);
    logit[a] = dot / sqrt((double)d);
    if (logit[a] > mx) mx = logit[a];
  }
  double Z = 0.0;
  for (int a = 0; a < n; ++a) Z += exp(logit[a] - mx);
  for (int e = 0; e < d; ++e) {
    double acc = 0.0;
    for (int a = 0; a < n; ++a) acc += exp(logit[a] - mx) / Z * val(V, (long)a * d + e, kv_dtype);
    out[e] = acc;
  }
  free(logit);
}

/* Eq. 2 for one token, H = L*Hq (R-layer, R-gqa), raw unless scaled (R-scale). */
double orc_score_token(const void* q, int q_dtype, const void* k, int kv_dtype, int L, int Hq, int Hkv, int d,
                       int scaled) {
  const int group = Hq / Hkv;
  double sum = 0.0;
  for (int l = 0; l < L; ++l)
    for (int h = 0; h < Hq; ++h) {
      const long qo = ((long)l * Hq + h) * d;
      const long ko = ((long)l * Hkv + h / group) * d;
      double dot = 0.0;
      for (int e = 0; e < d; ++e) dot += val(q, qo + e, q_dtype) * val(k, ko + e, kv_dtype);
      sum += fabs(dot);
    }
  double sj = sum / (double)(L * Hq);
  if (scaled) sj = sj / sqrt((double)d);
  return sj;
}
