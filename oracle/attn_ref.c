/*
 * ORACLE (test infrastructure only) — plain-C restatement of the reference's
 * compiled attention kernel, used as the CPU baseline port.
 *
 * Follows pkg/src/roundkv/_attn_ext.pyx:20-81 operation for operation:
 *   vis[j] = k_pos[j] <= q_pos[i] && allowed[j]                      (:43-48)
 *   row with no visible key -> return i                             (:49-50)
 *   score = sum_d double(q)*double(k) * (1/sqrt(d)), running max    (:51-61)
 *   w = exp(score - max), w_sum                                     (:62-69)
 *   out = sum_j (w/w_sum) * double(v), cap[i,j] += w/w_sum          (:70-80)
 * and the wrapper's row normalisation of the capture (:113-114).
 * Extension over the reference: GQA by head mapping h -> h / (hq/hkv)
 * (equivalent to the reference on repeat_kv-expanded K/V), and a thread
 * count: (row, head) pairs are spread over POSIX threads.  The capture matrix
 * is accumulated per thread and reduced in head order afterwards so results
 * do not depend on the thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const float *q, *k, *v;
  const int64_t *q_pos, *k_pos;
  const uint8_t* allowed;
  int n, hq, hkv, d, s;
  float* out;
  double* cap_h;      /* [hq][n][s] per-head probabilities (capture) or NULL */
  int next;           /* work counter */
  int bad_row;
  pthread_mutex_t lock;
} job_t;

static void one_pair(job_t* J, int i, int h, double* buf, double* acc, unsigned char* vis) {
  const int d = J->d, s = J->s, G = J->hq / J->hkv, kh = h / G;
  const double inv_scale = 1.0 / sqrt((double)d);
  int any = 0;
  for (int j = 0; j < s; ++j) {
    vis[j] = J->k_pos[j] <= J->q_pos[i] && (J->allowed == NULL || J->allowed[j]);
    any |= vis[j];
  }
  if (!any) {
    pthread_mutex_lock(&J->lock);
    if (J->bad_row < 0 || i < J->bad_row) J->bad_row = i;
    pthread_mutex_unlock(&J->lock);
    return;
  }
  const float* qi = J->q + ((int64_t)i * J->hq + h) * d;
  double row_max = -1e308;
  for (int j = 0; j < s; ++j) {
    if (!vis[j]) continue;
    const float* kj = J->k + ((int64_t)j * J->hkv + kh) * d;
    double score = 0.0;
    for (int e = 0; e < d; ++e) score += (double)qi[e] * (double)kj[e];
    score *= inv_scale;
    buf[j] = score;
    if (score > row_max) row_max = score;
  }
  double w_sum = 0.0;
  for (int j = 0; j < s; ++j) {
    if (vis[j]) {
      double w = exp(buf[j] - row_max);
      buf[j] = w;
      w_sum += w;
    } else {
      buf[j] = 0.0;
    }
  }
  for (int e = 0; e < d; ++e) acc[e] = 0.0;
  double* cap = J->cap_h ? J->cap_h + ((int64_t)h * J->n + i) * s : NULL;
  for (int j = 0; j < s; ++j) {
    if (!vis[j]) continue;
    double w = buf[j] / w_sum;
    if (cap) cap[j] = w;
    const float* vj = J->v + ((int64_t)j * J->hkv + kh) * d;
    for (int e = 0; e < d; ++e) acc[e] += w * (double)vj[e];
  }
  float* o = J->out + ((int64_t)i * J->hq + h) * d;
  for (int e = 0; e < d; ++e) o[e] = (float)acc[e];
}

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  double* buf = (double*)malloc(sizeof(double) * (J->s > 0 ? J->s : 1));
  double* acc = (double*)malloc(sizeof(double) * J->d);
  unsigned char* vis = (unsigned char*)malloc(J->s > 0 ? J->s : 1);
  const int total = J->n * J->hq;
  for (;;) {
    pthread_mutex_lock(&J->lock);
    int t = J->next++;
    pthread_mutex_unlock(&J->lock);
    if (t >= total) break;
    one_pair(J, t / J->hq, t % J->hq, buf, acc, vis);
  }
  free(buf);
  free(acc);
  free(vis);
  return NULL;
}

/* returns -1 on success, else the first row with no visible key */
int attn_ref_forward(const float* q, int n, int hq, int d, const float* k, const float* v, int s, int hkv,
                     const int64_t* q_pos, const int64_t* k_pos, const uint8_t* allowed, float* out,
                     double* cap /* [n][s] or NULL */, int threads) {
  job_t J;
  memset(&J, 0, sizeof(J));
  J.q = q; J.k = k; J.v = v; J.q_pos = q_pos; J.k_pos = k_pos; J.allowed = allowed;
  J.n = n; J.hq = hq; J.hkv = hkv; J.d = d; J.s = s; J.out = out;
  J.bad_row = -1;
  pthread_mutex_init(&J.lock, NULL);
  if (cap) J.cap_h = (double*)calloc((size_t)hq * n * (s > 0 ? s : 1), sizeof(double));
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, worker, &J);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&J.lock);
  if (J.bad_row >= 0) {
    free(J.cap_h);
    return J.bad_row;
  }
  if (cap) {
    /* cap[i,j] += w over heads in head order (:75-76), then cap /= rowsum (:113-114) */
    for (int i = 0; i < n; ++i) {
      double* row = cap + (int64_t)i * s;
      for (int j = 0; j < s; ++j) row[j] = 0.0;
      for (int h = 0; h < hq; ++h) {
        const double* src = J.cap_h + ((int64_t)h * n + i) * s;
        for (int j = 0; j < s; ++j) row[j] += src[j];
      }
      double tot = 0.0;
      for (int j = 0; j < s; ++j) tot += row[j];
      for (int j = 0; j < s; ++j) row[j] /= tot;
    }
    free(J.cap_h);
  }
  return -1;
}

/* ------------------------------------------------------------------------
 * Eq. 1 round masses straight from q and K, for full-size parity checks where
 * the [n][s] capture (or the per-head copies above) would not fit in memory.
 * Per row i, exactly the reference's arithmetic for the capture
 * (_attn_ext.pyx:41-76 with capture=True: sequential fp64 dot products,
 * running max, w = exp(score - max), w_sum in key order, cap[j] += w / w_sum in
 * head order), the wrapper's row normalisation (:113-114), then
 * aggregate_round_attention (stats.py:59-94): raw[bin] += capn[j] over the keys
 * of each bin's spans (lo, hi, bin); bins >= n_bins are ignored.  Rows are spread
 * over threads; per-row bin sums are added in row order, so the result does not
 * depend on the thread count.  Four keys are processed at a time: every key's
 * dot product stays a sequential sum over the head dimension.
 * ---------------------------------------------------------------------- */
typedef struct {
  const float *q, *k;
  const int64_t *q_pos, *k_pos;
  const int32_t* spans;
  int n, hq, hkv, d, s, n_spans, n_bins;
  double* row_bins;   /* [n][n_bins] */
  int next;
  pthread_mutex_t lock;
} mjob_t;

static void mass_row(mjob_t* J, int i, double* cap, double* buf) {
  const int d = J->d, s = J->s, G = J->hq / J->hkv;
  const double inv_scale = 1.0 / sqrt((double)d);
  const int64_t qp = J->q_pos[i];
  for (int j = 0; j < s; ++j) cap[j] = 0.0;
  for (int h = 0; h < J->hq; ++h) {
    const float* qi = J->q + ((int64_t)i * J->hq + h) * d;
    const int kh = h / G;
    double row_max = -1e308;
    int j = 0;
    for (; j + 4 <= s; j += 4) {
      const float* k0 = J->k + ((int64_t)(j + 0) * J->hkv + kh) * d;
      const float* k1 = J->k + ((int64_t)(j + 1) * J->hkv + kh) * d;
      const float* k2 = J->k + ((int64_t)(j + 2) * J->hkv + kh) * d;
      const float* k3 = J->k + ((int64_t)(j + 3) * J->hkv + kh) * d;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      for (int e = 0; e < d; ++e) {
        const double qe = (double)qi[e];
        s0 += qe * (double)k0[e];
        s1 += qe * (double)k1[e];
        s2 += qe * (double)k2[e];
        s3 += qe * (double)k3[e];
      }
      buf[j] = s0 * inv_scale;
      buf[j + 1] = s1 * inv_scale;
      buf[j + 2] = s2 * inv_scale;
      buf[j + 3] = s3 * inv_scale;
    }
    for (; j < s; ++j) {
      const float* kj = J->k + ((int64_t)j * J->hkv + kh) * d;
      double sc = 0.0;
      for (int e = 0; e < d; ++e) sc += (double)qi[e] * (double)kj[e];
      buf[j] = sc * inv_scale;
    }
    for (j = 0; j < s; ++j)
      if (J->k_pos[j] <= qp && buf[j] > row_max) row_max = buf[j];
    double w_sum = 0.0;
    for (j = 0; j < s; ++j) {
      if (J->k_pos[j] <= qp) {
        buf[j] = exp(buf[j] - row_max);
        w_sum += buf[j];
      } else {
        buf[j] = 0.0;
      }
    }
    for (j = 0; j < s; ++j)
      if (J->k_pos[j] <= qp) cap[j] += buf[j] / w_sum;
  }
  double tot = 0.0;
  for (int j = 0; j < s; ++j) tot += cap[j];
  double* rb = J->row_bins + (int64_t)i * J->n_bins;
  for (int b = 0; b < J->n_bins; ++b) rb[b] = 0.0;
  for (int a = 0; a < J->n_spans; ++a) {
    const int lo = J->spans[3 * a], hi = J->spans[3 * a + 1], b = J->spans[3 * a + 2];
    if (b < 0 || b >= J->n_bins) continue;
    for (int j = lo; j < hi; ++j) rb[b] += cap[j] / tot;
  }
}

static void* mass_worker(void* arg) {
  mjob_t* J = (mjob_t*)arg;
  double* cap = (double*)malloc(sizeof(double) * (J->s > 0 ? J->s : 1));
  double* buf = (double*)malloc(sizeof(double) * (J->s > 0 ? J->s : 1));
  for (;;) {
    pthread_mutex_lock(&J->lock);
    int i = J->next++;
    pthread_mutex_unlock(&J->lock);
    if (i >= J->n) break;
    mass_row(J, i, cap, buf);
  }
  free(cap);
  free(buf);
  return NULL;
}

void attn_ref_round_masses(const float* q, int n, int hq, int d, const float* k, int s, int hkv,
                           const int64_t* q_pos, const int64_t* k_pos, const int32_t* spans, int n_spans,
                           int n_bins, double* raw /* [n_bins] */, int threads) {
  mjob_t J;
  memset(&J, 0, sizeof(J));
  J.q = q; J.k = k; J.q_pos = q_pos; J.k_pos = k_pos; J.spans = spans;
  J.n = n; J.hq = hq; J.hkv = hkv; J.d = d; J.s = s; J.n_spans = n_spans; J.n_bins = n_bins;
  J.row_bins = (double*)calloc((size_t)(n > 0 ? n : 1) * (n_bins > 0 ? n_bins : 1), sizeof(double));
  pthread_mutex_init(&J.lock, NULL);
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, mass_worker, &J);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&J.lock);
  for (int b = 0; b < n_bins; ++b) raw[b] = 0.0;
  for (int i = 0; i < n; ++i)
    for (int b = 0; b < n_bins; ++b) raw[b] += J.row_bins[(int64_t)i * n_bins + b];
  free(J.row_bins);
}
