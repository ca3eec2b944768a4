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
