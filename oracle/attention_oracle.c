/* TEST INFRASTRUCTURE ONLY — the CPU checker for the sliced causal attention
 * kernels.  Never linked into the product; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg load it (as oracle/_ref/liboracle.so).
 *
 * A plain-C fp64 restatement of the reference numeric kernel
 * (/root/reference/proj/src/attention.cpp), extended to the multi-head / GQA
 * layout the GPU path uses and to the backward pass the reference lacks:
 *
 *   orc_accumulate_chunk   follows accumulate_chunk   attention.cpp:21-61
 *   orc_merge_partials     follows merge_partials     attention.cpp:63-82
 *   orc_finalize           follows finalize           attention.cpp:84-92
 *   orc_chunk_attention    follows chunk_attention    attention.cpp:94-111
 *   orc_fwd_rows / orc_bwd_rows / orc_bwd_keys  sampled rows and keys of one
 *                          head at bench size (same algebra; see below)
 *   orc_attn_bwd_head      NEW (not in the reference): exact softmax-attention
 *                          gradients; pinned against the reference forward by
 *                          finite differences in tests/test_oracle.py, the way
 *                          tests/test_attention.cpp:203-248 pins dO/dQ.
 *
 * Parity of the restatement itself is pinned against the compiled reference
 * (oracle/_ref/libpipelab_ref.so) and the committed fixtures in tests/golden/.
 *
 * Layout conventions (row-major):
 *   single head:  q[rows][d], k/v[total_kv][d]
 *   multi head:   q[rows][a][d], k/v[total_kv][g][d], o like q,
 *                 lse[a][rows] (natural log; -inf for fully masked rows),
 *                 query head h reads kv head h / (a/g).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Streaming state of one head: unnormalised output + running max / sumexp. */
typedef struct {
  int rows, d;
  double *partial, *row_max, *row_sumexp;
} orc_state;

static void state_init(orc_state *st, int rows, int d, double *partial, double *mx,
                       double *sm) {
  st->rows = rows;
  st->d = d;
  st->partial = partial;
  st->row_max = mx;
  st->row_sumexp = sm;
  memset(partial, 0, sizeof(double) * (size_t)rows * d);
  for (int r = 0; r < rows; ++r) {
    mx[r] = -INFINITY;
    sm[r] = 0.0;
  }
}

/* attention.cpp:21-61.  q rows align with the last rows of the kv range of
 * total_kv positions; with causal, row r sees keys at global positions
 * <= total_kv - rows + r, and the scan stops at the first masked key. */
void orc_accumulate_chunk(orc_state *st, const double *q, int qs, const double *k,
                          const double *v, int ks, int len, int64_t chunk_pos,
                          int64_t total_kv, int causal) {
  const int d = st->d;
  const double scale = 1.0 / sqrt((double)d);
  double *scores = (double *)malloc(sizeof(double) * (len > 0 ? len : 1));
  for (int r = 0; r < st->rows; ++r) {
    int64_t limit = causal ? total_kv - st->rows + r : INT64_MAX;
    int usable = 0;
    double cmax = -INFINITY;
    for (int j = 0; j < len; ++j) {
      if (chunk_pos + j > limit) break;
      double s = 0.0;
      for (int c = 0; c < d; ++c) s += q[(size_t)r * qs + c] * k[(size_t)j * ks + c];
      s *= scale;
      scores[j] = s;
      if (s > cmax) cmax = s;
      ++usable;
    }
    if (usable == 0) continue;
    double m_old = st->row_max[r];
    double m_new = m_old > cmax ? m_old : cmax;
    double corr = m_old == -INFINITY ? 0.0 : exp(m_old - m_new);
    st->row_sumexp[r] *= corr;
    double *o = st->partial + (size_t)r * d;
    for (int c = 0; c < d; ++c) o[c] *= corr;
    for (int j = 0; j < usable; ++j) {
      double w = exp(scores[j] - m_new);
      st->row_sumexp[r] += w;
      for (int c = 0; c < d; ++c) o[c] += w * v[(size_t)j * ks + c];
    }
    st->row_max[r] = m_new;
  }
  free(scores);
}

/* attention.cpp:63-82 (both states non-empty). */
void orc_merge_partials(int rows, int d, const double *pa, const double *ma, const double *la,
                        const double *pb, const double *mb, const double *lb, double *po,
                        double *mo, double *lo) {
  for (int r = 0; r < rows; ++r) {
    double m = ma[r] > mb[r] ? ma[r] : mb[r];
    mo[r] = -INFINITY;
    lo[r] = 0.0;
    for (int c = 0; c < d; ++c) po[(size_t)r * d + c] = 0.0;
    if (m == -INFINITY) continue;
    double wa = ma[r] == -INFINITY ? 0.0 : exp(ma[r] - m);
    double wb = mb[r] == -INFINITY ? 0.0 : exp(mb[r] - m);
    mo[r] = m;
    lo[r] = la[r] * wa + lb[r] * wb;
    for (int c = 0; c < d; ++c)
      po[(size_t)r * d + c] = pa[(size_t)r * d + c] * wa + pb[(size_t)r * d + c] * wb;
  }
}

/* attention.cpp:84-92: rows with sumexp <= 0 (fully masked) output 0. */
void orc_finalize(int rows, int d, const double *partial, const double *sm, double *out,
                  int os) {
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < d; ++c)
      out[(size_t)r * os + c] = sm[r] <= 0.0 ? 0.0 : partial[(size_t)r * d + c] / sm[r];
}

/* attention.cpp:94-111 for one head with strided q/k/v/out.  Chunks are
 * consecutive row ranges of k/v given by chunk_sizes.  lse (optional) is
 * row_max + log(row_sumexp), -inf for fully masked rows. */
int orc_chunk_attention(const double *q, int qs, int rows, int d, const double *k,
                        const double *v, int ks, const int *chunk_sizes, int nchunks,
                        int causal, double *out, int os, double *lse, double *row_max,
                        double *row_sumexp) {
  int64_t total_kv = 0;
  for (int c = 0; c < nchunks; ++c) total_kv += chunk_sizes[c];
  double *partial = (double *)malloc(sizeof(double) * (size_t)rows * d + 8);
  double *mx = (double *)malloc(sizeof(double) * rows + 8);
  double *sm = (double *)malloc(sizeof(double) * rows + 8);
  orc_state st;
  state_init(&st, rows, d, partial, mx, sm);
  int64_t pos = 0;
  for (int c = 0; c < nchunks; ++c) {
    orc_accumulate_chunk(&st, q, qs, k + (size_t)pos * ks, v + (size_t)pos * ks, ks,
                         chunk_sizes[c], pos, total_kv, causal);
    pos += chunk_sizes[c];
  }
  orc_finalize(rows, d, partial, sm, out, os);
  for (int r = 0; r < rows; ++r) {
    if (lse) lse[r] = sm[r] <= 0.0 ? -INFINITY : mx[r] + log(sm[r]);
    if (row_max) row_max[r] = mx[r];
    if (row_sumexp) row_sumexp[r] = sm[r];
  }
  free(partial);
  free(mx);
  free(sm);
  return 0;
}

/* NEW: exact gradients of causal (bottom-right aligned) softmax attention for
 * one head, fp64.  Given q, k, v, dO and the forward lse:
 *   P  = exp(scale*q.k - lse)          (0 where masked)
 *   D  = rowsum(dO * O)                (O recomputed from P, v)
 *   dV = P^T dO ; dP = dO v^T ; dS = P*(dP - D)
 *   dQ = scale dS k ; dK = scale dS^T q
 * dq/dk/dv are ACCUMULATED (+=), matching how the GPU path accumulates dK/dV
 * of a chunk across the slices that attend it. */
int orc_attn_bwd_head(const double *q, int qs, int rows, int d, const double *k,
                      const double *v, int ks, int64_t total_kv, int causal,
                      const double *dout, int dos, const double *lse, double *dq, int dqs,
                      double *dk, double *dv, int dks) {
  const double scale = 1.0 / sqrt((double)d);
  double *p = (double *)malloc(sizeof(double) * (total_kv > 0 ? total_kv : 1));
  double *o = (double *)malloc(sizeof(double) * d);
  for (int r = 0; r < rows; ++r) {
    int64_t limit = causal ? total_kv - rows + r : total_kv - 1;
    if (limit >= total_kv) limit = total_kv - 1;
    if (limit < 0 || lse[r] == -INFINITY) continue;
    for (int c = 0; c < d; ++c) o[c] = 0.0;
    for (int64_t j = 0; j <= limit; ++j) {
      double s = 0.0;
      for (int c = 0; c < d; ++c) s += q[(size_t)r * qs + c] * k[(size_t)j * ks + c];
      p[j] = exp(s * scale - lse[r]);
      for (int c = 0; c < d; ++c) o[c] += p[j] * v[(size_t)j * ks + c];
    }
    double D = 0.0;
    for (int c = 0; c < d; ++c) D += dout[(size_t)r * dos + c] * o[c];
    for (int64_t j = 0; j <= limit; ++j) {
      double dp = 0.0;
      for (int c = 0; c < d; ++c) dp += dout[(size_t)r * dos + c] * v[(size_t)j * ks + c];
      double ds = p[j] * (dp - D) * scale;
      for (int c = 0; c < d; ++c) {
        dv[(size_t)j * dks + c] += p[j] * dout[(size_t)r * dos + c];
        dq[(size_t)r * dqs + c] += ds * k[(size_t)j * ks + c];
        dk[(size_t)j * dks + c] += ds * q[(size_t)r * qs + c];
      }
    }
  }
  free(p);
  free(o);
  return 0;
}

/* ---- multi-head drivers (fp32 in, fp64 math), threaded over heads -------- */

typedef struct {
  const float *q, *k, *v, *dout;
  int rows, a, g, d, causal, threads, next;
  int64_t total_kv;
  const int *chunk_sizes;
  int nchunks;
  double *o, *lse, *dq, *dk, *dv;
  const double *lse_in;
  pthread_mutex_t mu;
} mh_job;

static void gather(const float *src, int rows, int stride_heads, int h, int d, double *dst) {
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < d; ++c)
      dst[(size_t)r * d + c] = (double)src[((size_t)r * stride_heads + h) * d + c];
}

static int next_head(mh_job *jb) {
  pthread_mutex_lock(&jb->mu);
  int h = jb->next++;
  pthread_mutex_unlock(&jb->mu);
  return h;
}

static void *fwd_worker(void *arg) {
  mh_job *jb = (mh_job *)arg;
  const int d = jb->d;
  double *qh = (double *)malloc(sizeof(double) * (size_t)jb->rows * d);
  double *kh = (double *)malloc(sizeof(double) * (size_t)jb->total_kv * d + 8);
  double *vh = (double *)malloc(sizeof(double) * (size_t)jb->total_kv * d + 8);
  double *oh = (double *)malloc(sizeof(double) * (size_t)jb->rows * d);
  for (int h; (h = next_head(jb)) < jb->a;) {
    int kvh = h / (jb->a / jb->g);
    gather(jb->q, jb->rows, jb->a, h, d, qh);
    gather(jb->k, (int)jb->total_kv, jb->g, kvh, d, kh);
    gather(jb->v, (int)jb->total_kv, jb->g, kvh, d, vh);
    orc_chunk_attention(qh, d, jb->rows, d, kh, vh, d, jb->chunk_sizes, jb->nchunks,
                        jb->causal, oh, d, jb->lse + (size_t)h * jb->rows, NULL, NULL);
    for (int r = 0; r < jb->rows; ++r)
      for (int c = 0; c < d; ++c) jb->o[((size_t)r * jb->a + h) * d + c] = oh[(size_t)r * d + c];
  }
  free(qh); free(kh); free(vh); free(oh);
  return NULL;
}

static void run_threads(mh_job *jb, void *(*fn)(void *)) {
  int nt = jb->threads < 1 ? 1 : jb->threads;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nt);
  for (int t = 0; t < nt; ++t) pthread_create(&th[t], NULL, fn, jb);
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  free(th);
}

/* Multi-head forward: q[rows][a][d], k/v[total][g][d] (fp32 values, usually
 * bf16-rounded), chunks partition the kv rows.  o[rows][a][d], lse[a][rows]. */
int orc_mha_fwd(const float *q, int rows, int a, int d, const float *k, const float *v, int g,
                const int *chunk_sizes, int nchunks, int causal, double *o, double *lse,
                int threads) {
  mh_job jb;
  memset(&jb, 0, sizeof jb);
  jb.q = q; jb.k = k; jb.v = v; jb.rows = rows; jb.a = a; jb.g = g; jb.d = d;
  jb.causal = causal; jb.threads = threads; jb.chunk_sizes = chunk_sizes; jb.nchunks = nchunks;
  for (int c = 0; c < nchunks; ++c) jb.total_kv += chunk_sizes[c];
  jb.o = o; jb.lse = lse;
  pthread_mutex_init(&jb.mu, NULL);
  run_threads(&jb, fwd_worker);
  pthread_mutex_destroy(&jb.mu);
  return 0;
}

static void *bwd_worker(void *arg) {
  mh_job *jb = (mh_job *)arg;
  const int d = jb->d;
  const int grp = jb->a / jb->g;
  const size_t nkv = (size_t)jb->total_kv * d + 8;
  double *qh = (double *)malloc(sizeof(double) * (size_t)jb->rows * d);
  double *doh = (double *)malloc(sizeof(double) * (size_t)jb->rows * d);
  double *dqh = (double *)malloc(sizeof(double) * (size_t)jb->rows * d);
  double *kh = (double *)malloc(sizeof(double) * nkv);
  double *vh = (double *)malloc(sizeof(double) * nkv);
  double *dkh = (double *)malloc(sizeof(double) * nkv);
  double *dvh = (double *)malloc(sizeof(double) * nkv);
  /* one work item per kv head so dK/dV of a kv head have a single writer */
  for (int kvh; (kvh = next_head(jb)) < jb->g;) {
    gather(jb->k, (int)jb->total_kv, jb->g, kvh, d, kh);
    gather(jb->v, (int)jb->total_kv, jb->g, kvh, d, vh);
    memset(dkh, 0, sizeof(double) * nkv);
    memset(dvh, 0, sizeof(double) * nkv);
    for (int h = kvh * grp; h < (kvh + 1) * grp; ++h) {
      gather(jb->q, jb->rows, jb->a, h, d, qh);
      gather(jb->dout, jb->rows, jb->a, h, d, doh);
      memset(dqh, 0, sizeof(double) * (size_t)jb->rows * d);
      orc_attn_bwd_head(qh, d, jb->rows, d, kh, vh, d, jb->total_kv, jb->causal, doh, d,
                        jb->lse_in + (size_t)h * jb->rows, dqh, d, dkh, dvh, d);
      for (int r = 0; r < jb->rows; ++r)
        for (int c = 0; c < d; ++c)
          jb->dq[((size_t)r * jb->a + h) * d + c] += dqh[(size_t)r * d + c];
    }
    for (int64_t j = 0; j < jb->total_kv; ++j)
      for (int c = 0; c < d; ++c) {
        jb->dk[((size_t)j * jb->g + kvh) * d + c] += dkh[(size_t)j * d + c];
        jb->dv[((size_t)j * jb->g + kvh) * d + c] += dvh[(size_t)j * d + c];
      }
  }
  free(qh); free(doh); free(dqh); free(kh); free(vh); free(dkh); free(dvh);
  return NULL;
}

/* Multi-head backward.  dq[rows][a][d], dk/dv[total][g][d] are accumulated. */
int orc_mha_bwd(const float *q, int rows, int a, int d, const float *k, const float *v, int g,
                int64_t total_kv, int causal, const float *dout, const double *lse, double *dq,
                double *dk, double *dv, int threads) {
  mh_job jb;
  memset(&jb, 0, sizeof jb);
  jb.q = q; jb.k = k; jb.v = v; jb.dout = dout; jb.rows = rows; jb.a = a; jb.g = g; jb.d = d;
  jb.causal = causal; jb.threads = threads; jb.total_kv = total_kv;
  jb.lse_in = lse; jb.dq = dq; jb.dk = dk; jb.dv = dv;
  pthread_mutex_init(&jb.mu, NULL);
  run_threads(&jb, bwd_worker);
  pthread_mutex_destroy(&jb.mu);
  return 0;
}

/* ---- sampled rows / keys of one head at full (bench) size ----------------
 * For the bench-scale parity tests (tests/test_attn_scale_gpu.py): exact fp64
 * values of a few query rows / key rows of a slice whose full oracle would be
 * far too expensive on the CPU.  One head: q[rows][qs], k/v[total_kv][ks]
 * (fp32 values, bf16-rounded by the caller), causal bottom-right aligned as
 * attention.cpp:34-35 (row r sees keys <= total_kv - rows + r).
 *
 *   orc_fwd_rows   O and natural-log LSE of the selected rows: the reference
 *                  fold (accumulate_chunk :49-59 + finalize :84-92) over the
 *                  whole visible prefix in one pass-pair (max, then sums).
 *   orc_bwd_rows   dQ of the selected rows, and
 *   orc_bwd_keys   dK/dV of the selected keys, both for the backward taken as
 *                  the kernel defines it: a function of (Q, K, V, O, dO, LSE)
 *                  with O / LSE given (D_i = rowsum(dO_i * O_i)), the same
 *                  algebra as orc_attn_bwd_head above.
 * Work is split over `threads` pthreads by selected item. */
typedef struct {
  const float *q, *k, *v, *dout, *o;
  const double *lse;
  int qs, ks, dos, os, rows, d, causal, n, threads, next;
  int64_t total_kv;
  const int *sel;
  double *out0, *out1;
  pthread_mutex_t mu;
} smp_job;

static int smp_next(smp_job *jb) {
  pthread_mutex_lock(&jb->mu);
  int x = jb->next++;
  pthread_mutex_unlock(&jb->mu);
  return x;
}

static int64_t smp_limit(const smp_job *jb, int r) {
  int64_t lim = jb->causal ? jb->total_kv - jb->rows + r : jb->total_kv - 1;
  return lim >= jb->total_kv ? jb->total_kv - 1 : lim;
}

static double smp_dot(const float *a, const float *b, int d) {
  double s = 0.0;
  for (int c = 0; c < d; ++c) s += (double)a[c] * (double)b[c];
  return s;
}

static void *fwd_rows_worker(void *arg) {
  smp_job *jb = (smp_job *)arg;
  const int d = jb->d;
  const double scale = 1.0 / sqrt((double)d);
  double *acc = (double *)malloc(sizeof(double) * d);
  for (int x; (x = smp_next(jb)) < jb->n;) {
    const int r = jb->sel[x];
    const int64_t lim = smp_limit(jb, r);
    const float *qr = jb->q + (size_t)r * jb->qs;
    double m = -INFINITY, l = 0.0;
    for (int64_t j = 0; j <= lim; ++j) {
      const double s = smp_dot(qr, jb->k + (size_t)j * jb->ks, d) * scale;
      if (s > m) m = s;
    }
    for (int c = 0; c < d; ++c) acc[c] = 0.0;
    for (int64_t j = 0; j <= lim; ++j) {
      const double e = exp(smp_dot(qr, jb->k + (size_t)j * jb->ks, d) * scale - m);
      l += e;
      const float *vj = jb->v + (size_t)j * jb->ks;
      for (int c = 0; c < d; ++c) acc[c] += e * vj[c];
    }
    for (int c = 0; c < d; ++c) jb->out0[(size_t)x * d + c] = l > 0.0 ? acc[c] / l : 0.0;
    jb->out1[x] = l > 0.0 ? m + log(l) : -INFINITY;
  }
  free(acc);
  return NULL;
}

static double smp_delta(const smp_job *jb, int r) {
  return smp_dot(jb->dout + (size_t)r * jb->dos, jb->o + (size_t)r * jb->os, jb->d);
}

static void *bwd_rows_worker(void *arg) {
  smp_job *jb = (smp_job *)arg;
  const int d = jb->d;
  const double scale = 1.0 / sqrt((double)d);
  for (int x; (x = smp_next(jb)) < jb->n;) {
    const int r = jb->sel[x];
    const int64_t lim = smp_limit(jb, r);
    const float *qr = jb->q + (size_t)r * jb->qs, *dor = jb->dout + (size_t)r * jb->dos;
    const double D = smp_delta(jb, r);
    double *dq = jb->out0 + (size_t)x * d;
    for (int c = 0; c < d; ++c) dq[c] = 0.0;
    if (jb->lse[r] == -INFINITY) continue;
    for (int64_t j = 0; j <= lim; ++j) {
      const float *kj = jb->k + (size_t)j * jb->ks;
      const double p = exp(smp_dot(qr, kj, d) * scale - jb->lse[r]);
      const double ds = p * (smp_dot(dor, jb->v + (size_t)j * jb->ks, d) - D) * scale;
      for (int c = 0; c < d; ++c) dq[c] += ds * kj[c];
    }
  }
  return NULL;
}

static void *bwd_keys_worker(void *arg) {
  smp_job *jb = (smp_job *)arg;
  const int d = jb->d;
  const double scale = 1.0 / sqrt((double)d);
  for (int x; (x = smp_next(jb)) < jb->n;) {
    const int64_t j = jb->sel[x];
    const float *kj = jb->k + (size_t)j * jb->ks, *vj = jb->v + (size_t)j * jb->ks;
    double *dk = jb->out0 + (size_t)x * d, *dv = jb->out1 + (size_t)x * d;
    for (int c = 0; c < d; ++c) dk[c] = dv[c] = 0.0;
    for (int r = 0; r < jb->rows; ++r) {
      if (smp_limit(jb, r) < j || jb->lse[r] == -INFINITY) continue;
      const float *qr = jb->q + (size_t)r * jb->qs, *dor = jb->dout + (size_t)r * jb->dos;
      const double p = exp(smp_dot(qr, kj, d) * scale - jb->lse[r]);
      const double ds = p * (smp_dot(dor, vj, d) - smp_delta(jb, r)) * scale;
      for (int c = 0; c < d; ++c) {
        dv[c] += p * dor[c];
        dk[c] += ds * qr[c];
      }
    }
  }
  return NULL;
}

static void smp_run(smp_job *jb, void *(*fn)(void *)) {
  pthread_mutex_init(&jb->mu, NULL);
  int nt = jb->threads < 1 ? 1 : jb->threads;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nt);
  for (int t = 0; t < nt; ++t) pthread_create(&th[t], NULL, fn, jb);
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&jb->mu);
}

/* o[nsel][d], lse[nsel] */
int orc_fwd_rows(const float *q, int qs, int rows, int d, const float *k, const float *v, int ks,
                 int64_t total_kv, int causal, const int *sel, int nsel, double *o, double *lse,
                 int threads) {
  smp_job jb;
  memset(&jb, 0, sizeof jb);
  jb.q = q; jb.qs = qs; jb.rows = rows; jb.d = d; jb.k = k; jb.v = v; jb.ks = ks;
  jb.total_kv = total_kv; jb.causal = causal; jb.sel = sel; jb.n = nsel; jb.out0 = o; jb.out1 = lse;
  jb.threads = threads;
  smp_run(&jb, fwd_rows_worker);
  return 0;
}

/* dq[nsel][d]; lse[rows] (natural log), o/dout[rows][os/dos] */
int orc_bwd_rows(const float *q, int qs, int rows, int d, const float *k, const float *v, int ks,
                 int64_t total_kv, int causal, const float *o, int os, const float *dout, int dos,
                 const double *lse, const int *sel, int nsel, double *dq, int threads) {
  smp_job jb;
  memset(&jb, 0, sizeof jb);
  jb.q = q; jb.qs = qs; jb.rows = rows; jb.d = d; jb.k = k; jb.v = v; jb.ks = ks; jb.o = o; jb.os = os;
  jb.dout = dout; jb.dos = dos; jb.lse = lse; jb.total_kv = total_kv; jb.causal = causal; jb.sel = sel;
  jb.n = nsel; jb.out0 = dq; jb.threads = threads;
  smp_run(&jb, bwd_rows_worker);
  return 0;
}

/* dk/dv[nsel][d] for key rows sel[] */
int orc_bwd_keys(const float *q, int qs, int rows, int d, const float *k, const float *v, int ks,
                 int64_t total_kv, int causal, const float *o, int os, const float *dout, int dos,
                 const double *lse, const int *sel, int nsel, double *dk, double *dv, int threads) {
  smp_job jb;
  memset(&jb, 0, sizeof jb);
  jb.q = q; jb.qs = qs; jb.rows = rows; jb.d = d; jb.k = k; jb.v = v; jb.ks = ks; jb.o = o; jb.os = os;
  jb.dout = dout; jb.dos = dos; jb.lse = lse; jb.total_kv = total_kv; jb.causal = causal; jb.sel = sel;
  jb.n = nsel; jb.out0 = dk; jb.out1 = dv; jb.threads = threads;
  smp_run(&jb, bwd_keys_worker);
  return 0;
}
