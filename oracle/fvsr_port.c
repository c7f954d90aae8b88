/* TEST INFRASTRUCTURE ONLY — see fvsr_port.h for the reference map.
 *
 * Arithmetic order is restated exactly: every fp32 sum is sequential in the
 * reference's order with separate multiply and add (compile with
 * -ffp-contract=off, no -march), so coarse scores, and therefore the selected
 * block ids, are bit-identical to the reference.  exp is expf, as std::exp(float)
 * resolves to it in the reference build.
 */
#include "fvsr_port.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* Seeded RNG — P/include/vsr/rng.hpp:12-53.  std::mt19937_64 is fully        */
/* specified by the C++ standard; the Box-Muller pair uses libm in double.    */
/* ------------------------------------------------------------------------- */

typedef struct { uint64_t mt[312]; int idx; } mt64_t;

static void mt64_seed(mt64_t* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64_t* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

void fp_gaussian(uint64_t seed, float* out, long n) {
  mt64_t* s = (mt64_t*)malloc(sizeof(mt64_t));
  if (!s) return;
  mt64_seed(s, seed);
  int have_spare = 0;
  double spare = 0.0;
  for (long i = 0; i < n; ++i) {
    double g;
    if (have_spare) {
      have_spare = 0;
      g = spare;
    } else {
      double u1 = (double)(mt64_next(s) >> 11) * 0x1.0p-53;
      const double u2 = (double)(mt64_next(s) >> 11) * 0x1.0p-53;
      if (u1 < 1e-300) u1 = 1e-300;
      const double r = sqrt(-2.0 * log(u1));
      const double a = 6.283185307179586476925286766559 * u2;
      spare = r * sin(a);
      have_spare = 1;
      g = r * cos(a);
    }
    out[i] = (float)g * 1.0f;
  }
  free(s);
}

/* ------------------------------------------------------------------------- */
/* Token grid and (2,8,8) partition — P/include/vsr/grid.hpp:22-87,          */
/* P/src/partition.cpp:38-62.                                                */
/* ------------------------------------------------------------------------- */

static int grid_check(const fp_grid* g) {
  if (g->n_frames < 1 || g->rows < 1 || g->cols < 1) return FP_CONFIG; /* grid.hpp:50 */
  for (int i = 0; i < g->n_frames; ++i) {
    if (g->frame_ids[i] < 0) return FP_CONFIG;                                   /* :53 */
    if (i > 0 && g->frame_ids[i] <= g->frame_ids[i - 1]) return FP_CONFIG;       /* :55 */
  }
  return FP_OK;
}

static long grid_tokens(const fp_grid* g) { return (long)g->n_frames * g->rows * g->cols; }

typedef struct {
  long L;
  int nb;
  int* assign;  /* [L] */
  int* keys;    /* [nb][3] */
  long* start;  /* [nb+1] offsets into members */
  long* members;/* [L] grouped by block, ascending token order */
} part_t;

typedef struct { int k0, k1, k2; long tok; } keytok_t;

static int keytok_cmp(const void* a, const void* b) {
  const keytok_t* x = (const keytok_t*)a;
  const keytok_t* y = (const keytok_t*)b;
  if (x->k0 != y->k0) return x->k0 < y->k0 ? -1 : 1;
  if (x->k1 != y->k1) return x->k1 < y->k1 ? -1 : 1;
  if (x->k2 != y->k2) return x->k2 < y->k2 ? -1 : 1;
  return x->tok < y->tok ? -1 : (x->tok > y->tok ? 1 : 0);
}

static void part_free(part_t* p) {
  free(p->assign);
  free(p->keys);
  free(p->start);
  free(p->members);
  memset(p, 0, sizeof(*p));
}

/* std::map<key, tokens> iteration order == lexicographic key order; members are
 * pushed in ascending token order (partition.cpp:41-45). */
static int part_build(const fp_grid* g, part_t* p) {
  memset(p, 0, sizeof(*p));
  int st = grid_check(g);
  if (st) return st;
  const long L = grid_tokens(g);
  const long per = (long)g->rows * g->cols;
  keytok_t* kt = (keytok_t*)malloc(sizeof(keytok_t) * (size_t)L);
  p->assign = (int*)malloc(sizeof(int) * (size_t)L);
  p->members = (long*)malloc(sizeof(long) * (size_t)L);
  p->keys = (int*)malloc(sizeof(int) * 3 * (size_t)L);
  p->start = (long*)malloc(sizeof(long) * (size_t)(L + 1));
  if (!kt || !p->assign || !p->members || !p->keys || !p->start) {
    free(kt);
    part_free(p);
    return FP_NOMEM;
  }
  for (long tok = 0; tok < L; ++tok) {
    const long f = tok / per, r = tok % per;
    const int t = g->frame_ids[f], h = (int)(r / g->cols), w = (int)(r % g->cols);
    kt[tok].k0 = t / 2; /* kBlockT, partition.hpp:11 (frame ids are >= 0) */
    kt[tok].k1 = h / 8; /* kBlockH */
    kt[tok].k2 = w / 8; /* kBlockW */
    kt[tok].tok = tok;
  }
  qsort(kt, (size_t)L, sizeof(keytok_t), keytok_cmp);
  int nb = 0;
  for (long i = 0; i < L; ++i) {
    if (i == 0 || kt[i].k0 != kt[i - 1].k0 || kt[i].k1 != kt[i - 1].k1 ||
        kt[i].k2 != kt[i - 1].k2) {
      p->keys[3 * nb + 0] = kt[i].k0;
      p->keys[3 * nb + 1] = kt[i].k1;
      p->keys[3 * nb + 2] = kt[i].k2;
      p->start[nb] = i;
      ++nb;
    }
    p->members[i] = kt[i].tok;
    p->assign[kt[i].tok] = nb - 1;
  }
  p->start[nb] = L;
  p->L = L;
  p->nb = nb;
  free(kt);
  return FP_OK;
}

/* BlockPartition::find_block, partition.cpp:8-14 (keys are sorted). */
static int part_find(const part_t* p, const int* key) {
  int lo = 0, hi = p->nb;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    const int* k = p->keys + 3 * mid;
    int less = k[0] != key[0] ? k[0] < key[0] : (k[1] != key[1] ? k[1] < key[1] : k[2] < key[2]);
    if (less) lo = mid + 1; else hi = mid;
  }
  if (lo < p->nb && p->keys[3 * lo] == key[0] && p->keys[3 * lo + 1] == key[1] &&
      p->keys[3 * lo + 2] == key[2])
    return lo;
  return -1;
}

int fp_block_count(const fp_grid* g, int* nblocks) {
  part_t p;
  int st = part_build(g, &p);
  if (st) return st;
  *nblocks = p.nb;
  part_free(&p);
  return FP_OK;
}

int fp_partition(const fp_grid* g, int* assignment, int* keys, int* nblocks) {
  part_t p;
  int st = part_build(g, &p);
  if (st) return st;
  memcpy(assignment, p.assign, sizeof(int) * (size_t)p.L);
  memcpy(keys, p.keys, sizeof(int) * 3 * (size_t)p.nb);
  *nblocks = p.nb;
  part_free(&p);
  return FP_OK;
}

/* ------------------------------------------------------------------------- */
/* Token masks — MaskMatrix (mask.hpp:16-59), build_locality_mask            */
/* (mask.cpp:109-147).                                                        */
/* ------------------------------------------------------------------------- */

typedef struct {
  long rows, cols, wpr;
  uint64_t* owned;
  const uint64_t* bits;
} mask_t;

static inline int mask_allowed(const mask_t* m, long i, long j) {
  return (int)((m->bits[i * m->wpr + (j >> 6)] >> (j & 63)) & 1u);
}

static int mask_build(const fp_grid* gq, const fp_grid* gk, const fp_mask* d, mask_t* m) {
  memset(m, 0, sizeof(*m));
  m->rows = grid_tokens(gq);
  m->cols = grid_tokens(gk);
  m->wpr = (m->cols + 63) / 64;
  if (d->kind == 2) {
    if (d->words_per_row != m->wpr) return FP_SHAPE;
    m->bits = d->bits;
    return FP_OK;
  }
  m->owned = (uint64_t*)calloc((size_t)(m->rows * m->wpr), sizeof(uint64_t));
  if (!m->owned) return FP_NOMEM;
  m->bits = m->owned;
  if (d->kind == 0) {
    for (long i = 0; i < m->rows; ++i)
      for (long j = 0; j < m->cols; ++j) m->owned[i * m->wpr + (j >> 6)] |= (uint64_t)1 << (j & 63);
    return FP_OK;
  }
  /* locality: mask.cpp:113-116 validation */
  if (d->extent_h < 1 || d->extent_w < 1) return FP_CONFIG;
  if (d->extent_h > gq->rows || d->extent_w > gq->cols) return FP_CONFIG;
  if (gk->rows != gq->rows || gk->cols != gq->cols) return FP_CONFIG;
  const int rh = d->extent_h / 2, rw = d->extent_w / 2;
  const long perq = (long)gq->rows * gq->cols, perk = (long)gk->rows * gk->cols;
  for (long i = 0; i < m->rows; ++i) {
    const int hi_ = (int)((i % perq) / gq->cols), wi = (int)((i % perq) % gq->cols);
    int h_lo, h_hi, w_lo, w_hi;
    if (d->mode == 1) { /* boundary_truncated, mask.cpp:130-134 */
      h_lo = hi_ - rh; h_hi = hi_ + rh + 1;
      w_lo = wi - rw;  w_hi = wi + rw + 1;
    } else {            /* boundary_preserved, mask.cpp:135-140 */
      int a = hi_ - rh, amax = gq->rows - d->extent_h;
      h_lo = a < 0 ? 0 : (a > amax ? amax : a);
      h_hi = h_lo + d->extent_h;
      int b = wi - rw, bmax = gq->cols - d->extent_w;
      w_lo = b < 0 ? 0 : (b > bmax ? bmax : b);
      w_hi = w_lo + d->extent_w;
    }
    for (long j = 0; j < m->cols; ++j) {
      const int hj = (int)((j % perk) / gk->cols), wj = (int)((j % perk) % gk->cols);
      if (hj >= h_lo && hj < h_hi && wj >= w_lo && wj < w_hi)
        m->owned[i * m->wpr + (j >> 6)] |= (uint64_t)1 << (j & 63);
    }
  }
  return FP_OK;
}

static void mask_free(mask_t* m) { free(m->owned); memset(m, 0, sizeof(*m)); }

/* ------------------------------------------------------------------------- */
/* plan_sparse — P/src/sparse.cpp:72-133                                     */
/* ------------------------------------------------------------------------- */

/* avg_pool_blocks, tensor.cpp:161-186: tokens in ascending order accumulate into
 * their block row (dst[j] += src[j]); then dst[j] *= (1.0f / count). */
static int avg_pool(const float* x, long L, int c, const part_t* p, float* out) {
  int* counts = (int*)calloc((size_t)p->nb, sizeof(int));
  if (!counts) return FP_NOMEM;
  memset(out, 0, sizeof(float) * (size_t)p->nb * (size_t)c);
  for (long i = 0; i < L; ++i) {
    const int b = p->assign[i];
    counts[b]++;
    const float* src = x + i * c;
    float* dst = out + (long)b * c;
    for (int j = 0; j < c; ++j) dst[j] += src[j];
  }
  for (int b = 0; b < p->nb; ++b) {
    if (counts[b] == 0) { free(counts); return FP_EMPTY_BLOCK; }
    const float inv = 1.0f / (float)counts[b];
    float* dst = out + (long)b * c;
    for (int j = 0; j < c; ++j) dst[j] *= inv;
  }
  free(counts);
  return FP_OK;
}

typedef struct { float s; int id; } cand_t;

/* stable_sort comparator of sparse.cpp:111-116: score desc, then id asc.  ids are
 * distinct, so the order is total and qsort reproduces stable_sort. */
static int cand_cmp(const void* a, const void* b) {
  const cand_t* x = (const cand_t*)a;
  const cand_t* y = (const cand_t*)b;
  if (x->s != y->s) return x->s > y->s ? -1 : 1;
  return x->id < y->id ? -1 : (x->id > y->id ? 1 : 0);
}

static int int_cmp(const void* a, const void* b) {
  const int x = *(const int*)a, y = *(const int*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

int fp_plan(const float* q, const float* k, int d, const fp_grid* gq, const fp_grid* gk,
            const fp_mask* md, long topk, int cap, int* sel, int* sel_count, int* diag,
            float* coarse_out, uint8_t* allowed_out) {
  if (d < 1) return FP_SHAPE;
  part_t pq, pk;
  mask_t m;
  int st = part_build(gq, &pq);
  if (st) return st;
  st = part_build(gk, &pk);
  if (st) { part_free(&pq); return st; }
  st = mask_build(gq, gk, md, &m);
  if (st) { part_free(&pq); part_free(&pk); return st; }
  if (topk < 1) { st = FP_CONFIG; goto done0; } /* sparse.cpp:83 */

  const int bnq = pq.nb, bnk = pk.nb;
  float* pooled_q = (float*)malloc(sizeof(float) * (size_t)bnq * d);
  float* pooled_k = (float*)malloc(sizeof(float) * (size_t)bnk * d);
  float* coarse = (float*)malloc(sizeof(float) * (size_t)bnq * bnk);
  uint8_t* allowed = (uint8_t*)calloc((size_t)bnq * bnk, 1);
  cand_t* order = (cand_t*)malloc(sizeof(cand_t) * (size_t)bnk);
  uint64_t* colset = (uint64_t*)calloc((size_t)m.wpr, sizeof(uint64_t));
  if (!pooled_q || !pooled_k || !coarse || !allowed || !order || !colset) { st = FP_NOMEM; goto done; }

  st = avg_pool(q, pq.L, d, &pq, pooled_q);
  if (st) goto done;
  st = avg_pool(k, pk.L, d, &pk, pooled_k);
  if (st) goto done;
  /* matmul's finite checks, tensor.cpp:126-127 */
  for (long i = 0; i < (long)bnq * d; ++i) if (!isfinite(pooled_q[i])) { st = FP_SHAPE; goto done; }
  for (long i = 0; i < (long)bnk * d; ++i) if (!isfinite(pooled_k[i])) { st = FP_SHAPE; goto done; }

  /* coarse = matmul(pooled_q, transpose2d(pooled_k)) * scale (sparse.cpp:95-99).
   * matmul's tiled i-k-j loop accumulates each out[i][j] over k in ascending
   * order starting from 0.0f (tensor.cpp:132-147). */
  const float scale = 1.0f / sqrtf((float)d);
  for (int qb = 0; qb < bnq; ++qb)
    for (int kb = 0; kb < bnk; ++kb) {
      float acc = 0.0f;
      for (int c = 0; c < d; ++c) {
        const float prod = pooled_q[(long)qb * d + c] * pooled_k[(long)kb * d + c];
        acc = acc + prod;
      }
      coarse[(long)qb * bnk + kb] = acc * scale;
    }

  /* coarse_allowed_mask, sparse.cpp:47-70: any allowed token pair in the block pair */
  for (int kb = 0; kb < bnk; ++kb) {
    memset(colset, 0, sizeof(uint64_t) * (size_t)m.wpr);
    for (long t = pk.start[kb]; t < pk.start[kb + 1]; ++t) {
      const long j = pk.members[t];
      colset[j >> 6] |= (uint64_t)1 << (j & 63);
    }
    for (int qb = 0; qb < bnq; ++qb) {
      for (long t = pq.start[qb]; t < pq.start[qb + 1]; ++t) {
        const uint64_t* row = m.bits + pq.members[t] * m.wpr;
        int hit = 0;
        for (long a = 0; a < m.wpr; ++a)
          if (row[a] & colset[a]) { hit = 1; break; }
        if (hit) { allowed[(long)qb * bnk + kb] = 1; break; }
      }
    }
  }

  /* selection, sparse.cpp:103-130 */
  for (int qb = 0; qb < bnq; ++qb) {
    int n = 0;
    for (int kb = 0; kb < bnk; ++kb)
      if (allowed[(long)qb * bnk + kb]) { order[n].s = coarse[(long)qb * bnk + kb]; order[n].id = kb; ++n; }
    qsort(order, (size_t)n, sizeof(cand_t), cand_cmp);
    int dg = part_find(&pk, pq.keys + 3 * qb);
    if (dg >= 0 && !allowed[(long)qb * bnk + dg]) dg = -1;
    diag[qb] = dg;
    int* s = sel + (long)qb * cap;
    int cnt = 0;
    if (dg >= 0) { if (cnt >= cap) { st = FP_SHAPE; goto done; } s[cnt++] = dg; }
    for (int i = 0; i < n; ++i) {
      if (cnt >= topk) break;
      if (order[i].id != dg) { if (cnt >= cap) { st = FP_SHAPE; goto done; } s[cnt++] = order[i].id; }
    }
    qsort(s, (size_t)cnt, sizeof(int), int_cmp);
    for (int i = cnt; i < cap; ++i) s[i] = -1;
    sel_count[qb] = cnt;
  }
  if (coarse_out) memcpy(coarse_out, coarse, sizeof(float) * (size_t)bnq * bnk);
  if (allowed_out) memcpy(allowed_out, allowed, (size_t)bnq * bnk);

done:
  free(pooled_q); free(pooled_k); free(coarse); free(allowed); free(order); free(colset);
done0:
  part_free(&pq); part_free(&pk); mask_free(&m);
  return st;
}

/* ------------------------------------------------------------------------- */
/* sparse_attention_exec — exec_block_range, P/src/sparse.cpp:141-206        */
/* ------------------------------------------------------------------------- */

int fp_exec(const float* q, const float* k, const float* v, int d, const fp_grid* gq,
            const fp_grid* gk, const fp_mask* md, int cap, const int* sel,
            const int* sel_count, float scale, long row_begin, long row_end, float* out) {
  part_t pq, pk;
  mask_t m;
  int st = part_build(gq, &pq);
  if (st) return st;
  st = part_build(gk, &pk);
  if (st) { part_free(&pq); return st; }
  st = mask_build(gq, gk, md, &m);
  if (st) { part_free(&pq); part_free(&pk); return st; }
  const long Lq = pq.L;
  if (row_end < 0 || row_end > Lq) row_end = Lq;           /* sparse.cpp:224 */
  if (row_begin < 0 || row_begin > row_end) { st = FP_CONFIG; goto done0; } /* :225 */

  float* block_scores = (float*)malloc(sizeof(float) * 128);
  float* acc = (float*)malloc(sizeof(float) * (size_t)d);
  if (!block_scores || !acc) { st = FP_NOMEM; goto done; }
  memset(out, 0, sizeof(float) * (size_t)Lq * d);
  for (int qb = 0; qb < pq.nb; ++qb) {
    const int* s = sel + (long)qb * cap;
    for (long t = pq.start[qb]; t < pq.start[qb + 1]; ++t) {
      const long i = pq.members[t];
      if (i < row_begin || i >= row_end) continue;
      const float* qi = q + i * d;
      float run_max = -INFINITY, run_sum = 0.0f;
      for (int c = 0; c < d; ++c) acc[c] = 0.0f;
      for (int si = 0; si < sel_count[qb]; ++si) {
        const int kb = s[si];
        if (kb < 0 || kb >= pk.nb) { st = FP_INVARIANT; goto done; }
        /* pass 1: scores and local max over mask-allowed members */
        float local_max = -INFINITY;
        int nb = 0;
        for (long u = pk.start[kb]; u < pk.start[kb + 1]; ++u) {
          const long j = pk.members[u];
          if (!mask_allowed(&m, i, j)) { block_scores[nb++] = -INFINITY; continue; }
          const float* kj = k + j * d;
          float dot = 0.0f;
          for (int c = 0; c < d; ++c) dot += qi[c] * kj[c];
          dot *= scale;
          block_scores[nb++] = dot;
          if (dot > local_max) local_max = dot;
        }
        if (local_max == -INFINITY) continue;
        /* pass 2: merge under the combined running max */
        const float new_max = run_max > local_max ? run_max : local_max;
        if (run_sum > 0.0f && new_max > run_max) {
          const float rescale = expf(run_max - new_max);
          run_sum *= rescale;
          for (int c = 0; c < d; ++c) acc[c] *= rescale;
        }
        nb = 0;
        for (long u = pk.start[kb]; u < pk.start[kb + 1]; ++u) {
          const long j = pk.members[u];
          const float sc = block_scores[nb++];
          if (sc == -INFINITY) continue;
          const float w = expf(sc - new_max);
          run_sum += w;
          const float* vj = v + j * d;
          for (int c = 0; c < d; ++c) acc[c] += w * vj[c];
        }
        run_max = new_max;
      }
      if (!(run_sum > 0.0f)) { st = FP_DEGENERATE; goto done; } /* sparse.cpp:198-200 */
      float* oi = out + i * d;
      const float inv = 1.0f / run_sum;
      for (int c = 0; c < d; ++c) oi[c] = acc[c] * inv;
    }
  }
done:
  free(block_scores); free(acc);
done0:
  part_free(&pq); part_free(&pk); mask_free(&m);
  return st;
}

/* ------------------------------------------------------------------------- */
/* sparsity_report — P/src/sparse.cpp:256-285                                */
/* ------------------------------------------------------------------------- */

int fp_report(const fp_grid* gq, const fp_grid* gk, const fp_mask* md, int cap,
              const int* sel, const int* sel_count, uint64_t* executed_pairs,
              uint64_t* dense_pairs, uint64_t* selected_blocks, uint64_t* allowed_blocks) {
  part_t pq, pk;
  mask_t m;
  int st = part_build(gq, &pq);
  if (st) return st;
  st = part_build(gk, &pk);
  if (st) { part_free(&pq); return st; }
  st = mask_build(gq, gk, md, &m);
  if (st) { part_free(&pq); part_free(&pk); return st; }
  uint64_t ex = 0, dense = 0, nsel = 0, nallow = 0;
  for (int qb = 0; qb < pq.nb; ++qb) {
    nsel += (uint64_t)sel_count[qb];
    for (long t = pq.start[qb]; t < pq.start[qb + 1]; ++t) {
      const long i = pq.members[t];
      for (int si = 0; si < sel_count[qb]; ++si) {
        const int kb = sel[(long)qb * cap + si];
        for (long u = pk.start[kb]; u < pk.start[kb + 1]; ++u)
          ex += (uint64_t)mask_allowed(&m, i, pk.members[u]);
      }
    }
    /* coarse-allowed block pairs of this q-block */
    for (int kb = 0; kb < pk.nb; ++kb) {
      int hit = 0;
      for (long t = pq.start[qb]; t < pq.start[qb + 1] && !hit; ++t)
        for (long u = pk.start[kb]; u < pk.start[kb + 1]; ++u)
          if (mask_allowed(&m, pq.members[t], pk.members[u])) { hit = 1; break; }
      nallow += (uint64_t)hit;
    }
  }
  for (long i = 0; i < m.rows; ++i)
    for (long a = 0; a < m.wpr; ++a) dense += (uint64_t)__builtin_popcountll(m.bits[i * m.wpr + a]);
  *executed_pairs = ex;
  *dense_pairs = dense;
  *selected_blocks = nsel;
  *allowed_blocks = nallow;
  part_free(&pq); part_free(&pk); mask_free(&m);
  return st;
}
