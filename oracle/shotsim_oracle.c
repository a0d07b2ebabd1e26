/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's multi-shot
 * statevector path (see shotsim_oracle.h for who may load it and how it is
 * pinned). Every function names the reference file:line it restates.
 * Build: oracle/Makefile (gcc -std=c11 -O2 -ffp-contract=off).
 */
#define _GNU_SOURCE
#include "shotsim_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double re, im;
} cx;

static __thread char g_err[256];
const char* oracle_last_error(void) { return g_err; }

#define FAIL(code, ...)                                \
  do {                                                 \
    snprintf(g_err, sizeof g_err, __VA_ARGS__);        \
    return (code);                                     \
  } while (0)

/* ---- rng.cpp:9-46 ------------------------------------------------------ */
void oracle_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    c1 = (uint32_t)p1;
    c3 = (uint32_t)p0;
    c0 = n0;
    c2 = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

double oracle_uniform(uint64_t seed, uint64_t shot, uint64_t event) {
  const uint32_t ctr[4] = {(uint32_t)shot, (uint32_t)(shot >> 32), (uint32_t)event,
                           (uint32_t)(event >> 32)};
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t o[4];
  oracle_philox(ctr, key, o);
  const uint64_t bits = ((uint64_t)o[0] << 32) | o[1];
  return (double)(bits >> 11) * 0x1.0p-53;
}

/* ---- complex arithmetic as libstdc++ std::complex<double> (no FMA) ----- */
static inline cx cmul(cx a, cx b) {
  cx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}
static inline cx cadd(cx a, cx b) {
  cx r = {a.re + b.re, a.im + b.im};
  return r;
}
static inline cx cscale(cx a, double d) {
  cx r = {a.re * d, a.im * d};
  return r;
}
static inline double norm2(cx a) { return a.re * a.re + a.im * a.im; }

/* ---- common.hpp:36-67, common.cpp:12-26 -------------------------------- */
static uint64_t scatter_bits(uint64_t value, const uint32_t* pos, unsigned k) {
  uint64_t out = 0;
  for (unsigned b = 0; b < k; ++b)
    if ((value >> b) & 1) out |= (uint64_t)1 << pos[b];
  return out;
}
static uint64_t expand_index(uint64_t g, const uint32_t* sorted, unsigned k) {
  for (unsigned i = 0; i < k; ++i) {
    const unsigned p = sorted[i];
    const uint64_t low = g & (((uint64_t)1 << p) - 1);
    g = ((g >> p) << (p + 1)) | low;
  }
  return g;
}
static double pairwise_sum(const double* v, uint64_t count) {
  if (count <= 8) {
    double s = 0.0;
    for (uint64_t i = 0; i < count; ++i) s += v[i];
    return s;
  }
  const uint64_t half = count / 2;
  return pairwise_sum(v, half) + pairwise_sum(v + half, count - half);
}
static void sort_small(uint32_t* q, unsigned k) {
  for (unsigned i = 1; i < k; ++i)
    for (unsigned j = i; j > 0 && q[j - 1] > q[j]; --j) {
      uint32_t t = q[j];
      q[j] = q[j - 1];
      q[j - 1] = t;
    }
}

#define SUM_BLOCK 512u

/* ---- kernels_scalar.cpp:24-126 ------------------------------------------ */
static void apply_matrix1(cx* a, uint64_t dim, unsigned t, const cx* m) {
  const uint64_t mask = (uint64_t)1 << t, lo = mask - 1;
  for (uint64_t i = 0; i < dim / 2; ++i) {
    const uint64_t i0 = ((i & ~lo) << 1) | (i & lo), i1 = i0 | mask;
    const cx v0 = a[i0], v1 = a[i1];
    a[i0] = cadd(cmul(m[0], v0), cmul(m[1], v1));
    a[i1] = cadd(cmul(m[2], v0), cmul(m[3], v1));
  }
}

static void apply_matrix2(cx* a, uint64_t dim, unsigned q0, unsigned q1, const cx* m) {
  const uint64_t d0 = (uint64_t)1 << q0, d1 = (uint64_t)1 << q1;
  const unsigned pl = q0 < q1 ? q0 : q1, ph = q0 < q1 ? q1 : q0;
  const uint64_t ml = ((uint64_t)1 << pl) - 1, mh = ((uint64_t)1 << ph) - 1;
  for (uint64_t i = 0; i < dim / 4; ++i) {
    uint64_t b = ((i & ~ml) << 1) | (i & ml);
    b = ((b & ~mh) << 1) | (b & mh);
    const cx v[4] = {a[b], a[b + d0], a[b + d1], a[b + d0 + d1]};
    const uint64_t idx[4] = {b, b + d0, b + d1, b + d0 + d1};
    for (int r = 0; r < 4; ++r) {
      cx s = cadd(cmul(m[4 * r], v[0]), cmul(m[4 * r + 1], v[1]));
      s = cadd(s, cmul(m[4 * r + 2], v[2]));
      s = cadd(s, cmul(m[4 * r + 3], v[3]));
      a[idx[r]] = s;
    }
  }
}

static int popcount64(uint64_t v) { return __builtin_popcountll(v); }

static void apply_pauli(cx* a, uint64_t dim, uint64_t x, uint64_t z, unsigned num_y,
                        unsigned x_max) {
  static const cx phases[4] = {{1.0, 0.0}, {0.0, -1.0}, {-1.0, 0.0}, {0.0, 1.0}};
  const cx ph = phases[num_y & 3u];
  if (x == 0) {
    for (uint64_t j = 0; j < dim; ++j) {
      cx v = cmul(ph, a[j]);
      if (popcount64(j & z) & 1) {
        v.re = -v.re;
        v.im = -v.im;
      }
      a[j] = v;
    }
    return;
  }
  const uint64_t mask_l = ((uint64_t)1 << x_max) - 1;
  const uint64_t mask_u = ~((((uint64_t)1 << x_max) << 1) - 1);
  for (uint64_t i = 0; i < dim / 2; ++i) {
    const uint64_t i0 = ((i << 1) & mask_u) | (i & mask_l), i1 = i0 ^ x;
    cx t0 = cmul(ph, a[i1]), t1 = cmul(ph, a[i0]);
    if (popcount64(i0 & z) & 1) {
      t0.re = -t0.re;
      t0.im = -t0.im;
    }
    if (popcount64(i1 & z) & 1) {
      t1.re = -t1.re;
      t1.im = -t1.im;
    }
    a[i0] = t0;
    a[i1] = t1;
  }
}

static double expval1(const cx* a, uint64_t dim, unsigned t, const cx* m) {
  const uint64_t mask = (uint64_t)1 << t, lo = mask - 1, pairs = dim / 2;
  const uint64_t nblk = pairs <= SUM_BLOCK ? 1 : (pairs + SUM_BLOCK - 1) / SUM_BLOCK;
  double* part = malloc(nblk * sizeof(double));
  for (uint64_t b = 0; b < nblk; ++b) {
    const uint64_t beg = pairs <= SUM_BLOCK ? 0 : b * SUM_BLOCK;
    const uint64_t end = pairs <= SUM_BLOCK ? pairs : (beg + SUM_BLOCK < pairs ? beg + SUM_BLOCK : pairs);
    double s = 0.0;
    for (uint64_t i = beg; i < end; ++i) {
      const uint64_t i0 = ((i & ~lo) << 1) | (i & lo), i1 = i0 | mask;
      const cx r0 = cadd(cmul(m[0], a[i0]), cmul(m[1], a[i1]));
      const cx r1 = cadd(cmul(m[2], a[i0]), cmul(m[3], a[i1]));
      s += norm2(r0);
      s += norm2(r1);
    }
    part[b] = s;
  }
  const double r = pairs <= SUM_BLOCK ? part[0] : pairwise_sum(part, nblk);
  free(part);
  return r;
}

/* statevector.cpp:56-80 (k = 2 here; any k supported) */
static double expval_generic(const cx* a, unsigned n, const uint32_t* qubits, unsigned k,
                             const cx* m) {
  uint32_t sorted[SSB_MAX_OP_QUBITS];
  memcpy(sorted, qubits, k * sizeof(uint32_t));
  sort_small(sorted, k);
  const uint64_t side = (uint64_t)1 << k, groups = (uint64_t)1 << (n - k);
  uint64_t off[16];
  for (uint64_t l = 0; l < side; ++l) off[l] = scatter_bits(l, qubits, k);
  double* part = malloc(groups * sizeof(double));
  for (uint64_t g = 0; g < groups; ++g) {
    const uint64_t base = expand_index(g, sorted, k);
    cx in[16];
    for (uint64_t l = 0; l < side; ++l) in[l] = a[base + off[l]];
    double s = 0.0;
    for (uint64_t r = 0; r < side; ++r) {
      cx acc = {0.0, 0.0};
      for (uint64_t c = 0; c < side; ++c) acc = cadd(acc, cmul(m[r * side + c], in[c]));
      s += norm2(acc);
    }
    part[g] = s;
  }
  const double r = pairwise_sum(part, groups);
  free(part);
  return r;
}

/* ---- statevector.cpp:96-197 -------------------------------------------- */
static void load_matrix(const ssb_flat_program* p, uint32_t idx, unsigned k, cx* m) {
  const double* src = p->matrices + (size_t)idx * SSB_MATRIX_STRIDE;
  for (unsigned i = 0; i < (1u << (2 * k)); ++i) {
    m[i].re = src[2 * i];
    m[i].im = src[2 * i + 1];
  }
}

static void apply_matrix(cx* a, unsigned n, const uint32_t* q, unsigned k, const cx* m) {
  if (k == 1) apply_matrix1(a, (uint64_t)1 << n, q[0], m);
  else apply_matrix2(a, (uint64_t)1 << n, q[0], q[1], m);
}

static double expval_matrix(const cx* a, unsigned n, const uint32_t* q, unsigned k, const cx* m) {
  if (k == 1) return expval1(a, (uint64_t)1 << n, q[0], m);
  return expval_generic(a, n, q, k, m);
}

static int apply_matrix_scaled(cx* a, unsigned n, const uint32_t* q, unsigned k, const cx* m,
                               double prob) {
  if (prob <= 0.0) FAIL(SSB_ERR_DEGENERATE, "channel branch has zero probability");
  const double inv = 1.0 / sqrt(prob);
  cx s[16];
  for (unsigned i = 0; i < (1u << (2 * k)); ++i) s[i] = cscale(m[i], inv);
  apply_matrix(a, n, q, k, s);
  return 0;
}

static double outcome_probability(const cx* a, unsigned n, const uint32_t* q, unsigned k,
                                  uint64_t outcome) {
  uint32_t sorted[64];
  memcpy(sorted, q, k * sizeof(uint32_t));
  sort_small(sorted, k);
  const uint64_t offset = scatter_bits(outcome, q, k);
  const uint64_t groups = (uint64_t)1 << (n - k);
  if (groups <= SUM_BLOCK) {
    double s = 0.0;
    for (uint64_t g = 0; g < groups; ++g) s += norm2(a[expand_index(g, sorted, k) | offset]);
    return s;
  }
  const uint64_t nblk = (groups + SUM_BLOCK - 1) / SUM_BLOCK;
  double* part = malloc(nblk * sizeof(double));
  for (uint64_t b = 0; b < nblk; ++b) {
    double s = 0.0;
    const uint64_t end = (b + 1) * SUM_BLOCK < groups ? (b + 1) * SUM_BLOCK : groups;
    for (uint64_t g = b * SUM_BLOCK; g < end; ++g) s += norm2(a[expand_index(g, sorted, k) | offset]);
    part[b] = s;
  }
  const double r = pairwise_sum(part, nblk);
  free(part);
  return r;
}

static int pick_outcome(const double* probs, uint64_t count, double u, uint64_t* out) {
  double cum = 0.0;
  uint64_t last = count;
  for (uint64_t m = 0; m < count; ++m) {
    cum += probs[m];
    if (u < cum) {
      *out = m;
      return 0;
    }
    if (probs[m] > 0.0) last = m;
  }
  if (last == count) FAIL(SSB_ERR_DEGENERATE, "distribution sums to zero");
  *out = last;
  return 0;
}

static int project(cx* a, unsigned n, const uint32_t* q, unsigned k, uint64_t outcome, double prob) {
  if (prob <= 0.0) FAIL(SSB_ERR_DEGENERATE, "collapse onto zero-probability outcome");
  uint64_t qmask = 0;
  for (unsigned i = 0; i < k; ++i) qmask |= (uint64_t)1 << q[i];
  const uint64_t offset = scatter_bits(outcome, q, k);
  const double inv = 1.0 / sqrt(prob);
  const cx zero = {0.0, 0.0};
  for (uint64_t j = 0; j < ((uint64_t)1 << n); ++j) a[j] = ((j & qmask) == offset) ? cscale(a[j], inv) : zero;
  return 0;
}

static int measure_single(cx* a, unsigned n, const uint32_t* q, unsigned k, double u, uint64_t* m) {
  double probs[1u << SSB_MAX_OP_QUBITS];
  for (uint64_t o = 0; o < ((uint64_t)1 << k); ++o) probs[o] = outcome_probability(a, n, q, k, o);
  int rc = pick_outcome(probs, (uint64_t)1 << k, u, m);
  if (rc) return rc;
  return project(a, n, q, k, *m, probs[*m]);
}

static void x_fix(cx* a, unsigned n, const uint32_t* q, unsigned k, uint64_t m) {
  if (m == 0) return;
  const uint64_t x = scatter_bits(m, q, k);
  unsigned xmax = 63 - (unsigned)__builtin_clzll(x);
  apply_pauli(a, (uint64_t)1 << n, x, 0, 0, xmax);
}

/* ---- exec_naive.cpp:29-129 ---------------------------------------------- */
static int apply_kraus_single(const ssb_flat_program* p, cx* a, unsigned n,
                              const ssb_flat_channel* ch, const uint32_t* q, double u) {
  double cum = 0.0, prob = 0.0;
  cx m[16];
  for (uint32_t i = 0; i < ch->num_matrices; ++i) {
    load_matrix(p, ch->matrix_begin + i, ch->arity, m);
    prob = expval_matrix(a, n, q, ch->arity, m);
    cum += prob;
    if (u < cum) return apply_matrix_scaled(a, n, q, ch->arity, m, prob);
  }
  load_matrix(p, ch->matrix_begin + ch->num_matrices - 1, ch->arity, m);
  return apply_matrix_scaled(a, n, q, ch->arity, m, prob);
}

static uint64_t write_bits(uint64_t creg, const uint32_t* clbits, unsigned k, uint64_t outcome) {
  for (unsigned b = 0; b < k; ++b)
    creg = (creg & ~((uint64_t)1 << clbits[b])) | (((outcome >> b) & 1) << clbits[b]);
  return creg;
}

static uint64_t apply_sample_outcome(const ssb_flat_program* p, uint64_t creg, uint64_t outcome) {
  for (uint32_t i = 0; i < p->num_sample_writes; ++i) {
    const unsigned c = p->sample_write_clbit[i], b = p->sample_write_pos[i];
    creg = (creg & ~((uint64_t)1 << c)) | (((outcome >> b) & 1) << c);
  }
  return creg;
}

static int sample_terminal(const ssb_flat_program* p, const cx* a, double u, uint64_t* outcome) {
  const unsigned k = p->num_sample_qubits;
  const uint64_t count = (uint64_t)1 << k;
  double* probs = malloc(count * sizeof(double));
  for (uint64_t m = 0; m < count; ++m) probs[m] = outcome_probability(a, p->num_qubits, p->sample_qubits, k, m);
  const int rc = pick_outcome(probs, count, u, outcome);
  free(probs);
  return rc;
}

static int pick_term(const ssb_flat_program* p, const ssb_flat_op* op, double u) {
  for (uint32_t t = 0; t < op->term_count; ++t)
    if (u < p->terms[op->term_begin + t].cumulative) return (int)t;
  return (int)op->term_count - 1;
}

static int run_single_shot(const ssb_flat_program* p, uint64_t shot, uint64_t seed, cx* a,
                           uint64_t* creg_out) {
  const unsigned n = p->num_qubits;
  const uint64_t dim = (uint64_t)1 << n;
  memset(a, 0, dim * sizeof(cx));
  a[0].re = 1.0;
  uint64_t creg = 0;
  const uint64_t end = p->sampling_eligible ? p->terminal_measure_begin : p->num_ops;
  int rc = 0;
  for (uint64_t i = 0; i < end && rc == 0; ++i) {
    const ssb_flat_op* op = &p->ops[i];
    if (op->has_condition && (creg & op->cond_mask) != op->cond_value) continue;
    switch (op->kind) {
      case SSB_OP_GATE: {
        cx m[16];
        load_matrix(p, op->matrix, op->num_qubits, m);
        apply_matrix(a, n, op->qubits, op->num_qubits, m);
        break;
      }
      case SSB_OP_PAULI: {
        const int t = pick_term(p, op, oracle_uniform(seed, shot, op->event));
        const ssb_flat_term* tm = &p->terms[op->term_begin + t];
        if (!tm->identity) apply_pauli(a, dim, tm->x_mask, tm->z_mask, tm->num_y, tm->x_max);
        break;
      }
      case SSB_OP_KRAUS:
        rc = apply_kraus_single(p, a, n, &p->channels[op->channel], op->qubits,
                                oracle_uniform(seed, shot, op->event));
        break;
      case SSB_OP_MEASURE: {
        uint64_t m = 0;
        rc = measure_single(a, n, op->qubits, op->num_qubits, oracle_uniform(seed, shot, op->event), &m);
        creg = write_bits(creg, op->clbits, op->num_qubits, m);
        break;
      }
      case SSB_OP_RESET: {
        uint64_t m = 0;
        rc = measure_single(a, n, op->qubits, op->num_qubits, oracle_uniform(seed, shot, op->event), &m);
        if (!rc) x_fix(a, n, op->qubits, op->num_qubits, m);
        break;
      }
      default: break;
    }
  }
  if (rc) return rc;
  if (p->sampling_eligible) {
    uint64_t outcome = 0;
    rc = sample_terminal(p, a, oracle_uniform(seed, shot, p->num_events), &outcome);
    if (rc) return rc;
    creg = apply_sample_outcome(p, creg, outcome);
  }
  *creg_out = creg;
  return 0;
}

typedef struct {
  const ssb_flat_program* p;
  const uint64_t* ids;
  uint64_t begin, end, seed;
  uint64_t* values;
  int rc;
  char err[256];
} chunk_t;

static void* run_chunk(void* arg) {
  chunk_t* c = arg;
  cx* a = malloc(((size_t)1 << c->p->num_qubits) * sizeof(cx));
  for (uint64_t i = c->begin; i < c->end && c->rc == 0; ++i) {
    c->rc = run_single_shot(c->p, c->ids[i], c->seed, a, &c->values[i]);
    if (c->rc) memcpy(c->err, g_err, sizeof c->err);
  }
  free(a);
  return NULL;
}

int oracle_run_shots(const ssb_flat_program* p, const uint64_t* ids, uint64_t count,
                     uint64_t seed, unsigned threads, uint64_t* values_out, double* amps_out) {
  if (p->num_qubits < 1 || p->num_qubits > 30) FAIL(SSB_ERR_INVALID_ARGUMENT, "qubit count must be in [1, 30]");
  if (threads < 1) threads = 1;
  if (threads > count) threads = count ? (unsigned)count : 1;
  chunk_t* ch = calloc(threads, sizeof(chunk_t));
  pthread_t* th = calloc(threads, sizeof(pthread_t));
  uint64_t at = 0;
  for (unsigned t = 0; t < threads; ++t) {
    const uint64_t len = count / threads + (t < count % threads ? 1 : 0);
    ch[t] = (chunk_t){p, ids, at, at + len, seed, values_out, 0, {0}};
    at += len;
    if (threads > 1) pthread_create(&th[t], NULL, run_chunk, &ch[t]);
    else run_chunk(&ch[t]);
  }
  int rc = 0;
  for (unsigned t = 0; t < threads; ++t) {
    if (threads > 1) pthread_join(th[t], NULL);
    if (ch[t].rc && !rc) {
      rc = ch[t].rc;
      memcpy(g_err, ch[t].err, sizeof g_err);
    }
  }
  free(ch);
  free(th);
  if (rc == 0 && amps_out && count > 0) {
    uint64_t v;
    rc = run_single_shot(p, ids[count - 1], seed, (cx*)amps_out, &v);
  }
  return rc;
}

int oracle_final_states(const ssb_flat_program* p, const uint64_t* ids, uint64_t count,
                        uint64_t seed, double* amps_out, uint64_t* cregs_out) {
  const uint64_t dim = (uint64_t)1 << p->num_qubits;
  for (uint64_t i = 0; i < count; ++i) {
    uint64_t v = 0;
    const int rc = run_single_shot(p, ids[i], seed, (cx*)amps_out + i * dim, &v);
    if (rc) return rc;
    if (cregs_out) cregs_out[i] = v;
  }
  return 0;
}

/* ---- exec_branch.cpp:25-295 --------------------------------------------- */
typedef struct {
  uint64_t* v;
  uint64_t n, cap;
} u64vec;

static void vpush(u64vec* v, uint64_t x) {
  if (v->n == v->cap) {
    v->cap = v->cap ? 2 * v->cap : 16;
    v->v = realloc(v->v, v->cap * sizeof(uint64_t));
  }
  v->v[v->n++] = x;
}

typedef struct {
  cx* state;
  u64vec shots;
  uint64_t creg;
} node_t;

typedef struct {
  uint64_t key;
  double param;
  int transform;
  u64vec shots;
} group_t;

/* classify_site (exec_branch.cpp:32-102): groups in ascending key order. */
static int classify(const ssb_flat_program* p, const node_t* node, const ssb_flat_op* site,
                    uint64_t seed, group_t** out, uint64_t* ngroups) {
  const unsigned n = p->num_qubits;
  if (site->has_condition && (node->creg & site->cond_mask) != site->cond_value) {
    group_t* g = calloc(1, sizeof(group_t));
    g->transform = 0;
    for (uint64_t i = 0; i < node->shots.n; ++i) vpush(&g->shots, node->shots.v[i]);
    *out = g;
    *ngroups = 1;
    return 0;
  }
  uint64_t nkeys = 0;
  if (site->kind == SSB_OP_PAULI) nkeys = site->term_count;
  else if (site->kind == SSB_OP_KRAUS) nkeys = p->channels[site->channel].num_matrices;
  else nkeys = (uint64_t)1 << site->num_qubits;
  group_t* b = calloc(nkeys, sizeof(group_t));
  int* used = calloc(nkeys, sizeof(int));
  int rc = 0;
  if (site->kind == SSB_OP_PAULI) {
    for (uint64_t i = 0; i < node->shots.n; ++i) {
      const uint64_t s = node->shots.v[i];
      const int t = pick_term(p, site, oracle_uniform(seed, s, site->event));
      if (!used[t]) {
        used[t] = 1;
        b[t].key = t;
        b[t].transform = !p->terms[site->term_begin + t].identity;
      }
      vpush(&b[t].shots, s);
    }
  } else if (site->kind == SSB_OP_KRAUS) {
    const ssb_flat_channel* ch = &p->channels[site->channel];
    double max_u = 0.0;
    for (uint64_t i = 0; i < node->shots.n; ++i) {
      const double u = oracle_uniform(seed, node->shots.v[i], site->event);
      if (u > max_u) max_u = u;
    }
    double* pr = calloc(ch->num_matrices, sizeof(double));
    double* cum = calloc(ch->num_matrices, sizeof(double));
    uint64_t nc = 0;
    double acc = 0.0;
    cx m[16];
    for (uint32_t i = 0; i < ch->num_matrices; ++i) {
      load_matrix(p, ch->matrix_begin + i, ch->arity, m);
      pr[nc] = expval_matrix(node->state, n, site->qubits, ch->arity, m);
      acc += pr[nc];
      cum[nc++] = acc;
      if (max_u < acc) break;
    }
    for (uint64_t i = 0; i < node->shots.n; ++i) {
      const uint64_t s = node->shots.v[i];
      const double u = oracle_uniform(seed, s, site->event);
      uint64_t sel = nc - 1;
      for (uint64_t j = 0; j < nc; ++j)
        if (u < cum[j]) {
          sel = j;
          break;
        }
      if (!used[sel]) {
        used[sel] = 1;
        b[sel].key = sel;
        b[sel].param = pr[sel];
        b[sel].transform = 1;
      }
      vpush(&b[sel].shots, s);
    }
    free(pr);
    free(cum);
  } else {
    double probs[1u << SSB_MAX_OP_QUBITS];
    for (uint64_t o = 0; o < nkeys; ++o) probs[o] = outcome_probability(node->state, n, site->qubits, site->num_qubits, o);
    for (uint64_t i = 0; i < node->shots.n && !rc; ++i) {
      const uint64_t s = node->shots.v[i];
      uint64_t mo = 0;
      rc = pick_outcome(probs, nkeys, oracle_uniform(seed, s, site->event), &mo);
      if (rc) break;
      if (!used[mo]) {
        used[mo] = 1;
        b[mo].key = mo;
        b[mo].param = probs[mo];
        b[mo].transform = 1;
      }
      vpush(&b[mo].shots, s);
    }
  }
  uint64_t ng = 0;
  for (uint64_t k = 0; k < nkeys; ++k)
    if (used[k]) b[ng++] = b[k];
  free(used);
  *out = b;
  *ngroups = ng;
  return rc;
}

static int apply_decision(const ssb_flat_program* p, node_t* child, const group_t* g,
                          const ssb_flat_op* site) {
  if (!g->transform) return 0;
  const unsigned n = p->num_qubits;
  switch (site->kind) {
    case SSB_OP_PAULI: {
      const ssb_flat_term* t = &p->terms[site->term_begin + g->key];
      apply_pauli(child->state, (uint64_t)1 << n, t->x_mask, t->z_mask, t->num_y, t->x_max);
      return 0;
    }
    case SSB_OP_KRAUS: {
      const ssb_flat_channel* ch = &p->channels[site->channel];
      cx m[16];
      load_matrix(p, ch->matrix_begin + (uint32_t)g->key, ch->arity, m);
      return apply_matrix_scaled(child->state, n, site->qubits, ch->arity, m, g->param);
    }
    case SSB_OP_MEASURE: {
      const int rc = project(child->state, n, site->qubits, site->num_qubits, g->key, g->param);
      child->creg = write_bits(child->creg, site->clbits, site->num_qubits, g->key);
      return rc;
    }
    case SSB_OP_RESET: {
      const int rc = project(child->state, n, site->qubits, site->num_qubits, g->key, g->param);
      if (!rc) x_fix(child->state, n, site->qubits, site->num_qubits, g->key);
      return rc;
    }
    default: return 0;
  }
}

typedef struct {
  uint64_t parent, gi, count, key;
} cand_t;

static int cand_cmp(const void* a, const void* b) {
  const cand_t *x = a, *y = b;
  if (x->count != y->count) return x->count > y->count ? -1 : 1;
  if (x->parent != y->parent) return x->parent < y->parent ? -1 : 1;
  return x->key < y->key ? -1 : (x->key > y->key);
}

static int is_site(const ssb_flat_op* op) {
  return op->kind == SSB_OP_PAULI || op->kind == SSB_OP_KRAUS || op->kind == SSB_OP_MEASURE ||
         op->kind == SSB_OP_RESET;
}

int oracle_run_branch(const ssb_flat_program* p, uint64_t shots, uint64_t seed, uint64_t budget,
                      uint64_t* values_out, uint64_t* peak_out, uint64_t* passes_out) {
  if (shots < 1) FAIL(SSB_ERR_INVALID_ARGUMENT, "shots must be >= 1");
  if (budget < 1) FAIL(SSB_ERR_INVALID_ARGUMENT, "branch budget must be >= 1");
  const unsigned n = p->num_qubits;
  const uint64_t dim = (uint64_t)1 << n;
  const uint64_t end = p->sampling_eligible ? p->terminal_measure_begin : p->num_ops;
  u64vec waiting = {0};
  for (uint64_t s = 0; s < shots; ++s) vpush(&waiting, s);
  uint64_t peak = 0, passes = 0;
  int rc = 0;
  while (waiting.n > 0 && rc == 0) {
    ++passes;
    uint64_t nlive = 1;
    node_t* live = calloc(1, sizeof(node_t));
    live[0].state = calloc(dim, sizeof(cx));
    live[0].state[0].re = 1.0;
    live[0].shots = waiting;
    memset(&waiting, 0, sizeof waiting);
    if (peak < 1) peak = 1;
    uint64_t i = 0;
    while (i < end && rc == 0) {
      uint64_t j = i;
      while (j < end && !is_site(&p->ops[j])) ++j;
      for (uint64_t x = 0; x < nlive; ++x) /* advance_node, exec_branch.cpp:155-162 */
        for (uint64_t o = i; o < j; ++o) {
          const ssb_flat_op* op = &p->ops[o];
          if (op->kind != SSB_OP_GATE) continue;
          if (op->has_condition && (live[x].creg & op->cond_mask) != op->cond_value) continue;
          cx m[16];
          load_matrix(p, op->matrix, op->num_qubits, m);
          apply_matrix(live[x].state, n, op->qubits, op->num_qubits, m);
        }
      if (j == end) break;
      const ssb_flat_op* site = &p->ops[j];
      group_t** groups = calloc(nlive, sizeof(group_t*));
      uint64_t* ng = calloc(nlive, sizeof(uint64_t));
      uint64_t total = 0;
      for (uint64_t x = 0; x < nlive && rc == 0; ++x) {
        rc = classify(p, &live[x], site, seed, &groups[x], &ng[x]);
        total += ng[x];
      }
      if (rc == 0 && total > budget) {
        cand_t* c = malloc(total * sizeof(cand_t));
        uint64_t nc = 0;
        for (uint64_t x = 0; x < nlive; ++x)
          for (uint64_t g = 0; g < ng[x]; ++g) c[nc++] = (cand_t){x, g, groups[x][g].shots.n, groups[x][g].key};
        qsort(c, nc, sizeof(cand_t), cand_cmp);
        uint8_t** keep = calloc(nlive, sizeof(uint8_t*));
        for (uint64_t x = 0; x < nlive; ++x) keep[x] = calloc(ng[x] ? ng[x] : 1, 1);
        for (uint64_t k = 0; k < budget; ++k) keep[c[k].parent][c[k].gi] = 1;
        for (uint64_t x = 0; x < nlive; ++x) {
          uint64_t w = 0;
          for (uint64_t g = 0; g < ng[x]; ++g) {
            if (keep[x][g]) {
              groups[x][w++] = groups[x][g];
            } else {
              for (uint64_t s = 0; s < groups[x][g].shots.n; ++s) vpush(&waiting, groups[x][g].shots.v[s]);
              free(groups[x][g].shots.v);
            }
          }
          ng[x] = w;
          free(keep[x]);
        }
        free(keep);
        free(c);
      }
      /* materialize (exec_branch.cpp:141-153) */
      uint64_t nnext = 0;
      for (uint64_t x = 0; x < nlive; ++x) nnext += ng[x];
      node_t* next = calloc(nnext ? nnext : 1, sizeof(node_t));
      uint64_t at = 0;
      for (uint64_t x = 0; x < nlive && rc == 0; ++x) {
        if (ng[x] == 0) {
          free(live[x].state);
          free(live[x].shots.v);
          continue;
        }
        const uint64_t first = at;
        for (uint64_t g = 0; g < ng[x]; ++g) {
          next[at].creg = live[x].creg;
          next[at].shots = groups[x][g].shots;
          if (g == 0) {
            next[at].state = live[x].state;
          } else {
            next[at].state = malloc(dim * sizeof(cx));
            memcpy(next[at].state, next[first].state, dim * sizeof(cx));
          }
          ++at;
        }
        for (uint64_t g = 0; g < ng[x] && rc == 0; ++g) rc = apply_decision(p, &next[first + g], &groups[x][g], site);
        free(live[x].shots.v);
      }
      for (uint64_t x = 0; x < nlive; ++x) free(groups[x]);
      free(groups);
      free(ng);
      free(live);
      live = next;
      nlive = at;
      if (nlive > peak) peak = nlive;
      i = j + 1;
    }
    for (uint64_t x = 0; x < nlive; ++x) {
      if (rc == 0) {
        if (p->sampling_eligible) {
          const unsigned k = p->num_sample_qubits;
          const uint64_t count = (uint64_t)1 << k;
          double* probs = malloc(count * sizeof(double));
          for (uint64_t m = 0; m < count; ++m) probs[m] = outcome_probability(live[x].state, n, p->sample_qubits, k, m);
          for (uint64_t s = 0; s < live[x].shots.n && rc == 0; ++s) {
            const uint64_t shot = live[x].shots.v[s];
            uint64_t outcome = 0;
            rc = pick_outcome(probs, count, oracle_uniform(seed, shot, p->num_events), &outcome);
            values_out[shot] = apply_sample_outcome(p, live[x].creg, outcome);
          }
          free(probs);
        } else {
          for (uint64_t s = 0; s < live[x].shots.n; ++s) values_out[live[x].shots.v[s]] = live[x].creg;
        }
      }
      free(live[x].state);
      free(live[x].shots.v);
    }
    free(live);
  }
  free(waiting.v);
  if (peak_out) *peak_out = peak;
  if (passes_out) *passes_out = passes;
  return rc;
}
