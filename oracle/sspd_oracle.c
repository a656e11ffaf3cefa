/*
 * sspd_oracle.c -- plain-C restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see sspd_oracle.h).  Each function names the
 * reference file:line it restates (relative to /root/reference/proj).
 * Parity of this restatement is pinned by tests/test_oracle.py against
 * tests/golden/ (generated from the compiled reference, oracle/_ref).
 */
#include "sspd_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* The reference shifts 32-bit values by computed amounts that can reach 32
 * or more for large r (hashing.hpp:70, hashing.cpp:57).  That is undefined in
 * C++; on x86-64 the hardware masks the count to 5 bits, which is what the
 * compiled reference does.  Mirror it so parity holds for every legal r. */
static inline uint32_t shr32(uint32_t x, uint32_t s) { return x >> (s & 31u); }

/* splitmix64 (src/hashing.cpp:8-14). */
uint64_t so_splitmix64(uint64_t* state) {
  *state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* TabulationHash ctor: 4 tables x 256 entries, filled in order
 * (src/hashing.cpp:18-22). */
void so_tab_init(so_tab* t, uint64_t seed) {
  uint64_t state = seed;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 256; ++j) t->t[i][j] = so_splitmix64(&state);
}

/* TabulationHash::operator() (include/sspd/hashing.hpp:30-33). */
uint64_t so_tab_hash(const so_tab* t, uint32_t key) {
  return t->t[0][key & 0xff] ^ t->t[1][(key >> 8) & 0xff] ^
         t->t[2][(key >> 16) & 0xff] ^ t->t[3][key >> 24];
}

/* HashSeeds: H1 from the first splitmix64 output of seed, row 0 from the
 * second (src/hashing.cpp:24-34). */
void so_seeds_init(so_seeds* s, uint64_t seed) {
  s->seed = seed;
  uint64_t st = seed;
  uint64_t h1_seed = so_splitmix64(&st);
  uint64_t row0_seed = so_splitmix64(&st);
  so_tab_init(&s->h1, h1_seed);
  so_tab_init(&s->row0, row0_seed);
}

/* hash_opposite (include/sspd/hashing.hpp:56-59). */
uint32_t so_hash_opposite(const so_seeds* s, uint32_t oip, uint32_t eta) {
  return (uint32_t)(so_tab_hash(&s->h1, oip) % eta);
}

static inline uint32_t column_mask(const so_cfg* cfg) { return (1u << cfg->q) - 1u; }

/* Row-0 column (src/hashing.cpp:39-40; src/rsea.cpp:31-32). */
uint32_t so_col0(const so_seeds* s, uint32_t cip, const so_cfg* cfg) {
  return (uint32_t)so_tab_hash(&s->row0, cip) & column_mask(cfg);
}

/* rhfg_from_row0 (include/sspd/hashing.hpp:68-71). */
uint32_t so_rhfg_from_row0(uint32_t row, uint32_t cip, uint32_t col0, const so_cfg* cfg) {
  return (shr32(cip, (row - 1) * cfg->delta) ^ col0) & column_mask(cfg);
}

/* rhfg (src/hashing.cpp:36-43). */
int so_rhfg(const so_seeds* s, uint32_t row, uint32_t cip, const so_cfg* cfg, uint32_t* col) {
  if (row >= cfg->r) return -1;
  uint32_t c0 = so_col0(s, cip, cfg);
  *col = row == 0 ? c0 : so_rhfg_from_row0(row, cip, c0, cfg);
  return 0;
}

/* recover_block (include/sspd/hashing.hpp:74-76). */
uint32_t so_recover_block(uint32_t col0, uint32_t coli) { return col0 ^ coli; }

/* blocks_consistent (include/sspd/hashing.hpp:80-84). */
int so_blocks_consistent(uint32_t b_lo, uint32_t b_hi, const so_cfg* cfg) {
  const uint32_t overlap_mask = (1u << (cfg->q - cfg->delta)) - 1u;
  return shr32(b_lo, cfg->delta) == (b_hi & overlap_mask);
}

/* assemble_ip (src/hashing.cpp:45-61): OR the blocks into a 64-bit value at
 * offsets j*delta, truncate to 32 bits, then verify every block against the
 * slice of the result. */
int so_assemble_ip(const uint32_t* blocks, const so_cfg* cfg, uint32_t* ip) {
  const uint32_t nb = cfg->r - 1;
  uint64_t acc = 0;
  for (uint32_t j = 0; j < nb; ++j) {
    uint32_t sh = j * cfg->delta;
    acc |= (uint64_t)blocks[j] << (sh & 63u);
  }
  const uint32_t out = (uint32_t)(acc & 0xffffffffULL);
  for (uint32_t j = 0; j < nb; ++j) {
    uint32_t slice = shr32(out, j * cfg->delta) & column_mask(cfg);
    if (slice != blocks[j]) return 0;
  }
  *ip = out;
  return 1;
}

/* validate_config (src/hashing.cpp:63-87): same checks, same order, same
 * diagnostic text. */
int so_validate_config(const so_cfg* cfg, uint32_t eta, uint32_t k, double theta,
                       char* msg, size_t msg_len) {
  int n = 0;
  char buf[160];
#define SO_PROBLEM(...)                                     \
  do {                                                      \
    if (n == 0 && msg && msg_len) {                         \
      snprintf(buf, sizeof buf, __VA_ARGS__);               \
      snprintf(msg, msg_len, "%s", buf);                    \
    }                                                       \
    ++n;                                                    \
  } while (0)
  if (cfg->q < 1 || cfg->q > 16) SO_PROBLEM("q must be in [1, 16], got %u", cfg->q);
  if (cfg->delta == 0 || cfg->delta >= cfg->q)
    SO_PROBLEM("delta must satisfy 0 < delta < q, got delta=%u q=%u", cfg->delta, cfg->q);
  if (cfg->r < 3) SO_PROBLEM("r must be >= 3, got %u", cfg->r);
  if (cfg->r >= 3 && cfg->delta < cfg->q) {
    uint32_t coverage = (cfg->r - 2) * cfg->delta + cfg->q;
    if (coverage < 32) SO_PROBLEM("address coverage (r-2)*delta+q = %u < 32", coverage);
  }
  if (eta < 2) SO_PROBLEM("eta must be >= 2, got %u", eta);
  if (k < 1 || k > 65534) SO_PROBLEM("k must be in [1, 65534], got %u", k);
  if (theta < 1) {
    /* std::to_string(double) prints with "%f". */
    SO_PROBLEM("theta must be >= 1, got %f", theta);
  }
#undef SO_PROBLEM
  return n;
}

/* hot_cutoff (src/estimator.cpp:32-36). */
size_t so_hot_cutoff(size_t eta, double theta) {
  const double deta = (double)eta;
  return (size_t)ceil(deta * (1.0 - exp(-theta / deta)));
}

/* estimate_cardinality (src/estimator.cpp:25-30). */
double so_estimate_cardinality(size_t eta, size_t r_k) {
  const size_t z0 = eta - r_k;
  const double deta = (double)eta;
  if (z0 == 0) return deta * log(deta);
  return -deta * log((double)z0 / deta);
}

/* rec::active_count (include/sspd/estimator.hpp:26-31). */
size_t so_active_count(const uint16_t* rec, size_t eta, uint32_t k) {
  size_t n = 0;
  for (size_t i = 0; i < eta; ++i) n += (rec[i] < k);
  return n;
}

/* Rsea ctor (src/rsea.cpp:18-27): all recorders start at kNeverSeen. */
int so_grid_init(so_grid* g, const so_cfg* cfg, uint32_t eta) {
  memset(g, 0, sizeof *g);
  if (so_validate_config(cfg, eta, 1, 1.0, NULL, 0) != 0) return -1;
  g->cfg = *cfg;
  g->eta = eta;
  so_seeds_init(&g->seeds, cfg->seed);
  g->n = (size_t)cfg->r * ((size_t)1 << cfg->q) * eta;
  g->cells = (uint16_t*)malloc(g->n * sizeof(uint16_t));
  if (!g->cells) return -1;
  for (size_t i = 0; i < g->n; ++i) g->cells[i] = 0xffff;
  return 0;
}

int so_grid_copy(so_grid* dst, const so_grid* src) {
  *dst = *src;
  dst->cells = (uint16_t*)malloc(src->n * sizeof(uint16_t));
  if (!dst->cells) return -1;
  memcpy(dst->cells, src->cells, src->n * sizeof(uint16_t));
  return 0;
}

void so_grid_free(so_grid* g) {
  free(g->cells);
  g->cells = NULL;
}

/* Rsea::cell_offset (include/sspd/rsea.hpp:105-107). */
size_t so_cell_offset(const so_grid* g, uint32_t row, uint32_t col) {
  return ((size_t)row * ((size_t)1 << g->cfg.q) + col) * g->eta;
}

/* Rsea::update (src/rsea.cpp:29-38). */
void so_update(so_grid* g, uint32_t cip, uint32_t oip) {
  const uint32_t bucket = so_hash_opposite(&g->seeds, oip, g->eta);
  const uint32_t c0 = so_col0(&g->seeds, cip, &g->cfg);
  g->cells[so_cell_offset(g, 0, c0) + bucket] = 0;
  for (uint32_t row = 1; row < g->cfg.r; ++row) {
    uint32_t col = so_rhfg_from_row0(row, cip, c0, &g->cfg);
    g->cells[so_cell_offset(g, row, col) + bucket] = 0;
  }
}

/* Rsea::scan_batch (src/rsea.cpp:40-53): order- and worker-invariant, so a
 * serial loop is the restatement.  pairs = (cip, oip) interleaved. */
void so_scan(so_grid* g, const uint32_t* pairs, size_t n_pairs) {
  for (size_t i = 0; i < n_pairs; ++i) so_update(g, pairs[2 * i], pairs[2 * i + 1]);
}

/* Rsea::advance_slot + rec::advance (src/rsea.cpp:55-63;
 * include/sspd/estimator.hpp:21-24): saturating +1. */
void so_advance(so_grid* g) {
  for (size_t i = 0; i < g->n; ++i)
    if (g->cells[i] < 0xffff) ++g->cells[i];
}

void so_active_counts(const so_grid* g, uint32_t k, uint32_t* out) {
  const size_t cells = (size_t)g->cfg.r << g->cfg.q;
  for (size_t c = 0; c < cells; ++c)
    out[c] = (uint32_t)so_active_count(g->cells + c * g->eta, g->eta, k);
}

/* Rsea::hot_sets (src/rsea.cpp:65-84). */
size_t so_hot_sets(const so_grid* g, uint32_t k, double theta, uint32_t* cols,
                   uint32_t* counts) {
  const size_t cutoff = so_hot_cutoff(g->eta, theta);
  const uint32_t ncol = 1u << g->cfg.q;
  size_t total = 0;
  for (uint32_t row = 0; row < g->cfg.r; ++row) {
    counts[row] = 0;
    for (uint32_t col = 0; col < ncol; ++col) {
      const uint16_t* est = g->cells + so_cell_offset(g, row, col);
      if (so_active_count(est, g->eta, k) >= cutoff) {
        cols[total++] = col;
        ++counts[row];
      }
    }
  }
  return total;
}

/* Rsea::finalize_candidate (src/rsea.cpp:86-108): intersect-max of the r
 * estimators, R_k >= cutoff, assemble, row-0 re-hash check. */
int so_finalize(const so_grid* g, const uint32_t* cols, uint32_t k, double theta,
                so_det* det) {
  const uint32_t r = g->cfg.r;
  size_t r_k = 0;
  for (uint32_t b = 0; b < g->eta; ++b) {
    uint16_t m = g->cells[so_cell_offset(g, 0, cols[0]) + b];
    for (uint32_t row = 1; row < r; ++row) {
      uint16_t v = g->cells[so_cell_offset(g, row, cols[row]) + b];
      if (v > m) m = v;
    }
    r_k += (m < k);
  }
  if (r_k < so_hot_cutoff(g->eta, theta)) return 0;
  uint32_t blocks[64];
  for (uint32_t i = 1; i < r; ++i) blocks[i - 1] = so_recover_block(cols[0], cols[i]);
  uint32_t ip;
  if (!so_assemble_ip(blocks, &g->cfg, &ip)) return 0;
  if (so_col0(&g->seeds, ip, &g->cfg) != cols[0]) return 0;
  det->cip = ip;
  det->r_k = (uint32_t)r_k;
  det->estimate = so_estimate_cardinality(g->eta, r_k);
  return 1;
}

/* ---- growable buffers ---- */
typedef struct {
  uint32_t* v;
  size_t n, cap;
} u32vec;

static void u32_push(u32vec* a, uint32_t x) {
  if (a->n == a->cap) {
    a->cap = a->cap ? a->cap * 2 : 1024;
    a->v = (uint32_t*)realloc(a->v, a->cap * sizeof(uint32_t));
  }
  a->v[a->n++] = x;
}

typedef struct {
  so_det* v;
  size_t n, cap;
} detvec;

static void det_push(detvec* a, so_det d) {
  if (a->n == a->cap) {
    a->cap = a->cap ? a->cap * 2 : 64;
    a->v = (so_det*)realloc(a->v, a->cap * sizeof(so_det));
  }
  a->v[a->n++] = d;
}

static int det_cmp(const void* a, const void* b) {
  const so_det* x = (const so_det*)a;
  const so_det* y = (const so_det*)b;
  if (x->cip != y->cip) return x->cip < y->cip ? -1 : 1;
  /* larger estimate first so the first of each run is the one kept */
  if (x->estimate != y->estimate) return x->estimate > y->estimate ? -1 : 1;
  if (x->r_k != y->r_k) return x->r_k > y->r_k ? -1 : 1;
  return 0;
}

/* dedup_report (src/rsea.cpp:112-122): by cip, keep the larger estimate,
 * ascending cip. */
static void dedup(detvec* d) {
  if (d->n == 0) return;
  qsort(d->v, d->n, sizeof(so_det), det_cmp);
  size_t w = 0;
  for (size_t i = 0; i < d->n; ++i)
    if (w == 0 || d->v[w - 1].cip != d->v[i].cip) d->v[w++] = d->v[i];
  d->n = w;
}

typedef struct {
  uint32_t* cols;
  uint32_t counts[64];
  uint32_t start[64];
} hotlist;

static void hot_build(const so_grid* g, uint32_t k, double theta, hotlist* h) {
  h->cols = (uint32_t*)malloc(((size_t)g->cfg.r << g->cfg.q) * sizeof(uint32_t));
  so_hot_sets(g, k, theta, h->cols, h->counts);
  uint32_t s = 0;
  for (uint32_t row = 0; row < g->cfg.r; ++row) {
    h->start[row] = s;
    s += h->counts[row];
  }
}

/* Rsea::reconstruct_leveled (src/rsea.cpp:168-255). */
int so_reconstruct_leveled(const so_grid* g, uint32_t k, double theta, size_t cap,
                           so_det** out, size_t* n_out, uint32_t* ovf_level,
                           size_t* ovf_count) {
  const so_cfg* cfg = &g->cfg;
  hotlist h;
  hot_build(g, k, theta, &h);
  *out = NULL;
  *n_out = 0;
  for (uint32_t row = 0; row < cfg->r; ++row)
    if (h.counts[row] == 0) {  /* rsea.cpp:173-174 */
      free(h.cols);
      return 0;
    }
  const uint32_t* H0 = h.cols + h.start[0];
  const uint32_t* H1 = h.cols + h.start[1];
  const uint32_t* H2 = h.cols + h.start[2];
  u32vec rd = {0}, wr = {0};
  /* Level 2: all consistent triples (rsea.cpp:179-201). */
  for (uint32_t a = 0; a < h.counts[0]; ++a)
    for (uint32_t b = 0; b < h.counts[1]; ++b)
      for (uint32_t c = 0; c < h.counts[2]; ++c) {
        uint32_t c0 = H0[a], c1 = H1[b], c2 = H2[c];
        if (!so_blocks_consistent(so_recover_block(c0, c1), so_recover_block(c0, c2), cfg))
          continue;
        u32_push(&rd, c0);
        u32_push(&rd, c1);
        u32_push(&rd, c2);
      }
  size_t m = 3;
  if (rd.n / m > cap) {  /* collect(2), rsea.cpp:206-216 */
    *ovf_level = 2;
    *ovf_count = rd.n / m;
    free(rd.v);
    free(h.cols);
    return 1;
  }
  /* Levels 3..r-1 (rsea.cpp:218-237). */
  for (uint32_t row = 3; row < cfg->r; ++row) {
    const uint32_t* Hr = h.cols + h.start[row];
    const size_t nt = rd.n / m;
    wr.n = 0;
    for (size_t t = 0; t < nt; ++t) {
      const uint32_t* tup = rd.v + t * m;
      const uint32_t b_prev = so_recover_block(tup[0], tup[m - 1]);
      for (uint32_t j = 0; j < h.counts[row]; ++j) {
        const uint32_t col = Hr[j];
        if (!so_blocks_consistent(b_prev, so_recover_block(tup[0], col), cfg)) continue;
        for (size_t x = 0; x < m; ++x) u32_push(&wr, tup[x]);
        u32_push(&wr, col);
      }
    }
    ++m;
    if (wr.n / m > cap) {
      *ovf_level = row;
      *ovf_count = wr.n / m;
      free(rd.v);
      free(wr.v);
      free(h.cols);
      return 1;
    }
    u32vec tmp = rd;
    rd = wr;
    wr = tmp;
  }
  /* Finalization (rsea.cpp:239-254) and dedup. */
  detvec found = {0};
  const size_t nf = rd.n / cfg->r;
  for (size_t t = 0; t < nf; ++t) {
    so_det d;
    if (so_finalize(g, rd.v + t * cfg->r, k, theta, &d)) det_push(&found, d);
  }
  dedup(&found);
  free(rd.v);
  free(wr.v);
  free(h.cols);
  *out = found.v;
  *n_out = found.n;
  return 0;
}

typedef struct {
  const so_grid* g;
  uint32_t k;
  double theta;
  hotlist* h;
  uint32_t tuple[64];
  detvec* found;
} dfs_ctx;

/* The `extend` lambda of reconstruct_recursive (src/rsea.cpp:133-145). */
static void dfs_extend(dfs_ctx* c, uint32_t row) {
  const so_cfg* cfg = &c->g->cfg;
  if (row == cfg->r) {
    so_det d;
    if (so_finalize(c->g, c->tuple, c->k, c->theta, &d)) det_push(c->found, d);
    return;
  }
  const uint32_t b_prev = so_recover_block(c->tuple[0], c->tuple[row - 1]);
  const uint32_t* Hr = c->h->cols + c->h->start[row];
  for (uint32_t j = 0; j < c->h->counts[row]; ++j) {
    const uint32_t col = Hr[j];
    if (!so_blocks_consistent(b_prev, so_recover_block(c->tuple[0], col), cfg)) continue;
    c->tuple[row] = col;
    dfs_extend(c, row + 1);
  }
}

/* Rsea::reconstruct_recursive (src/rsea.cpp:126-166). */
int so_reconstruct_recursive(const so_grid* g, uint32_t k, double theta, so_det** out,
                             size_t* n_out) {
  hotlist h;
  hot_build(g, k, theta, &h);
  detvec found = {0};
  dfs_ctx c = {g, k, theta, &h, {0}, &found};
  const uint32_t* H0 = h.cols + h.start[0];
  const uint32_t* H1 = h.cols + h.start[1];
  const uint32_t* H2 = h.cols + h.start[2];
  for (uint32_t a = 0; a < h.counts[0]; ++a) {
    c.tuple[0] = H0[a];
    for (uint32_t b = 0; b < h.counts[1]; ++b) {
      c.tuple[1] = H1[b];
      const uint32_t b1 = so_recover_block(c.tuple[0], c.tuple[1]);
      for (uint32_t x = 0; x < h.counts[2]; ++x) {
        const uint32_t c2 = H2[x];
        if (!so_blocks_consistent(b1, so_recover_block(c.tuple[0], c2), &g->cfg)) continue;
        c.tuple[2] = c2;
        if (g->cfg.r == 3) {
          so_det d;
          if (so_finalize(g, c.tuple, k, theta, &d)) det_push(&found, d);
        } else {
          dfs_extend(&c, 3);
        }
      }
    }
  }
  dedup(&found);
  free(h.cols);
  *out = found.v;
  *n_out = found.n;
  return 0;
}

/* merge_rseas (src/snapshot.cpp:117-142). */
int so_merge(so_grid* out, const so_grid* const* grids, size_t n, int policy) {
  if (n == 0) return -1;
  const so_grid* f = grids[0];
  for (size_t i = 0; i < n; ++i) {
    const so_grid* x = grids[i];
    if (x->cfg.seed != f->cfg.seed || x->cfg.q != f->cfg.q || x->cfg.r != f->cfg.r ||
        x->cfg.delta != f->cfg.delta || x->eta != f->eta)
      return -1;
  }
  if (so_grid_copy(out, f) != 0) return -1;
  for (size_t gi = 1; gi < n; ++gi) {
    const uint16_t* in = grids[gi]->cells;
    if (policy == SO_UNION_MIN) {
      for (size_t i = 0; i < out->n; ++i)
        if (in[i] < out->cells[i]) out->cells[i] = in[i];
    } else {
      for (size_t i = 0; i < out->n; ++i)
        if (in[i] > out->cells[i]) out->cells[i] = in[i];
    }
  }
  return 0;
}

int so_grid_equal(const so_grid* a, const so_grid* b) {
  return a->n == b->n && memcmp(a->cells, b->cells, a->n * sizeof(uint16_t)) == 0;
}

/* slot_of (include/sspd/workload.hpp:64-66). */
static uint64_t slot_of(uint32_t ts, double mu, uint32_t start) {
  return (uint64_t)((ts - start) / mu);
}

/* run_detection (src/pipeline.cpp:16-89).  The alpha batching of the
 * reference does not change the grid (scan is order invariant), so each
 * node's slot is scanned in one call. */
int so_run_detection(const so_cfg* cfg, uint32_t eta, double mu, uint32_t k,
                     uint32_t start, double theta, int policy, size_t cap,
                     const uint32_t* recs, const size_t* shard_off, size_t n_shards,
                     uint64_t* n_slots_out, so_report_row** out, size_t* n_out) {
  *out = NULL;
  *n_out = 0;
  *n_slots_out = 0;
  if (n_shards == 0) return -1;
  if (so_validate_config(cfg, eta, k, theta, NULL, 0) != 0) return -1;
  uint64_t n_slots = 0;
  for (size_t i = 0; i < shard_off[n_shards]; ++i) {
    uint32_t ts = recs[3 * i];
    if (ts < start) return -1;
    uint64_t s = slot_of(ts, mu, start) + 1;
    if (s > n_slots) n_slots = s;
  }
  so_grid* nodes = (so_grid*)calloc(n_shards, sizeof(so_grid));
  size_t* cursor = (size_t*)calloc(n_shards, sizeof(size_t));
  for (size_t i = 0; i < n_shards; ++i) {
    so_grid_init(&nodes[i], cfg, eta);
    cursor[i] = shard_off[i];
  }
  size_t rows_cap = 0, rows_n = 0;
  so_report_row* rows = NULL;
  int rc = 0;
  for (uint64_t slot = 0; slot < n_slots && rc == 0; ++slot) {
    for (size_t i = 0; i < n_shards; ++i) {
      size_t* pos = &cursor[i];
      while (*pos < shard_off[i + 1] && slot_of(recs[3 * *pos], mu, start) == slot) {
        so_update(&nodes[i], recs[3 * *pos + 1], recs[3 * *pos + 2]);
        ++*pos;
      }
    }
    so_grid merged;
    const so_grid* target = &nodes[0];
    int have_merged = 0;
    if (n_shards > 1) {
      const so_grid** ptrs = (const so_grid**)malloc(n_shards * sizeof(so_grid*));
      for (size_t i = 0; i < n_shards; ++i) ptrs[i] = &nodes[i];
      so_merge(&merged, ptrs, n_shards, policy);
      free(ptrs);
      target = &merged;
      have_merged = 1;
    }
    so_det* dets;
    size_t nd;
    uint32_t lvl;
    size_t cnt;
    if (so_reconstruct_leveled(target, k, theta, cap, &dets, &nd, &lvl, &cnt) != 0) {
      rc = 1;
    } else {
      for (size_t d = 0; d < nd; ++d) {
        if (rows_n == rows_cap) {
          rows_cap = rows_cap ? rows_cap * 2 : 64;
          rows = (so_report_row*)realloc(rows, rows_cap * sizeof(so_report_row));
        }
        rows[rows_n].slot = slot;
        rows[rows_n].det = dets[d];
        ++rows_n;
      }
      free(dets);
    }
    if (have_merged) so_grid_free(&merged);
    for (size_t i = 0; i < n_shards; ++i) so_advance(&nodes[i]);
  }
  for (size_t i = 0; i < n_shards; ++i) so_grid_free(&nodes[i]);
  free(nodes);
  free(cursor);
  *n_slots_out = n_slots;
  *out = rows;
  *n_out = rows_n;
  return rc;
}

void so_free(void* p) { free(p); }

/* std::mt19937_64 parameters (C++ [rand.predef]). */
void so_mt64_seed(so_mt64* m, uint64_t seed) {
  m->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
  m->idx = 312;
}

uint64_t so_mt64_next(so_mt64* m) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (m->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (m->mt[i] & UM) | (m->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
      m->mt[i] = m->mt[(i + 156) % 312] ^ xa;
    }
    m->idx = 0;
  }
  uint64_t x = m->mt[m->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

void so_mt64_fill(so_mt64* m, uint64_t* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = so_mt64_next(m);
}

uint64_t so_fnv1a64(const void* data, size_t n_bytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ULL;
  for (size_t i = 0; i < n_bytes; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}
