/*
 * gen_core.c -- seeded synthetic-input generator shared by the oracle and the
 * product tests / bench.  It holds none of the method's arithmetic (no SpMM,
 * no cover, no plan): only counter-based random numbers.
 *
 * RNG: SplitMix64 finaliser applied to a (seed, stream, counter) triple, so
 * every value is a pure function of its coordinates -- reproducible, parallel
 * and independent of the thread count.
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC gen_core.c -o libshirogen.so
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t gen_hash(uint64_t seed, uint64_t stream, uint64_t i) {
  return mix64(mix64(mix64(seed) ^ stream) ^ i);
}

/* uniform in [0,1) with 24 random bits: exactly representable in fp32 */
static inline double u24(uint64_t h) { return (double)(h >> 40) * (1.0 / 16777216.0); }
/* uniform in [0,1) with 53 bits */
static inline double u53(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

enum { ST_RMAT = 0x100, ST_UNI_R = 0x200, ST_UNI_C = 0x201, ST_VAL = 0x300,
       ST_B = 0x400, ST_PERM = 0x500 };

/* R-MAT samples k0..k0+m-1: at each of `levels` levels pick a quadrant with
 * probabilities (a, b, c, 1-a-b-c) from gen_hash(seed, ST_RMAT + level, k).
 * Ids >= n are rejected (written as -1). */
void gen_rmat_samples(uint64_t seed, int64_t k0, int64_t m, int32_t levels,
                      double a, double b, double c, int64_t n, int64_t *rows,
                      int64_t *cols) {
  int64_t t;
#pragma omp parallel for schedule(static)
  for (t = 0; t < m; t++) {
    uint64_t k = (uint64_t)(k0 + t);
    int64_t i = 0, j = 0;
    for (int32_t l = 0; l < levels; l++) {
      double u = u53(gen_hash(seed, ST_RMAT + (uint64_t)l, k));
      int rb = 0, cb = 0;
      if (u < a) { rb = 0; cb = 0; }
      else if (u < a + b) { rb = 0; cb = 1; }
      else if (u < a + b + c) { rb = 1; cb = 0; }
      else { rb = 1; cb = 1; }
      i = (i << 1) | rb;
      j = (j << 1) | cb;
    }
    if (i >= n || j >= n) { rows[t] = -1; cols[t] = -1; }
    else { rows[t] = i; cols[t] = j; }
  }
}

/* Uniform (Erdos-Renyi) samples: row and column uniform in [0, n). */
void gen_uniform_samples(uint64_t seed, int64_t k0, int64_t m, int64_t n,
                         int64_t *rows, int64_t *cols) {
  int64_t t;
#pragma omp parallel for schedule(static)
  for (t = 0; t < m; t++) {
    uint64_t k = (uint64_t)(k0 + t);
    rows[t] = (int64_t)(u53(gen_hash(seed, ST_UNI_R, k)) * (double)n);
    cols[t] = (int64_t)(u53(gen_hash(seed, ST_UNI_C, k)) * (double)n);
  }
}

/* Scrambling keys: the permutation is argsort of these (Graph500 style). */
void gen_perm_keys(uint64_t seed, int64_t n, uint64_t *out) {
  int64_t i;
#pragma omp parallel for schedule(static)
  for (i = 0; i < n; i++) out[i] = gen_hash(seed, ST_PERM, (uint64_t)i);
}

/* A values keyed by the final (row, col) position:
 * mode 0: uniform (0, 1];  mode 1: integers {1,2,3,4};  mode 2: all ones. */
void gen_fill_values(uint64_t seed, const int64_t *rows, const int32_t *cols,
                     int64_t nnz, int64_t n, int32_t mode, float *out) {
  int64_t k;
#pragma omp parallel for schedule(static)
  for (k = 0; k < nnz; k++) {
    uint64_t h = gen_hash(seed, ST_VAL, (uint64_t)rows[k] * (uint64_t)n + (uint64_t)cols[k]);
    if (mode == 0) out[k] = (float)(1.0 - u24(h));
    else if (mode == 1) out[k] = (float)(1 + (h >> 62));
    else out[k] = 1.0f;
  }
}

/* Dense B rows row_lo .. row_lo+nrows-1 (global ids), N columns, row-major:
 * mode 0: uniform [0, 1);  mode 1: integers {0..7};  mode 2: integers {0,1}. */
void gen_fill_B(uint64_t seed, int64_t row_lo, int64_t nrows, int64_t N,
                int32_t mode, float *out) {
  int64_t r;
#pragma omp parallel for schedule(static)
  for (r = 0; r < nrows; r++) {
    for (int64_t x = 0; x < N; x++) {
      uint64_t h = gen_hash(seed, ST_B, (uint64_t)(row_lo + r) * (uint64_t)N + (uint64_t)x);
      float v;
      if (mode == 0) v = (float)u24(h);
      else if (mode == 1) v = (float)(h >> 61);
      else v = (float)(h >> 63);
      out[r * N + x] = v;
    }
  }
}

/* Directed R-MAT CSR for very large configs (c5), without materialising the
 * samples: pass 1 counts samples per (scrambled) row, pass 2 regenerates the
 * same counter-based samples and scatters their columns, then every row is
 * sorted and deduplicated.  Result = the distinct entries among samples
 * 0..m-1 (Graph500 convention: m = edge factor x n samples).  perm: old id ->
 * new id (scrambling), or NULL.  Outputs: row_ptr[n+1] (caller-allocated),
 * *col_out (malloc'd, int32, length *nnz_out).  Deterministic, independent of
 * the thread count.  Returns 0 on success. */
static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

int gen_rmat_csr(uint64_t seed, int64_t m, int32_t levels, double a, double b, double c,
                 int64_t n, const int64_t *perm, int64_t *row_ptr, int32_t **col_out,
                 int64_t *nnz_out) {
  int64_t *cnt = calloc(n + 1, sizeof(int64_t));
  if (!cnt) return 1;
  const int64_t CH = 1 << 22;
  int64_t k0;
  /* pass 1: counts */
#pragma omp parallel for schedule(dynamic, 1)
  for (k0 = 0; k0 < m; k0 += CH) {
    int64_t e = k0 + CH < m ? k0 + CH : m;
    for (int64_t k = k0; k < e; k++) {
      int64_t i = 0, j = 0;
      for (int32_t l = 0; l < levels; l++) {
        double u = u53(gen_hash(seed, ST_RMAT + (uint64_t)l, (uint64_t)k));
        int rb = (u >= a + b) ? 1 : 0;
        int cb = (u >= a && u < a + b) || (u >= a + b + c) ? 1 : 0;
        i = (i << 1) | rb;
        j = (j << 1) | cb;
      }
      if (i >= n || j >= n) continue;
      if (perm) i = perm[i];
#pragma omp atomic
      cnt[i + 1]++;
    }
  }
  for (int64_t r = 0; r < n; r++) cnt[r + 1] += cnt[r];
  const int64_t total = cnt[n];
  int32_t *col = malloc(sizeof(int32_t) * (total > 0 ? total : 1));
  int64_t *fill = malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  if (!col || !fill) return 1;
  memcpy(fill, cnt, sizeof(int64_t) * n);
  /* pass 2: scatter columns (order inside a row fixed by the sort below) */
#pragma omp parallel for schedule(dynamic, 1)
  for (k0 = 0; k0 < m; k0 += CH) {
    int64_t e = k0 + CH < m ? k0 + CH : m;
    for (int64_t k = k0; k < e; k++) {
      int64_t i = 0, j = 0;
      for (int32_t l = 0; l < levels; l++) {
        double u = u53(gen_hash(seed, ST_RMAT + (uint64_t)l, (uint64_t)k));
        int rb = (u >= a + b) ? 1 : 0;
        int cb = (u >= a && u < a + b) || (u >= a + b + c) ? 1 : 0;
        i = (i << 1) | rb;
        j = (j << 1) | cb;
      }
      if (i >= n || j >= n) continue;
      if (perm) { i = perm[i]; j = perm[j]; }
      int64_t pos;
#pragma omp atomic capture
      pos = fill[i]++;
      col[pos] = (int32_t)j;
    }
  }
  free(fill);
  /* sort + dedup every row, compact in place row by row */
  int64_t *keep = malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  int64_t r;
#pragma omp parallel for schedule(dynamic, 4096)
  for (r = 0; r < n; r++) {
    int32_t *p = col + cnt[r];
    int64_t len = cnt[r + 1] - cnt[r], w = 0;
    if (len > 1) qsort(p, (size_t)len, sizeof(int32_t), cmp_i32);
    for (int64_t t = 0; t < len; t++)
      if (t == 0 || p[t] != p[t - 1]) p[w++] = p[t];
    keep[r] = w;
  }
  row_ptr[0] = 0;
  for (r = 0; r < n; r++) row_ptr[r + 1] = row_ptr[r] + keep[r];
  for (r = 0; r < n; r++)      /* compact (sequential: destinations never pass sources) */
    if (row_ptr[r] != cnt[r]) memmove(col + row_ptr[r], col + cnt[r], sizeof(int32_t) * keep[r]);
  free(keep);
  free(cnt);
  *nnz_out = row_ptr[n];
  *col_out = realloc(col, sizeof(int32_t) * (row_ptr[n] > 0 ? row_ptr[n] : 1));
  return 0;
}

void gen_free(void *p) { free(p); }
