/*
 * ltl_oracle.c -- CPU restatement of the reference LTL step (TEST INFRASTRUCTURE).
 *
 * See ltl_oracle.h for the contract.  Every function cites the reference
 * lines it restates (paths relative to /root/reference/proj).  The arithmetic
 * is exact integer arithmetic throughout, so agreement with the reference is
 * bit-for-bit, and tests/test_oracle.py pins it against the reference's KATs
 * and against golden fixtures produced by the reference build (oracle/_ref).
 *
 * The window sums are computed as running (sliding) sums along each axis with
 * explicit modular indices.  That is the same multiset of cells the reference
 * visits through its modular halo (src/grid.cpp:75-94) -- duplicates included
 * when 2r+1 > n -- just without re-adding the whole window per cell.
 */
#include "ltl_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* include/catsim/grid.hpp:31-43 */
uint64_t orc_splitmix64_next(uint64_t* state) {
  *state += 0x9E3779B97F4A7C15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* src/grid.cpp:21-39: density = m * 2^(e-53); compare z against m * 2^(e+11)
 * in 128-bit integers so the predicate is exact at every mantissa boundary. */
int orc_alive_threshold(uint64_t z, double density) {
  if (isnan(density) || density <= 0.0) return 0;
  if (density >= 1.0) return 1;
  int e = 0;
  const double frac = frexp(density, &e);
  const uint64_t m = (uint64_t)ldexp(frac, 53);
  const int sh = e + 11;
  if (sh >= 0) return (unsigned __int128)z < ((unsigned __int128)m << sh);
  const int right = -sh;
  if (right >= 64) return z == 0;
  return ((unsigned __int128)z << right) < (unsigned __int128)m;
}

/* src/grid.cpp:61-73 */
int orc_init_random(int32_t n, double density, uint64_t seed, int32_t fill_n,
                    uint8_t* interior) {
  if (!(density >= 0.0 && density <= 1.0)) return -1;
  if (fill_n < 0) fill_n = n;
  if (fill_n > n || n < 0) return -1;
  memset(interior, 0, (size_t)n * (size_t)n);
  uint64_t state = seed;
  for (int32_t y = 0; y < fill_n; ++y)
    for (int32_t x = 0; x < fill_n; ++x)
      interior[(size_t)y * n + x] =
          (uint8_t)orc_alive_threshold(orc_splitmix64_next(&state), density);
  return 0;
}

/* src/rule.cpp:99-111 */
int orc_apply_transition(int state, int reduction, const orc_rule* rule,
                         int center_multiplicity) {
  const int count = reduction - (center_multiplicity - rule->m) * state;
  if (count < 0) return -1;
  if (state) return (count >= rule->s1 && count <= rule->s2) ? 1 : 0;
  return (count >= rule->b1 && count <= rule->b2) ? 1 : 0;
}

static inline int32_t wrap(int64_t v, int32_t n) {
  int64_t m = v % n;
  return (int32_t)(m < 0 ? m + n : m);
}

/* Horizontal window sums, per row: H[y][x] = sum_{|dx|<=r} X[y][(x+dx) mod cols]
 * (the quantity src/cat_engine.cpp:123-161 builds with three banded MMAs). */
static void row_windows(const uint8_t* in, int32_t rows, int32_t cols, int r,
                        int32_t* h) {
  for (int32_t y = 0; y < rows; ++y) {
    const uint8_t* row = in + (size_t)y * cols;
    int32_t* out = h + (size_t)y * cols;
    int32_t s = 0;
    for (int dx = -r; dx <= r; ++dx) s += row[wrap(dx, cols)];
    out[0] = s;
    for (int32_t x = 1; x < cols; ++x) {
      s += row[wrap((int64_t)x + r, cols)];
      s -= row[wrap((int64_t)x - 1 - r, cols)];
      out[x] = s;
    }
  }
}

/* Vertical window sums of an int32 field: V[y][x] = sum_{|dy|<=r} F[(y+dy) mod rows][x]. */
static void col_windows_i32(const int32_t* f, int32_t rows, int32_t cols, int r,
                            int32_t* v) {
  int32_t* acc = (int32_t*)calloc((size_t)cols, sizeof(int32_t));
  for (int dy = -r; dy <= r; ++dy) {
    const int32_t* src = f + (size_t)wrap(dy, rows) * cols;
    for (int32_t x = 0; x < cols; ++x) acc[x] += src[x];
  }
  memcpy(v, acc, (size_t)cols * sizeof(int32_t));
  for (int32_t y = 1; y < rows; ++y) {
    const int32_t* add = f + (size_t)wrap((int64_t)y + r, rows) * cols;
    const int32_t* sub = f + (size_t)wrap((int64_t)y - 1 - r, rows) * cols;
    int32_t* out = v + (size_t)y * cols;
    for (int32_t x = 0; x < cols; ++x) {
      acc[x] += add[x] - sub[x];
      out[x] = acc[x];
    }
  }
  free(acc);
}

static void col_windows_u8(const uint8_t* f, int32_t rows, int32_t cols, int r,
                           int32_t* v) {
  int32_t* acc = (int32_t*)calloc((size_t)cols, sizeof(int32_t));
  for (int dy = -r; dy <= r; ++dy) {
    const uint8_t* src = f + (size_t)wrap(dy, rows) * cols;
    for (int32_t x = 0; x < cols; ++x) acc[x] += src[x];
  }
  memcpy(v, acc, (size_t)cols * sizeof(int32_t));
  for (int32_t y = 1; y < rows; ++y) {
    const uint8_t* add = f + (size_t)wrap((int64_t)y + r, rows) * cols;
    const uint8_t* sub = f + (size_t)wrap((int64_t)y - 1 - r, rows) * cols;
    int32_t* out = v + (size_t)y * cols;
    for (int32_t x = 0; x < cols; ++x) {
      acc[x] += (int32_t)add[x] - (int32_t)sub[x];
      out[x] = acc[x];
    }
  }
  free(acc);
}

/* Moore: R = box sum, center once (tests/oracle.hpp:19-25,
 * src/cat_engine.cpp:163-208).  VN: R = row window + column window, center
 * twice (tests/oracle.hpp:28-33, src/cat_engine.cpp:210-258). */
void orc_reductions(const uint8_t* in, int32_t rows, int32_t cols,
                    const orc_rule* rule, int32_t* h, int32_t* red) {
  if (rows <= 0 || cols <= 0) return;
  row_windows(in, rows, cols, rule->r, h);
  if (rule->kind == 0) {
    col_windows_i32(h, rows, cols, rule->r, red);
  } else {
    col_windows_u8(in, rows, cols, rule->r, red);
    const size_t cells = (size_t)rows * cols;
    for (size_t i = 0; i < cells; ++i) red[i] += h[i];
  }
}

/* One generation: reductions, then src/rule.cpp:99-111 per cell with the
 * engines' multiplicity (1 Moore, 2 VN; src/cat_engine.cpp:288,
 * src/reference.cpp:28). */
int orc_step(const uint8_t* in, uint8_t* out, int32_t rows, int32_t cols,
             const orc_rule* rule) {
  if (rows <= 0 || cols <= 0) return 0;
  const size_t cells = (size_t)rows * cols;
  int32_t* h = (int32_t*)malloc(cells * sizeof(int32_t));
  int32_t* red = (int32_t*)malloc(cells * sizeof(int32_t));
  orc_reductions(in, rows, cols, rule, h, red);
  const int mult = rule->kind == 0 ? 1 : 2;
  int status = 0;
  for (size_t i = 0; i < cells; ++i) {
    const int next = orc_apply_transition(in[i], red[i], rule, mult);
    if (next < 0) status = -1;
    out[i] = (uint8_t)(next < 0 ? 0 : next);
  }
  free(h);
  free(red);
  return status;
}

/* src/cat_engine.cpp:308-321 (steps = 0 returns the input). */
int orc_simulate(const uint8_t* in, uint8_t* out, int32_t rows, int32_t cols,
                 const orc_rule* rule, int32_t steps) {
  const size_t cells = (size_t)rows * (size_t)(cols > 0 ? cols : 0);
  if (steps < 0) return -1;
  if (out != in) memmove(out, in, cells);
  if (steps == 0 || cells == 0) return 0;
  uint8_t* tmp = (uint8_t*)malloc(cells);
  int status = 0;
  for (int32_t s = 0; s < steps; ++s) {
    if (orc_step(out, tmp, rows, cols, rule) != 0) status = -1;
    memcpy(out, tmp, cells);
  }
  free(tmp);
  return status;
}

uint64_t orc_fnv1a64(const uint8_t* data, uint64_t len) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (uint64_t i = 0; i < len; ++i) {
    h ^= data[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* src/grid.cpp:75-94: every halo cell copies its modular interior image. */
void orc_fill_periodic_halo(uint8_t* padded, int32_t n, int32_t halo) {
  if (n <= 0) return;
  const int32_t p = n + 2 * halo;
  for (int32_t y = 0; y < p; ++y) {
    const int32_t sy = halo + wrap((int64_t)y - halo, n);
    for (int32_t x = 0; x < p; ++x) {
      const int interior = y >= halo && y < halo + n && x >= halo && x < halo + n;
      if (interior) continue;
      const int32_t sx = halo + wrap((int64_t)x - halo, n);
      padded[(size_t)y * p + x] = padded[(size_t)sy * p + sx];
    }
  }
}
