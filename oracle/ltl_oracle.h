/*
 * ltl_oracle.h -- CPU restatement of the reference Larger-than-Life step.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library,
 * the C-ABI, the catsim host API) may link or call this.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg use it, and only as
 * the checker.
 *
 * Parity status: PINNED.  tests/test_oracle.py checks this restatement against
 *   (1) the reference's own known-answer tests (splitmix64 stream,
 *       alive_threshold edges, init_random first-row pin -- proj/tests/test_grid.cpp),
 *   (2) golden fixtures produced by the reference itself (oracle/_ref, built
 *       from /root/reference/proj/src by oracle/Makefile) in tests/golden/.
 *
 * Semantics follow the torus definition of proj/tests/oracle.hpp:14-67 and the
 * engines' center-multiplicity rule of proj/src/rule.cpp:99-111; all cited
 * lines are under /root/reference/proj.
 */
#ifndef LTL_ORACLE_H
#define LTL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirror of catsim::LtlRule (include/catsim/rule.hpp:17-32). kind: 0 Moore, 1 VN. */
typedef struct {
  int32_t r, c, m, s1, s2, b1, b2, kind;
} orc_rule;

/* splitmix64 step, include/catsim/grid.hpp:31-43. */
uint64_t orc_splitmix64_next(uint64_t* state);

/* Exact "z / 2^64 < density", src/grid.cpp:21-39. */
int orc_alive_threshold(uint64_t z, double density);

/* init_random interior, src/grid.cpp:61-73: one draw per cell of the
 * top-left fill_n x fill_n block in row-major order; the rest stays dead.
 * Writes n*n bytes (row-major interior, no halo).  fill_n < 0 means n.
 * Returns 0, or -1 on invalid arguments (density outside [0,1], fill_n > n). */
int orc_init_random(int32_t n, double density, uint64_t seed, int32_t fill_n,
                    uint8_t* interior);

/* apply_transition, src/rule.cpp:99-111.  Returns the next state (0/1), or
 * -1 where the reference throws "internal consistency: negative count". */
int orc_apply_transition(int state, int reduction, const orc_rule* rule,
                         int center_multiplicity);

/* One generation on a rows x cols torus (row-major, no halo).  Box sum
 * (Moore, center once) or cross sum (VN, center twice) with modular wrap,
 * proj/tests/oracle.hpp:19-33, then the rule with the engines' multiplicity.
 * Returns 0, or -1 if any cell hit the negative-count guard. */
int orc_step(const uint8_t* in, uint8_t* out, int32_t rows, int32_t cols,
             const orc_rule* rule);

/* `steps` generations, ping-ponging a scratch buffer (src/cat_engine.cpp:308-321).
 * In/out may alias.  Returns 0 / -1 as orc_step. */
int orc_simulate(const uint8_t* in, uint8_t* out, int32_t rows, int32_t cols,
                 const orc_rule* rule, int32_t steps);

/* Raw neighbourhood reductions (no rule): H = horizontal window sums and
 * R = box (Moore) / cross (VN) sums, each rows*cols int32. */
void orc_reductions(const uint8_t* in, int32_t rows, int32_t cols,
                    const orc_rule* rule, int32_t* h, int32_t* red);

/* FNV-1a-64 over a byte buffer (offset 0xcbf29ce484222325, prime 0x100000001b3). */
uint64_t orc_fnv1a64(const uint8_t* data, uint64_t len);

/* Periodic halo of a padded (n + 2*halo)^2 row-major buffer, src/grid.cpp:75-94. */
void orc_fill_periodic_halo(uint8_t* padded, int32_t n, int32_t halo);

#ifdef __cplusplus
}
#endif
#endif
