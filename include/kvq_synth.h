/*
 * kvq_synth.h — seeded synthetic input generator in libkvq.so (device side).
 *
 * Input generation only: holds none of the method's arithmetic.  It is the
 * device implementation of the counter-based generator of SURVEY.md §8(d);
 * the CPU oracle implements the same generator independently
 * (oracle/kvq_oracle.c:kvqo_fill) and both are pinned to the same test vector
 * (tests/golden/survey_appendix.json: rng_seed42_first6_bits).
 *
 *   splitmix64(seed, i): z = seed + (i+1)*0x9E3779B97F4A7C15;
 *                        z = (z ^ z>>30) * 0xBF58476D1CE4E5B9;
 *                        z = (z ^ z>>27) * 0x94D049BB133111EB;  z ^= z>>31
 *   uniform(seed, i) = ((int32)(splitmix64(seed, i) >> 40) - 2^23) * 2^-23
 *
 * Element (t, d) of the global T x D matrix uses index i = t*D + d, so a rank
 * that generates only rows [row0, row0+rows) gets exactly those rows of the
 * unsharded matrix ("values in [-1, 1]"; reading Q12).
 */
#ifndef KVQ_SYNTH_H
#define KVQ_SYNTH_H

#include <stdint.h>

#include "kvq.h"

#ifdef __cplusplus
extern "C" {
#endif

enum {
    KVQ_DIST_UNIFORM = 0, /* uniform lattice k*2^-23 in [-1, 1) */
    KVQ_DIST_OUTLIER = 1, /* column d scaled by 2^(e_d), e_d = splitmix64(seed^0xC0FFEE, d) % 9 - 4 */
    KVQ_DIST_ONGRID = 2   /* x = c*s_d, s_d = j_d*2^-24 (j_d odd < 2^17), row 0 = +-127 (fact 6) */
};

/* out: device [rows][D] float32 = rows [row0, row0+rows) of the seeded matrix.
 * Asynchronous on `stream`.  KVQ_ERR_INVALID_VALUE for NULL/rows<1/D<1/bad dist. */
kvq_status kvq_synth_fill(float *out, int64_t row0, int64_t rows, int64_t D, uint64_t seed,
                          int dist, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* KVQ_SYNTH_H */
