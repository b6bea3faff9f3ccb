/*
 * xyzb_synth.h — seeded synthetic inputs with the shapes of BASELINE.json's
 * configs (libxyzb_synth.so). Host-side data generation for the bench and the
 * tests; not part of the search path. The LURIC data the paper measures on is
 * private, so these generators stand in for it. Recipes:
 *
 *  toy    : the reference's own recipe, rademacher_matrix + plant_interaction
 *           on make_stream(seed, 0x5e17) (proj/core/src/synthetic.cpp:12-38):
 *           one rng() per word, Y = X_j X_k on exactly round(gamma n) rows.
 *  gwas   : per column maf ~ U[0.05, 0.5]; X = +1 iff genotype > 0 for
 *           genotype ~ Bin(2, maf), i.e. P(+1) = 1 - (1 - maf)^2;
 *           P(Y = +1) = sigmoid(coef * sum_q X_aq X_bq) over planted pairs.
 *  gauss  : X ~ N(0,1) columns standardised (mean 0, sd 1), stored fp32-exact;
 *           Y = sum_q theta X_aq X_bq + noise_sd * N(0,1).
 *  ar1    : blocks of `block` columns, Z_j = rho Z_{j-1} + sqrt(1-rho^2) e,
 *           e standardised Irwin-Hall(4) (a near-Gaussian, cheap enough for
 *           1e10 entries), X = +1 iff Z > 0; Y = sign(sum_q X_aq X_bq) (ties
 *           +1), then each row flipped with probability `flip`.
 * All non-toy generators are counter-based (splitmix64 of seed/column/row),
 * so they are deterministic for any thread count.
 */
#ifndef XYZB_SYNTH_H
#define XYZB_SYNTH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* x_words: p * ceil(n/64) uint64 (column-major, padding 0); y: n int8 (+-1) */
int xyzb_synth_toy(uint64_t n, uint64_t p, uint64_t j, uint64_t k, double gamma, uint64_t seed,
                   uint64_t* x_words, int8_t* y);

/* pairs: 2 * n_pairs uint32 written (the planted pairs, j < k) */
int xyzb_synth_gwas(uint64_t n, uint64_t p, uint64_t n_pairs, double coef, uint64_t seed,
                    uint64_t* x_words, int8_t* y, uint32_t* pairs);

/* x: column-major p * n doubles (values exactly representable in fp32); y: n doubles */
int xyzb_synth_gauss(uint64_t n, uint64_t p, uint64_t n_pairs, double theta, double noise_sd,
                     uint64_t n_mains, double beta, uint64_t seed, double* x, double* y, uint32_t* pairs,
                     uint32_t* mains);

int xyzb_synth_ar1(uint64_t n, uint64_t p, uint64_t block, double rho, uint64_t n_pairs, double flip,
                   uint64_t seed, uint64_t* x_words, int8_t* y, uint32_t* pairs);

#ifdef __cplusplus
}
#endif

#endif
