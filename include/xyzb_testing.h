/*
 * xyzb_testing.h — test-only hook of libxyzb.so (NOT part of the drop-in
 * boundary in xyzb.h; no reference interface corresponds to it).
 *
 * The unit tests force rare engine paths with process-wide options; 0
 * restores the engine's own choice:
 *   batch_entries   runs per batch = max(1, value / p) (multi-batch searches)
 *   hit_cap         initial hit-buffer capacity (the regrow-and-redo path)
 *   item_cap        item-buffer capacity (regrow path)
 *   pair_cap        pair-list capacity (regrow path)
 *   grouping        1 = per-run cluster radix sort, 2 = partition path for any
 *                   M <= 24, 3 = the cluster of 16-bit tables for M = 19, 20
 *                   and sparse bucket spaces
 *   merge_large     the multi-kernel merge instead of the single-CTA merge
 *   sign_verify_off the exact verifies instead of the bit-plane ones (the sign
 *                   transform's fp32 columns; continuous-Y's fp64 set-bit sums)
 *   trace           host-side phase times of dataset creation on stderr
 *   brute_cuda      the CUDA-core exhaustive oracle instead of tcgen05
 *   binned          1 = the binned verify (binned_verify.cuh) for any binary
 *                   search it supports, -1 = never (the per-batch verify)
 *   binned_wshift   z-side windows of 2^value columns (several windows at
 *                   small p)
 *   binned_cap      initial window-region capacity in pairs (the regrow path)
 *   one_pass_join   1 = the binned verify's one-pass partition join even when
 *                   runs are expected near the guard (aborted runs' pairs are
 *                   then dropped while binned)
 *   part_fixed      the keyless partition pass with fixed-capacity regions (no
 *                   count pass): -1 = never, N > 0 = N records per partition
 *                   (a small N overflows: the counted redo)
 * Returns XYZB_OK, or XYZB_E_DATA for an unknown name.
 */
#ifndef XYZB_TESTING_H
#define XYZB_TESTING_H

#ifdef __cplusplus
extern "C" {
#endif

int xyzb_test_set_option(const char* name, long long value);

#ifdef __cplusplus
}
#endif

#endif /* XYZB_TESTING_H */
