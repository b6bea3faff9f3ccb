/*
 * xyzb.h — C ABI of the B200 xyz interaction-search engine (libxyzb.so).
 *
 * This is the drop-in boundary for the reference's hot path. Every entry
 * point below replaces one reference interface; the reference file:line is
 * cited beside it (paths relative to the reference repo root).
 *
 *   xyzb_dataset_create/destroy  X upload, kept resident in HBM across calls
 *   xyzb_dataset_open            (or X read from an XYZ1 file: read_dataset,
 *                                proj/core/src/dataset_io.cpp:91-129).
 *                                Replaces the per-call X argument of the three
 *                                xyz::xyz_search overloads
 *                                (proj/core/include/xyz/search.hpp:100-111),
 *                                PackedMatrix layout packed_matrix.hpp:10-14,
 *                                RealMatrix layout real_matrix.hpp:13-33.
 *   xyzb_search                  the three xyz::xyz_search overloads
 *                                (proj/core/src/search.cpp:325,367,415) with
 *                                run_search/run_pass (search.cpp:65-111,295-321).
 *   xyzb_project_keys            project_keys (proj/core/src/projection.cpp:32-57)
 *   xyzb_equal_pairs             equal_pairs  (proj/core/src/pair_search.cpp:26-55)
 *   xyzb_pair_strengths          interaction_strength / weighted_interaction_strength
 *                                (proj/core/src/transforms.cpp:33-76) and the
 *                                continuous-XY strength (search.cpp:477-493)
 *   xyzb_merge_results           the slot-ordered merge + dedup of run_pass
 *                                (search.cpp:96-108) applied across GPUs
 *   xyzb_brute_force             oracle::brute_force_search, binary overload
 *                                (proj/core/include/xyz/oracle.hpp:36-37,
 *                                proj/core/src/oracle.cpp:24-59, 84-91)
 *
 * Conventions: plain pointers and sizes, caller owns inputs (borrowed for the
 * call), the library owns device buffers (dataset handle) and result buffers
 * (freed by xyzb_result_free). Errors return a status code plus a message in
 * `err` (may be NULL). Status codes mirror the reference's exception taxonomy
 * and CLI exit codes (proj/core/include/xyz/errors.hpp:10-25,
 * proj/tools/xyz_main.cpp:601-619).
 *
 * Threading: one host thread per dataset at a time (not re-entrant on the same
 * handle); each dataset owns one CUDA stream on its device, and calls on
 * different datasets from different host threads run concurrently (device
 * buffers return to the shared pool after their own stream drains, not after
 * a device-wide synchronisation).
 */
#ifndef XYZB_H
#define XYZB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XYZB_ABI_VERSION 3

/* status codes */
enum {
    XYZB_OK = 0,
    XYZB_E_DATA = 3,     /* xyz::data_error   (errors.hpp:10-13), exit code 3 */
    XYZB_E_GUARD = 4,    /* xyz::guard_error  (errors.hpp:16-19), exit code 4 */
    XYZB_E_SOLVER = 5,   /* xyz::solver_error (errors.hpp:22-25), exit code 5 */
    XYZB_E_CUDA = 10,    /* CUDA runtime failure / no device */
    XYZB_E_INTERNAL = 11 /* capacity or invariant failure inside the engine */
};

/* SearchMode (search.hpp:14) */
enum { XYZB_MODE_BINARY = 0, XYZB_MODE_CONTINUOUS_Y = 1, XYZB_MODE_CONTINUOUS_XY = 2 };
/* BinarizeTransform (search.hpp:16) */
enum { XYZB_TRANSFORM_NONE = 0, XYZB_TRANSFORM_SIGN = 1, XYZB_TRANSFORM_UNBIASED = 2 };

typedef struct xyzb_dataset xyzb_dataset;

/* The design matrix. Exactly one of x_words / x_real / x_real32 is set.
 *  x_words:  binary X, column-major, W = ceil(n_rows/64) uint64 words per
 *            column, bit i%64 of word i/64 set iff X_ij = +1, padding bits 0
 *            (PackedMatrix, packed_matrix.hpp:10-14).
 *  x_real:   real X, column-major doubles (RealMatrix, real_matrix.hpp:13-33).
 *  x_real32: real X, column-major floats (half the upload of x_real; the
 *            search reads fp32 columns anyway; the fp64 comparisons of the
 *            transforms see double(x), as a RealMatrix built from the floats).
 * Devices: n_devices == 0 places the dataset on `device`. n_devices > 0
 * replicates X on devices[0..n_devices) (X replicated, runs
 * sharded): xyzb_search then splits the repetitions of each pass into
 * contiguous shards, one per device (one host thread and stream each), and
 * merges the shard results on devices[0] — the same report as one device.
 * This replaces the std::thread waves of run_pass (search.cpp:59-111). */
typedef struct {
    uint64_t n_rows;
    uint64_t n_cols;
    const uint64_t* x_words;
    const double* x_real;
    int32_t device; /* CUDA ordinal (n_devices == 0) */
    int32_t flags;  /* reserved, 0 */
    const float* x_real32;
    const int32_t* devices;
    uint64_t n_devices;
} xyzb_problem;

/* The response. Binary mode: y_sign (+1/-1 per row). Continuous modes: y_real. */
typedef struct {
    const int8_t* y_sign;
    const double* y_real;
} xyzb_response;

/* SearchConfig (search.hpp:18-33) plus engine extensions. */
typedef struct {
    uint64_t m;                      /* subsample size 1..64            */
    uint64_t l;                      /* repetitions per pass            */
    double gamma;                    /* strength threshold (0,1]        */
    int32_t mode;                    /* XYZB_MODE_*                     */
    int32_t transform;               /* XYZB_TRANSFORM_*                */
    int32_t search_negatives;        /* bool                            */
    int32_t stop_after_first_hit;    /* bool                            */
    int32_t estimate_complexity;     /* bool                            */
    int32_t threads;                 /* accepted, ignored by the GPU    */
    uint64_t seed;
    uint64_t max_candidates_per_rep; /* 0 -> 16 * n_cols                */
    uint64_t strength_sample_size;   /* 0 -> min(1e5, 10 * n_cols)      */
    /* engine extensions */
    uint64_t top_k;     /* 0 = no top-K list; else K (A.10 comparator)       */
    uint64_t rep_begin; /* run shard: repetitions [rep_begin, rep_end) of     */
    uint64_t rep_end;   /* each pass, 1-based end-exclusive; 0,0 = all 1..L   */
    int32_t top_k_mode; /* XYZB_TOPK_*                                        */
    int32_t reserved;   /* 0                                                   */
} xyzb_params;

/* top_k_mode:
 *  XYZB_TOPK_HITS        top-K of the hit list (strength >= gamma), A.10 order.
 *  XYZB_TOPK_CANDIDATES  top-K over ALL verified candidates (gamma ignored;
 *      needs top_k >= 1): the report's hits are the reference's A.8 hit list
 *      at gamma_effective = the strength of the K-th ranked distinct
 *      candidate (ties at that strength included), i.e. exactly what
 *      xyz_search returns with gamma = gamma_effective; top_k ranks them.
 *      SURVEY Appendix A.10's gamma-lowering procedure yields the same top-K. */
enum { XYZB_TOPK_HITS = 0, XYZB_TOPK_CANDIDATES = 1 };

/* InteractionHit (pair_search.hpp:29-35) */
typedef struct {
    uint32_t j;
    uint32_t k;
    double strength;
    uint32_t found_at_repetition;
    int32_t sign;
} xyzb_hit;

enum {
    XYZB_STAGE_DRAWS = 0,   /* host RNG draws + upload          */
    XYZB_STAGE_PROJECT = 1, /* keys                             */
    XYZB_STAGE_SORT = 2,    /* segmented LSD radix sort         */
    XYZB_STAGE_JOIN = 3,    /* bucket join + guard + scan       */
    XYZB_STAGE_VERIFY = 4,  /* strength verification            */
    XYZB_STAGE_MERGE = 5,   /* dedup + order + top-K            */
    XYZB_STAGE_ESTIMATE = 6,/* sample_strengths                 */
    XYZB_STAGE_OTHER = 7,
    XYZB_NUM_STAGES = 8
};

/* SearchReport (search.hpp:45-56) plus engine counters. */
typedef struct {
    xyzb_hit* hits;
    uint64_t n_hits;
    uint64_t* order_keys;  /* per hit: its block key v (x side); reference order is (run, v, j, k) */
    uint64_t* top_k;       /* indices into hits, A.10 order                  */
    uint64_t n_top_k;
    uint64_t repetitions_run;
    uint64_t candidates_checked;    /* engine: canonical pairs verified */
    uint64_t candidates_enumerated; /* sum |E_l| incl. the diagonal (= reference)       */
    uint64_t aborted_repetitions;
    double wall_time_s;
    double estimated_c;
    double gamma0;
    uint64_t m_used;
    uint64_t l_used;
    /* engine telemetry */
    uint64_t runs_executed;      /* runs computed on the device (before stop truncation) */
    uint64_t verified_pairs;     /* canonical off-diagonal pairs verified, non-aborted runs */
    double device_ms;            /* CUDA-event time on the stream from the search start to the merged
                                    hits in device memory (+ the complexity estimate if it ran); the
                                    copy of the results to the host is not included */
    double stage_ms[XYZB_NUM_STAGES];
    uint64_t stage_bytes[XYZB_NUM_STAGES]; /* algorithmic bytes per stage */
    uint64_t stage_launches[XYZB_NUM_STAGES];
    uint64_t kernel_launches;
    double verify_kernel_ms;     /* summed CUDA-event duration of the verify launches */
    uint64_t verify_launches;
    double gamma_effective;      /* the hit test's gamma (XYZB_TOPK_CANDIDATES: the K-th strength) */
    uint64_t devices_used;       /* devices the runs were sharded over */
    uint64_t attempts;           /* times the device ran the search: 1, or more after a buffer or partition
                                    capacity was outgrown and the search redone (device_ms covers them all);
                                    sharded: the largest of the shards */
} xyzb_result;

/* ---- lifecycle ---- */
int xyzb_abi_version(void);
void xyzb_params_init(xyzb_params* params); /* reference SearchConfig defaults */
int xyzb_device_count(void);

int xyzb_dataset_create(const xyzb_problem* problem, xyzb_dataset** out, char* err, size_t errlen);
void xyzb_dataset_destroy(xyzb_dataset* ds);

/* X straight from an XYZ1 file (read_dataset, proj/core/src/dataset_io.cpp:91-129:
 * magic "XYZ1", kind byte 0 binary / 1 real, 3 reserved bytes, n and p as
 * little-endian u64, then the column-major payload), streamed through pinned
 * staging to the device with the reference's validation and messages. */
int xyzb_dataset_open(const char* path, int32_t device, xyzb_dataset** out, char* err, size_t errlen);
int xyzb_dataset_shape(const xyzb_dataset* ds, uint64_t* n_rows, uint64_t* n_cols, int32_t* binary);

/* ---- the search (three xyz_search overloads, chosen by params->mode) ----
 * draws: optional host-drawn row indices, uint32 [passes][L][M] in pass order
 * (+1 then -1); NULL = the engine draws them itself with the reference's RNG
 * contract (make_stream(seed, offset + rep), draw_subsample). */
int xyzb_search(xyzb_dataset* ds, const xyzb_response* resp, const xyzb_params* params,
                const uint32_t* draws, xyzb_result* out, char* err, size_t errlen);

/* Merge per-shard results (each from xyzb_search with a rep shard) into one
 * report identical to the unsharded search: first-occurrence dedup by
 * (min(j,k), max(j,k), sign), reference order, counters summed, top-K. */
int xyzb_merge_results(xyzb_dataset* ds, const xyzb_result* parts, uint64_t n_parts,
                       const xyzb_params* params, xyzb_result* out, char* err, size_t errlen);

void xyzb_result_free(xyzb_result* res);

/* ---- stage primitives (parity tests of single stages) ---- */

/* Keys of every column under `n_draws` draws of M row indices each:
 * keys[d*p + j] = sum_s bit(X[draws[d*M+s], j]) << s  (binary datasets). */
int xyzb_project_keys(xyzb_dataset* ds, const uint32_t* draws, uint64_t n_draws, uint64_t m,
                      uint64_t* keys, char* err, size_t errlen);

/* Generic equal-key join of two key vectors of length p (pair_search.cpp:26-55).
 * Writes the candidate pairs in reference order (key asc, j asc, k asc) into
 * a library-owned array; total_pairs = sum |x|*|z|. */
int xyzb_equal_pairs(const uint64_t* x_keys, const uint64_t* z_keys, uint64_t p, int32_t device,
                     uint32_t** pairs_jk, uint64_t* n_pairs, uint64_t* total_pairs,
                     char* err, size_t errlen);

/* Strengths of explicit (j,k) pairs under a response, as the reference's
 * pass-+1 strength function of the dataset's mode computes them, bit for bit
 * (same evaluation order, no fused multiply-add): interaction_strength /
 * weighted_interaction_strength (transforms.cpp:33-76) and the continuous-XY
 * strength (search.cpp:273-287, 477-493). The drop-in's sample_strengths
 * (search.cpp:229-291) draws its pairs on the host and evaluates them here. */
int xyzb_pair_strengths(xyzb_dataset* ds, const xyzb_response* resp, const xyzb_params* params,
                        const uint32_t* pairs_jk, uint64_t n_pairs, double* strengths,
                        char* err, size_t errlen);

/* count_agreements(z_j, x_k) of two binary datasets on one device
 * (packed_matrix.cpp:37-47): interaction_strength(x, z, j, k) * n for an
 * arbitrary packed Z (sample_strengths' binary overload, search.cpp:229-242). */
int xyzb_pair_agreements(xyzb_dataset* z, xyzb_dataset* x, const uint32_t* pairs_jk, uint64_t n_pairs,
                         uint64_t* agree, char* err, size_t errlen);

/* One scored pair of the exhaustive search (oracle::ScoredPair, oracle.hpp:15-19). */
typedef struct {
    uint32_t j; /* j < k */
    uint32_t k;
    double strength;
} xyzb_scored_pair;

/* oracle::brute_force_search(PackedMatrix, span<int8>, BruteForceOptions)
 * on the device: the exact strength agree/n of every pair j < k.
 * has_gamma/gamma: keep pairs with strength >= gamma; has_top_k/top_k: keep
 * the top_k strongest (of those >= gamma when both are set; ties broken by
 * (j, k)); histogram_bins > 0: counts of strengths in [0, 1] bins
 * (bin = floor(s * bins), clamped); force: run above the reference's
 * p <= 20000 guard (else XYZB_E_GUARD with its message). Outputs:
 * *pairs (ordered by (j, k), freed by xyzb_free), *n_pairs, *pairs_scanned
 * (= p(p-1)/2), *histogram (histogram_bins entries or NULL, freed by
 * xyzb_free). Binary datasets only. */
int xyzb_brute_force(xyzb_dataset* ds, const int8_t* y_sign, int32_t has_gamma, double gamma, int32_t has_top_k,
                     uint64_t top_k, uint64_t histogram_bins, int32_t force, xyzb_scored_pair** pairs,
                     uint64_t* n_pairs, uint64_t* pairs_scanned, uint64_t** histogram, char* err, size_t errlen);

/* oracle::brute_force_search(PackedMatrix, span<const double>, BruteForceOptions)
 * (oracle.hpp:40-41, oracle.cpp:93-100): the weighted strength of every pair
 * j < k, bit-identical to scalar_weighted_strength (rows in order, fp64). Same
 * options, outputs and errors as xyzb_brute_force; y: n_rows doubles. */
int xyzb_brute_force_weighted(xyzb_dataset* ds, const double* y, int32_t has_gamma, double gamma, int32_t has_top_k,
                              uint64_t top_k, uint64_t histogram_bins, int32_t force, xyzb_scored_pair** pairs,
                              uint64_t* n_pairs, uint64_t* pairs_scanned, uint64_t** histogram, char* err,
                              size_t errlen);

/* ---- xyz-regression helpers (the loop around the screen) ----
 * A device-resident design for lasso_path (lasso.hpp:136-141): X (n x p,
 * column-major fp64, the caller's RealMatrix values) and the column means of
 * the caller's CenteredDesignView (lasso.cpp:40-47), so the exact scans of the
 * active-set loop run on the GPU while coordinate descent stays on the host:
 *   main:  out[j] = sum_i r_i (x_ij - m_j)                  (main_correlation, lasso.cpp:74-80)
 *   pair:  out[t] = sum_i r_i (x_ij - m_j)(x_ik - m_k)      (pair_correlation, lasso.cpp:82-92)
 * fp64 products and sums (summation order differs from the host loop; the
 * results agree to a few ulps of the sum of |terms|). */
typedef struct xyzb_design xyzb_design;
int xyzb_design_create(const double* x, uint64_t n_rows, uint64_t n_cols, const double* means, int32_t device,
                       xyzb_design** out, char* err, size_t errlen);
void xyzb_design_destroy(xyzb_design* d);
int xyzb_design_main_correlations(xyzb_design* d, const double* residual, double* out, char* err, size_t errlen);
/* pairs_jk: 2 * n_pairs column indices (j, k); j == k is a square term. */
int xyzb_design_pair_correlations(xyzb_design* d, const double* residual, const uint32_t* pairs_jk,
                                  uint64_t n_pairs, double* out, char* err, size_t errlen);

void xyzb_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* XYZB_H */
