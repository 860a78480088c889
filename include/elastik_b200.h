/*
 * elastik_b200.h -- C ABI of the B200-native elastic-distance engine
 * (libelastik_b200.so).  Plain pointers and sizes only.
 *
 * It replaces the reference package's native seam and the Python loops above it:
 *
 *   ek_distance_batch  <- elastik._speedups.run (pkg/src/elastik/_speedups.pyx:274-317),
 *                         called per pair by engines._dispatch (pkg/src/elastik/engines.py:29-57)
 *                         behind engines.distance / compute_* (engines.py:60-147)
 *   ek_nn              <- search.nn_search / classify_1nn (pkg/src/elastik/search.py:81-160)
 *   ek_pairwise        <- the all-pairs loop of distance(spec, "pruned_only", X[i], X[j])
 *                         (compute_pruned_only, engines.py:106-118)
 *   ek_subseq          <- search.subsequence_search + series.znormalize
 *                         (pkg/src/elastik/search.py:163-215, series.py:118-131)
 *
 * Conventions
 *   - kind codes follow elastik.kernels.KINDS (kernels.py:22): 0 dtw, 1 cdtw, 2 wdtw,
 *     3 erp, 4 msm, 5 twe; cost_mode 0 squared, 1 absolute (engines.py:20-21).
 *   - variant codes follow engines.VARIANTS (engines.py:18): 0 base, 1 ea, 2 eapruned,
 *     3 pruned_only.
 *   - series are float64, concatenated in one buffer; offsets/lengths are int64.
 *     Inputs are validated by the caller exactly like series.as_series
 *     (non-empty, 1-D, finite; series.py:19-31).
 *   - An abandoned pair or an infeasible window is +inf, never an error
 *     (SPEC.md:552).  Functions return 0 on success, < 0 on error, with the
 *     message in ek_last_error().
 *   - WDTW weights are host-computed (kernels.py:80-92, libm exp): the table for
 *     longest length m (m+1 entries) starts at wdtw_tables[wdtw_table_off[m]]
 *     for every m a call needs (offsets -1 elsewhere), m <= wdtw_max_len.
 *   - All calls are synchronous on the library's stream unless noted (_dev
 *     variants take device pointers and an explicit cudaStream_t as void*).
 */
#ifndef ELASTIK_B200_H
#define ELASTIK_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ek_spec {
  int32_t kind;          /* KINDS index */
  int32_t cost_mode;     /* 0 squared, 1 absolute */
  int64_t window;        /* Sakoe-Chiba half-width, < 0 means None (unbounded) */
  double erp_gap;
  double msm_c;
  double twe_nu;
  double twe_lambda;
  const double* wdtw_tables;     /* host memory, also for _dev calls */
  const int64_t* wdtw_table_off; /* indexed by longest length m */
  int64_t wdtw_max_len;
  int32_t precision;     /* 0 float64 (bit-identical to the reference), 1 float32 (optional
                            faster mode, within 1e-5 relative; ek_distance_batch / ek_nn /
                            ek_pairwise only, cells are the engine's band cells) */
} ek_spec;

/* status / diagnostics */
const char* ek_last_error(void);
int ek_device_count(void);
int ek_init(int device);
const char* ek_version(void);

/* One distance per pair (s_i, t_i) with its own cutoff (engines.distance).
 * windows: per-pair explicit window (engines.compute_ea/eapruned's `window`
 * argument) or NULL to use spec->window.  out_cells: band cells the GPU engine
 * evaluated (schedule-specific). */
int ek_distance_batch(const ek_spec* spec, int32_t variant, int64_t n_pairs, const double* series,
                      int64_t series_len, const int64_t* s_off, const int64_t* s_len, const int64_t* t_off,
                      const int64_t* t_len, const double* cutoffs, const int64_t* windows, double* out_cost,
                      int64_t* out_cells);

/* _speedups.run (pkg/src/elastik/_speedups.pyx:274-317) for many pairs: the native seam
 * engines._dispatch calls (engines.py:29-50), with its exact semantics:
 *   engine 0 base (_base: the full matrix; window and cutoff are ignored, cells = nl*nc),
 *          1 ea (_ea, :129-162), 2 eapruned (_eapruned, :165-271);
 *   lines / cols are taken as given (no re-orientation: make_recurrence already oriented
 *   them, and orient="st" may put the shorter series on the rows);
 *   windows[p] is run's `window` (required for engines 1 and 2, may be NULL for base);
 *   cutoffs[p] is run's `cutoff` (NULL = +inf).
 * (cost, cells) equal run's return value: the reference's own cells_computed for pairs of
 * up to 512 columns x 2048 rows (beyond that, the band cells the GPU evaluated).
 * WDTW: run's `weights` argument is the table for m = max(nl, nc); pass it as
 * spec->wdtw_tables with wdtw_table_off[m] = 0.  ERP: run's border arrays are the
 * sequential prefixes of kernels._erp_border, which the engines rebuild bit-identically. */
int ek_run_batch(const ek_spec* spec, int32_t engine, int64_t n_pairs, const double* series, int64_t series_len,
                 const int64_t* l_off, const int64_t* l_len, const int64_t* c_off, const int64_t* c_len,
                 const int64_t* windows, const double* cutoffs, double* out_cost, int64_t* out_cells);

/* 1-NN of every query against the candidates (nn_search per query, lb="none").
 * nn_idx = -1 when every candidate is +inf.  computed/abandoned/cells per query. */
int ek_nn(const ek_spec* spec, int32_t variant, const double* queries, int64_t q_total, const int64_t* q_off,
          const int64_t* q_len, int64_t n_queries, const double* cands, int64_t c_total, const int64_t* c_off,
          const int64_t* c_len, int64_t n_cands, int64_t* nn_idx, double* nn_dist, int64_t* cells,
          int64_t* computed, int64_t* abandoned);

/* ek_nn as a two-deep pipeline over a stream of batches (nn_search called batch after batch,
 * e.g. a serving loop; search.py:81-125 per query).  ek_nn_submit enqueues one batch's
 * upload, search and result read-back into pipeline slot 0 or 1 and returns without
 * waiting; ek_nn_collect waits for that slot's results (same outputs and errors as ek_nn).
 * Each slot keeps its own device copy of the batch, so batch k+1's upload crosses PCIe while
 * batch k is searched.  The host arrays must stay valid until the slot is collected (and
 * should be page-locked for the upload to be asynchronous).  A slot takes one batch at a
 * time: submitting to a slot that was not collected is an error. */
int ek_nn_submit(const ek_spec* spec, int32_t variant, const double* queries, int64_t q_total, const int64_t* q_off,
                 const int64_t* q_len, int64_t n_queries, const double* cands, int64_t c_total, const int64_t* c_off,
                 const int64_t* c_len, int64_t n_cands, int32_t slot);
int ek_nn_collect(int32_t slot, int64_t* nn_idx, double* nn_dist, int64_t* cells, int64_t* computed,
                  int64_t* abandoned);

/* Same with device-resident inputs/outputs (lengths as int32, offsets int64) on `stream`.
 * dense != 0 promises every series has length max_len (enables the LB_Keogh pre-filter
 * for dtw/cdtw, which drops only candidates whose bound proves a +inf result). */
int ek_nn_dev(const ek_spec* spec, int32_t variant, const double* d_queries, const int64_t* d_q_off,
              const int32_t* d_q_len, int64_t n_queries, const double* d_cands, const int64_t* d_c_off,
              const int32_t* d_c_len, int64_t n_cands, int32_t max_len, int32_t dense, int64_t* d_nn_idx,
              double* d_nn_dist, int64_t* d_cells, int64_t* d_computed, int64_t* d_abandoned, void* stream);

/* Full symmetric matrix D[n*n] of distance(spec, variant, X_i, X_j); diagonal 0.0.
 * cells: total band cells evaluated. */
int ek_pairwise(const ek_spec* spec, int32_t variant, const double* series, int64_t total, const int64_t* off,
                const int64_t* len, int64_t n, double* D, int64_t* cells);

/* Pairs [pair_lo, pair_hi) of the upper triangle in row-major order (the order of
 * numpy.triu_indices(n, 1)): out[p - pair_lo] = distance(spec, variant, X_i, X_j) for pair
 * p = (i, j).  The unit of the multi-GPU all-pairs shard: a rank passes its
 * contiguous pair range, the device maps indices to (i, j), no per-pair host arrays. */
int ek_pairwise_range(const ek_spec* spec, int32_t variant, const double* series, int64_t total, const int64_t* off,
                      const int64_t* len, int64_t n, int64_t pair_lo, int64_t pair_hi, double* out, int64_t* cells);

/* ek_pairwise on device arrays; dense != 0 promises every length equals max_len (the
 * |i-j| tables of WDTW / TWE are then shared per block). */
int ek_pairwise_dev(const ek_spec* spec, int32_t variant, const double* d_series, const int64_t* d_off,
                    const int32_t* d_len, int64_t n, int32_t max_len, int32_t dense, double* d_D, int64_t* cells,
                    void* stream);

/* Best window of `reference` against `query` (dtw/cdtw), every stride-1 offset,
 * z-normalising the query once and each window on the fly when normalize != 0.
 * Ties keep the lowest offset; best_off = -1 when every window is +inf. */
int ek_subseq(const ek_spec* spec, int32_t variant, const double* query, int64_t lq, const double* reference,
              int64_t n_ref, int32_t normalize, int64_t* best_off, double* best_dist, int64_t* cells,
              int64_t* computed, int64_t* abandoned);

int ek_subseq_dev(const ek_spec* spec, int32_t variant, const double* d_query, int64_t lq,
                  const double* d_reference, int64_t n_ref, int32_t normalize, int64_t* best_off,
                  double* best_dist, int64_t* cells, int64_t* computed, int64_t* abandoned, void* stream);

/* Distance profile: window_dist[o] = distance(spec, "base", query, window_o) for every
 * stride-1 offset o (n_ref - lq + 1 values), each window z-normalised when normalize != 0.
 * The per-offset loop of subsequence_search (search.py:189-213) without the running
 * cutoff; the reference obtains the same numbers by calling engines.distance per window. */
int ek_subseq_profile(const ek_spec* spec, const double* query, int64_t lq, const double* reference, int64_t n_ref,
                      int32_t normalize, double* window_dist);

/* Batched build_envelope (lower_bounds.py:23-57): for n series of equal length L
 * (series[off[s] .. off[s] + L)), upper / lower[s * L + i] = max / min of the series
 * over [i - window, i + window] (clipped), bit-identical to the reference's deque.
 * The GPU 1-NN path builds the same envelopes internally (rounded outward to floats). */
int ek_envelopes(const double* series, int64_t total, const int64_t* off, int64_t n, int64_t L, int64_t window,
                 double* upper, double* lower);

/* ---- Ingestion ----
 * ek_parse_tsv <- series.load_tsv (pkg/src/elastik/series.py:61-86), native fast path.
 * UCR text (one series per line, the numeric label first, truncated to int; fields split by
 * `sep`; \n, \r\n or \r line ends; blank lines skipped) into the packed layout every entry
 * point takes: values[offsets[s] .. + lengths[s]], labels[s].  Call with values == NULL to
 * count (n_series, n_values), then again with buffers of those sizes.  Returns 0, or 1 when
 * the fast path does not decide the file (any token outside the plain decimal grammar,
 * non-finite or overflowing values, a line without a value, non-ASCII text, an empty
 * dataset; *bad_line = its line): the caller then runs the reference's loader, which
 * accepts or raises exactly as series.load_tsv does.  Host only (no device needed). */
int ek_parse_tsv(const char* text, int64_t len, int32_t sep, int64_t* n_series, int64_t* n_values,
                 int64_t* labels, int64_t* offsets, int64_t* lengths, double* values, int64_t* bad_line);
/* Page-locked host buffers (cudaHostAlloc, portable) and device buffers; NULL on failure. */
void* ek_host_alloc(int64_t bytes);
int ek_host_free(void* p);
void* ek_dev_alloc(int64_t bytes);
int ek_dev_free(void* p);
/* dir 0: host -> device, 1: device -> host, 2: device -> device.  stream NULL: the library's
 * stream, synchronised before returning; else enqueued on `stream`. */
int ek_memcpy(void* dst, const void* src, int64_t bytes, int32_t dir, void* stream);
/* series.derivative (series.py:134-144) of n device series: d_out[d_out_off[s] + i] =
 * ((x[i+1] - x[i]) + (x[i+2] - x[i]) / 2) / 2 for i < d_len[s] - 2 (lengths >= 3 are the
 * caller's check, DegenerateInputError in the Python API). */
int ek_derivative_dev(const double* d_in, const int64_t* d_off, const int32_t* d_len, int64_t n, double* d_out,
                      const int64_t* d_out_off, void* stream);
/* series.znormalize (series.py:118-131) of n device series with numpy's pairwise-sum mean
 * and std (std < 1e-12 -> zeros); h_len: the lengths on the host (each >= 2). */
int ek_znormalize_dev(const double* d_in, const int64_t* d_off, const int32_t* d_len, const int32_t* h_len,
                      int64_t n, double* d_out, const int64_t* d_out_off, void* stream);

/* Number of kernel launches the library issued since the last reset (bench accounting). */
int64_t ek_launch_count(int32_t reset);

/* Measurement helpers (bench.py): record CUDA events between the phases of the
 * next ek_nn / ek_pairwise / ek_subseq call (host or _dev); read back per-phase device times.
 * on = 1: every phase; on = 2: only the marks that bracket the DP kernels of a 1-NN call
 * (fewer events inside a timed step); 0: none. */
void ek_set_profiling(int32_t on);
int32_t ek_phase_times(double* ms, const char** names, int32_t max);

/* Measured FP64 (non-tensor) DADD/DMUL throughput of the device, ops/s. */
double ek_fp64_peak_ops(void);
/* Measured FP32 (non-tensor) FADD/FMUL throughput (roofline of the FP32 mode), ops/s. */
double ek_fp32_peak_ops(void);

#ifdef __cplusplus
}
#endif
#endif /* ELASTIK_B200_H */
