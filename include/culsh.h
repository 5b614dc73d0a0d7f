/*
 * culsh.h -- C ABI of the B200-native CULSH-MF hot path (libculsh.so).
 *
 * Drop-in boundary: each entry point replaces one kernel seam of the reference
 * package lshmf (/root/reference/pkg/src/lshmf), cited per function as
 * file:line.  The reference's Python layer (lsh.py, factorization.py,
 * online.py, parallel.py) calls those numba kernels with plain numpy arrays;
 * the Python host layer paper_2111_11682_b200/ calls these functions with
 * plain device pointers obtained from torch tensors, through ctypes
 * (INTEGRATION.md shows the binding).
 *
 * Conventions
 *   - every pointer argument is a DEVICE pointer unless the name ends in _host;
 *   - `stream` is a cudaStream_t passed as void*; all work is enqueued on it;
 *   - return value: CULSH_OK (0), CULSH_DIVERGED (1, non-finite error seen,
 *     the reference's "return 1"), CULSH_EINVAL (-1, bad arguments; nothing
 *     launched), CULSH_ECUDA (-2, CUDA error); culsh_last_error() describes it;
 *   - the library never frees caller memory and never throws across the ABI;
 *   - no torch types appear here.
 */
#ifndef CULSH_H_
#define CULSH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CULSH_OK 0
#define CULSH_DIVERGED 1
#define CULSH_EINVAL (-1)
#define CULSH_ECUDA (-2)

/* ---------------------------------------------------------------- misc --- */

/* Last error message (thread-local), "" if none. */
const char *culsh_last_error(void);
/* Library version string, e.g. "culsh 0.1.0 sm_100a". */
const char *culsh_version(void);

/* ------------------------------------------------------------- simLSH --- */

/* Row-hash table: for rows [row_lo,row_hi) writes table[i][g][m][s], the byte s
 * (s < ceil(G/8)) of the low G bits of splitmix64(map_key(seed,g,m) ^ i).
 * Replaces lsh.py:68-78 _assign_bits / lsh.py:108-114 assign_row_hashes (the
 * reference's (M,q,p,G) u8 tensor, packed 8 bits per byte). */
int culsh_row_hash_table(uint64_t seed, int q, int p, int G, int64_t row_lo, int64_t row_hi,
                         uint8_t *table, void *stream);

/* Pack/unpack between the reference's (M,q,p,G) u8 bit tensor (RowHashes.bits,
 * lsh.py:81-105) and the packed table. */
int culsh_pack_bits(const uint8_t *bits, int64_t M, int q, int p, int G, uint8_t *table,
                    void *stream);
int culsh_unpack_bits(const uint8_t *table, int64_t M, int q, int p, int G, uint8_t *bits,
                      void *stream);

/* Sets *bad_out (device int) to 1 unless every psi(v) of the listed columns is an
 * integer and every column's sum of |psi| is < 2^31 (enables the exact-integer
 * accumulation path, bit-identical to the reference's fp64 sums). */
int culsh_psi_int_check(const int64_t *col_ptr, const double *col_vals, int64_t col_begin,
                        int64_t n_cols, const int32_t *col_list, int e, int *bad_out, void *stream);

/* Signed accumulation + threshold + group-key pack for columns
 * col_list[0..n_cols) (or col_begin + [0..n_cols) when col_list is NULL).
 *   acc  (N, q, p, G) f64   fresh (into=0) or added to in place (into=1)
 *   sig  (N, q, p, G) u8    optional (NULL to skip)
 *   keys (q, keys_ld) u64   optional, bit m*G+t of keys[g, j] = sig[j,g,m,t]
 * Replaces lsh.py:161-179 _accumulate_all, online.py:96-117 _accumulate_into,
 * lsh.py:182-183 _threshold and lsh.py:246-260 _pack_group_keys. */
int culsh_hash_accumulate(const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals,
                          int64_t col_begin, int64_t n_cols, const int32_t *col_list,
                          const uint8_t *table, int q, int p, int G, int e, int into, int int_path,
                          double *acc, uint8_t *sig, uint64_t *keys, int64_t keys_ld, void *stream);

/* Exact-integer bit-counting path for few-valued ratings (e.g. 1..5 stars).
 * culsh_value_set: per-block sets of distinct values of vals (out n_blocks x 17
 *   doubles: [count or -1 on overflow, v0..v15]); the caller merges them.
 * culsh_class_partition: per column, the row indices grouped by value class
 *   (class c = index of the value in class_vals[0..NC)); class_off (N, NC+1)
 *   offsets relative to col_ptr[j].
 * culsh_hash_count: acc/sig/keys for columns [col_begin, col_begin+n_cols) from
 *   Harley-Seal bit counts: acc = sum_c class_psi[c] * (2*count - n_c), exact, so
 *   bit-identical to lsh.py:161-183 whenever culsh_psi_int_check passes.
 *   The table must hold M+1 rows, row M all zeros (padding).  max_slice_mb > 0
 *   splits the work into row-range passes whose table slice stays L2-resident;
 *   acc carries the exact partial sums between passes (class segments are
 *   row-sorted).  variant 0: row records staged by the bulk-copy engine
 *   (cp.async.bulk + mbarrier); 1: register double-buffered loads.
 *   Needs q*p*ceil(G/8) % 4 == 0 and <= 512. */
int culsh_value_set(const double *vals, int64_t n, double *out, int n_blocks, void *stream);
int culsh_class_partition(const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals,
                          int64_t N, const double *class_vals, int NC, int32_t *rows_by_class,
                          int32_t *class_off, void *stream);
int culsh_hash_count(const int64_t *col_ptr, const int32_t *rows_by_class, const int32_t *class_off,
                     int NC, const int *class_psi, int64_t M, int max_slice_mb, int variant,
                     int64_t col_begin, int64_t n_cols,
                     const uint8_t *table, int q, int p, int G, double *acc, uint8_t *sig,
                     uint64_t *keys, int64_t keys_ld, void *stream);

/* Buckets + frequency top-K with seeded supplement for target columns
 * [j_base, j_base+n_cols) of an N_total-column key matrix keys (q, N_total).
 * entries (n_cols, K) i32.  *n_candidates_out (host) = total bucket-mate count.
 * Replaces lsh.py:401-414 _topk_from_group_keys (B2-B4: lsh.py:263-287,308-374)
 * and the new-column path of online.py:152-184 topk_for_new. */
int culsh_topk(const uint64_t *keys, int q, int64_t N_total, int key_bits, int64_t j_base,
               int64_t n_cols, int K, uint64_t seed, int32_t *entries,
               int64_t *n_candidates_out_host, void *stream);

/* Stage APIs of the same pipeline (lsh.py:290-305 coarse_candidates, 377-398 fine_topk):
 * culsh_pack_keys: keys (q, N) from a signature tensor sig (N, q, p, G) u8.
 * culsh_candidates: per target column the bucket mates over all q groups, each
 *   column's list sorted ascending.  Call with cand == NULL to get offsets
 *   (n_cols+1, device int64) and *n_candidates_out; then with a buffer of that size.
 * culsh_select_topk: frequency top-K + seeded supplement from caller-supplied
 *   candidate lists (cand, offsets; unsorted is fine). */
int culsh_pack_keys(const uint8_t *sig, int64_t N, int q, int p, int G, uint64_t *keys, void *stream);
int culsh_candidates(const uint64_t *keys, int q, int64_t N_total, int key_bits, int64_t j_base,
                     int64_t n_cols, int64_t *offsets, int32_t *cand, int64_t cand_capacity,
                     int64_t *n_candidates_out_host, void *stream);
int culsh_select_topk(const int32_t *cand, const int64_t *offsets, int64_t total, int64_t j_base,
                      int64_t n_cols, int K, uint64_t seed, int64_t N_total, int32_t *entries,
                      void *stream);

/* ---------------------------------------------------------------- SGD --- */

/* Learning rates and regularisers of one epoch (factorization.py:84-95). */
typedef struct {
    double gb, gbh, gu, gv, gw, gc;
    double lb, lbh, lu, lv, lw, lc;
} CulshRates;

/* Device view of SparseRatings (data.py:166-207) + residual baselines
 * (data.py:289-309).  csc2csr[idx] = CSR position of CSC entry idx. */
typedef struct {
    int64_t M, N, nnz;
    const int64_t *col_ptr;
    const int32_t *col_rows;
    const double *col_vals;
    const int64_t *row_ptr;
    const int32_t *row_cols;
    const double *row_vals;
    const int32_t *csc2csr;
    const double *base_b;
    const double *base_bhat;
} CulshData;

/* fp64 model (factorization.py:105-137 ModelParams), row-major arrays. */
typedef struct {
    double mu;
    double *b, *bhat, *U, *V, *W, *C;
    const int32_t *nbr;
    int F, K;
} CulshModel64;

/* CSC-entry ranges of one pass: seg[2j], seg[2j+1]; chain_lo[j] = first column
 * of the block j belongs to.  mode 0: rows [row_lo,row_hi) of columns
 * [col_lo,col_hi) (factorization.py:346-355); mode 1: DSGD stage s of D using
 * block_ptr (N, D+1) and col_bounds (D+1) (parallel.py:36-41,110-128). */
int culsh_pass_plan(const int64_t *col_ptr, const int32_t *col_rows, int64_t N, int mode,
                    int64_t col_lo, int64_t col_hi, int64_t row_lo, int64_t row_hi,
                    const int64_t *block_ptr, const int64_t *col_bounds, int D, int s,
                    int64_t *seg, int32_t *chain_lo, void *stream);

/* parallel.py:55-64 _block_pointers: out (N, nb). */
int culsh_block_pointers(const int64_t *col_ptr, const int32_t *col_rows, int64_t N,
                         const int64_t *row_bounds, int nb, int64_t *out, void *stream);

/* Deterministic serial-order column pass (bit-exact fp64).  row_mode: 0 never
 * update rows, 1 always, 2 only rows >= M_old.  row_last (M ints), ticket (1 int)
 * are scratch; *status (device int) is OR-ed with 1 on a non-finite error.
 * Replaces factorization.py:332-363 _full_pass_block, parallel.py:110-128
 * _stage_pass (all D blocks of a stage in one launch) and online.py:253-271
 * _online_col_pass.  variant 0: the full model; variant 3: the row-major basic-MF
 * pass (factorization.py:366-391 _basic_pass, K = 0) run on the TRANSPOSED data
 * (CulshData with rows and columns swapped, csc2csr = the CSR->CSC map). */
int culsh_sgd_exact_colpass(const CulshData *d, CulshModel64 *m, const CulshRates *r,
                            const int64_t *seg, const int32_t *chain_lo, int64_t col_lo,
                            int64_t col_hi, int row_mode, int64_t M_old, int variant,
                            int *row_last, int *ticket, int *status, void *stream);

/* Neighbour lookups (factorization.py:218-232) of every CSC entry of columns
 * [col_lo, col_hi), ahead of a column pass: mask (entries x (K<=32 ? 1 : K<=64 ? 2 : 4) u32, bit k
 * set iff row i rated J[j,k]) and rv (entries x K f64, the ratings found), entry
 * index relative to col_ptr[col_lo]. */
int culsh_exact_lookup(const CulshData *d, const CulshModel64 *m, int64_t col_lo, int64_t col_hi,
                       uint32_t *mask, double *rv, void *stream);

/* culsh_sgd_exact_colpass reading the lookups from culsh_exact_lookup (pre_base =
 * col_ptr[col_lo] of that call) instead of searching inside the dependent update
 * chain -- the same values, bit-identical result. */
int culsh_sgd_exact_colpass_pre(const CulshData *d, CulshModel64 *m, const CulshRates *r,
                                const int64_t *seg, const int32_t *chain_lo, int64_t col_lo,
                                int64_t col_hi, int row_mode, int64_t M_old, int variant,
                                int *row_last, int *ticket, int *status, const uint32_t *pre_mask,
                                const double *pre_rv, int64_t pre_base, void *stream);

/* online.py:230-250 _online_row_pass (rows [row_lo,row_hi), columns < N_old). */
int culsh_sgd_exact_rowpass(const CulshData *d, CulshModel64 *m, const CulshRates *r,
                            int64_t row_lo, int64_t row_hi, int64_t N_old, int *status,
                            void *stream);

/* fp32 model for the Hogwild performance mode. */
typedef struct {
    float mu;
    float *b, *bhat, *U, *V, *W, *C;
    int F, K;
} CulshModel32;

/* Per-rating explicit-neighbour stream for the Hogwild kernel, built once per
 * fit from (data, J^K) only (factorization.py:287-298 split into the data part):
 *   mask[idx] bit k set iff row i rated neighbour J[j,k]   (u32 words, K<=32 -> 1 word)
 *   resid[resid_ptr[j] + ...] = r(i,J[j,k]) - (mu + b_i + b_hat_J[j,k]) for set bits,
 *   in (entry, k) order.  Pass 1 (resid == NULL) fills mask and per-column counts
 *   col_nexpl (N); the caller prefix-sums counts into resid_ptr (N+1); pass 2 fills resid. */
int culsh_explicit_stream(const CulshData *d, double mu, const int32_t *nbr, int K,
                          uint32_t *mask, int64_t *col_nexpl, const int64_t *resid_ptr,
                          float *resid, void *stream);

/* One Hogwild epoch (warp per column, column parameters in registers, row
 * parameters lock-free; paper Alg. 3, factorization.py:266-329 rules in fp32).
 * Processes N_list columns col_order[0..N_list) (NULL = 0..N_list-1); column j
 * streams CSC entries [seg[2j], seg[2j+1]) (seg NULL = the whole column, a DSGD
 * block otherwise, see culsh_pass_plan).  rows/vals: CSC row index and fp32
 * value.  flags bit 0: start each column at a per-column hashed offset (warps
 * sweep rows out of phase: fewer concurrent writes to one u_i); bit 1: apply
 * row updates as vector atomic adds of the delta (no lost updates); bit 2: the
 * reserved (must be 0); bit 3: seg is
 * indexed by ticket (work segments: list entry t = column col_order[t], entries
 * [seg[2t], seg[2t+1] & (2^40-1)), S = seg[2t+1] >> 40 segments in that column; a
 * segment of a split column (S > 1) runs concurrently with the column's other
 * segments and atomically adds 1/S of its v/w/c/b_hat change); max_warps > 0
 * caps the number of concurrently active column warps (Hogwild staleness on
 * small matrices), 0 = every resident warp.  loss_out
 * (device double, optional) accumulates sum e^2; *status |= 1 on a non-finite
 * error.  Replaces factorization.py:332-363 _full_pass_block /
 * parallel.py:110-128 _stage_pass in the performance mode. */
int culsh_sgd_hogwild_epoch(int64_t N_list, const int64_t *col_ptr, const int64_t *seg,
                            const int32_t *rows, const float *vals, const uint32_t *mask,
                            const int64_t *resid_ptr, const float *resid, const int32_t *col_order,
                            CulshModel32 *m, const CulshRates *r, int flags, int max_warps,
                            int *ticket,
                            double *loss_out, int *status, void *stream);

/* Packed per-epoch rating stream for the Hogwild kernel (the form e2e ships over
 * PCIe every epoch): packed[idx] = row (bits 0-26) | value code into lut (bits
 * 27-30) | has-explicit-neighbour (bit 31); cmask holds the MW mask words of the
 * ratings with bit 31 set only, column j's from mptr[j].  Pass 1 (packed ==
 * NULL): mcount[j] = number of such ratings in column j; the caller prefix-sums
 * it into mptr (N+1).  Pass 2 fills packed and cmask.  *status |= 4 if a value is
 * not in lut (1..16 fp32 values) or a row index needs more than 27 bits.  Same
 * information as the (rows, vals, mask) triple of culsh_sgd_hogwild_epoch. */
int culsh_pack_stream(int64_t N, const int64_t *col_ptr, const int32_t *rows, const float *vals,
                      const uint32_t *mask, int MW, const float *lut, int n_lut, uint32_t *packed,
                      int64_t *mcount, const int64_t *mptr, uint32_t *cmask, int *status, void *stream);

/* culsh_sgd_hogwild_epoch over the packed stream (warp per column or per work
 * segment; flags bits 0, 1, 3 as there -- seg must be NULL or a per-ticket work
 * segment list).  Identical updates to the wide-stream kernel on the same data. */
int culsh_sgd_hogwild_epoch_packed(int64_t N_list, const int64_t *col_ptr, const int64_t *seg,
                                   const uint32_t *packed,
                                   const float *lut, const int64_t *mptr, const uint32_t *cmask,
                                   const int64_t *resid_ptr, const float *resid, const int32_t *col_order,
                                   CulshModel32 *m, const CulshRates *r, int flags, int max_warps,
                                   int *ticket, double *loss_out, int *status, void *stream);

/* Stream cursors at the start of every work segment (once per work list): seg4[4t..4t+3] =
 * {lo, hi | S << 40 (copied from seg2), compact-mask slot at lo (packed stream: mptr[j] +
 * flagged entries of column j before lo), residual offset at lo | (2-byte records: row of
 * the entry before lo) << 32}.  words / w16 / first_row / mptr describe the packed stream
 * (mptr NULL: wide stream, mask = one MW-word mask per entry).  The epoch kernels take seg4
 * with flags bit 4 (| bit 3) and skip the per-segment scan from the column start. */
int culsh_segment_cursors(int64_t n_list, const int64_t *col_ptr, const int32_t *col_order,
                          const int64_t *seg2, const uint32_t *words, const uint16_t *w16,
                          const int32_t *first_row, const int64_t *mptr, const uint32_t *mask, int MW,
                          int64_t *seg4, void *stream);

/* 2-byte per-rating stream (rows without rotation): words[idx] = row delta from the
 * previous entry of the column (12 bits; 0 for the first) | value code (3 bits) |
 * has-explicit-neighbour (1 bit); first_row[j] = row of column j's first entry.
 * *status |= 4 if a delta or the value table does not fit (use culsh_pack_stream). */
int culsh_pack16(int64_t N, const int64_t *col_ptr, const int32_t *rows, const float *vals,
                 const uint32_t *mask, int MW, const float *lut, int n_lut, uint16_t *words,
                 int32_t *first_row, int *status, void *stream);

/* culsh_sgd_hogwild_epoch_packed over the 2-byte stream (rows rebuilt by a warp prefix
 * sum; cmask / mptr as for the 4-byte stream; no rotation).  Identical updates. */
int culsh_sgd_hogwild_epoch_packed16(int64_t N_list, const int64_t *col_ptr, const int64_t *seg,
                                     const uint16_t *packed, const int32_t *first_row, const float *lut,
                                     const int64_t *mptr, const uint32_t *cmask, const int64_t *resid_ptr,
                                     const float *resid, const int32_t *col_order, CulshModel32 *m,
                                     const CulshRates *r, int flags, int max_warps, int *ticket,
                                     double *loss_out, int *status, void *stream);

/* --------------------------------------------------------------- eval --- */

/* Per-test-triplet squared error (fp64, exact _predict_one order) and the RMSE.
 * Replaces factorization.py:394-409 _rmse_kernel (sum by a fixed pairwise tree).
 * rmse_out: device double. */
int culsh_rmse(const CulshData *d, const CulshModel64 *m, const int32_t *t_rows,
               const int32_t *t_cols, const double *t_vals, int64_t n, int do_clamp,
               double clamp_lo, double clamp_hi, double unscale, double *sqerr_scratch,
               double *rmse_out, void *stream);

/* culsh_rmse / culsh_rmse_train on an fp32 model (a Hogwild fit) without widening it:
 * fp32 values loaded, arithmetic in fp64 in the reference's order -- the same bytes as on
 * the widened fp64 copy.  mu: the model's fp64 mu; F: logical factors (m->F is the row
 * stride, >= F for zero-padded widths); nbr: J^K. */
int culsh_rmse_m32(const CulshData *d, const CulshModel32 *m, double mu, int F, const int32_t *nbr,
                   const int32_t *t_rows, const int32_t *t_cols, const double *t_vals, int64_t n,
                   int do_clamp, double clamp_lo, double clamp_hi, double unscale, double *sqerr_scratch,
                   double *rmse_out, void *stream);
int culsh_rmse_train_m32(const CulshData *d, const CulshModel32 *m, double mu, int F, const int32_t *nbr,
                         const uint32_t *mask, const int64_t *group_base, const int32_t *pos,
                         const int64_t *perm, int do_clamp, double clamp_lo, double clamp_hi,
                         double unscale, double *sqerr_scratch, double *rmse_out, void *stream);

/* RMSE of the fp32 Hogwild model (predictions in fp32, sum in fp64). */
int culsh_rmse32(const CulshData *d, const CulshModel32 *m, const int32_t *nbr,
                 const int32_t *t_rows, const int32_t *t_cols, const double *t_vals, int64_t n,
                 double *sqerr_scratch, double *rmse_out, void *stream);

/* Lookup cache of the training set for culsh_rmse_train: the explicit-neighbour mask of
 * every CSC entry (culsh_explicit_stream) is turned into the CSC position of each
 * explicit pair r(i, J[j, k]).  Call with group_count != NULL to get the number of pairs
 * per 32-entry group, then (after an exclusive scan into group_base) with
 * group_count == NULL to fill pos (int32, CSC order). */
int culsh_train_lookup(const CulshData *d, const int32_t *nbr, int K, const uint32_t *mask,
                       int64_t *group_count, const int64_t *group_base, int32_t *pos, void *stream);

/* factorization.py:559-579 rmse over the TRAINING set itself (cli.py:204-210 calls it
 * every epoch): the CSC entries of d, neighbour values from the lookup cache, the squared
 * error of CSC position c stored at entry index perm[c] (NULL: identity) so the sum runs
 * in the reference's entry order (the exact serial sum at any nnz, culsh_sequential_sum). */
int culsh_rmse_train(const CulshData *d, const CulshModel64 *m, const uint32_t *mask,
                     const int64_t *group_base, const int32_t *pos, const int64_t *perm, int do_clamp,
                     double clamp_lo, double clamp_hi, double unscale, double *sqerr_scratch,
                     double *rmse_out, void *stream);

/* factorization.py:559-579 rmse over the TRAINING set in CSR order, for N <= 65536: one
 * warp per row (U[i] broadcast, the lanes' V rows staged; a per-warp shared bitmap of the
 * row's columns answers "rated J[j, k]?", rated ones binary-search the row for the value).
 * No lookup cache.  csr_entry[p] = entry index of CSR position p (NULL: identity); the
 * squared errors are the same bytes as culsh_rmse_train's and are summed in entry order.
 * The _m32 form reads a Hogwild fit's fp32 arrays (arguments as culsh_rmse_train_m32). */
int culsh_rmse_train_rows(const CulshData *d, const CulshModel64 *m, const int32_t *csr_entry,
                          int do_clamp, double clamp_lo, double clamp_hi, double unscale,
                          double *sqerr_scratch, double *rmse_out, void *stream);
int culsh_rmse_train_rows_m32(const CulshData *d, const CulshModel32 *m, double mu, int F,
                              const int32_t *nbr, const int32_t *csr_entry, int do_clamp,
                              double clamp_lo, double clamp_hi, double unscale,
                              double *sqerr_scratch, double *rmse_out, void *stream);

/* culsh_rmse over any test set grouped by row (same kernel as culsh_rmse_train_rows,
 * N <= 65536): row i's targets are [t_ptr[i], t_ptr[i+1]) (t_ptr: M+1 int64) with columns
 * t_cols, values t_vals and t_index = each target's position in the test set (the sum runs
 * in test-set order; NULL: identity).  n = number of targets.  Same squared errors as
 * culsh_rmse on the ungrouped triplets. */
int culsh_rmse_rows(const CulshData *d, const CulshModel64 *m, const int64_t *t_ptr, const int32_t *t_cols,
                    const double *t_vals, const int32_t *t_index, int64_t n, int do_clamp, double clamp_lo,
                    double clamp_hi, double unscale, double *sqerr_scratch, double *rmse_out, void *stream);
int culsh_rmse_rows_m32(const CulshData *d, const CulshModel32 *m, double mu, int F, const int32_t *nbr,
                        const int64_t *t_ptr, const int32_t *t_cols, const double *t_vals,
                        const int32_t *t_index, int64_t n, int do_clamp, double clamp_lo, double clamp_hi,
                        double unscale, double *sqerr_scratch, double *rmse_out, void *stream);

/* The reference's serial fp64 sum (factorization.py:394-409 `total += d * d`) of n >= 1
 * terms: out = fl(...fl(fl(0 + x[0]) + x[1]) ... + x[n-1]), bit for bit, in parallel for
 * non-negative terms (a run of additions inside one binade is an integer sum on that
 * binade's ulp grid plus a ties-to-even parity bit; chunks that change binade or hold any
 * other term are added one by one).  Every culsh_rmse* entry point sums this way. */
int culsh_sequential_sum(const double *x, int64_t n, double *out, void *stream);

/* factorization.py:235-263 _predict_one for n (i, j) pairs -> out (n) f64. */
int culsh_predict(const CulshData *d, const CulshModel64 *m, const int32_t *rows,
                  const int32_t *cols, int64_t n, double *out, void *stream);

/* ----------------------------------------------------------- ratings --- */

/* csc2csr[idx] for every CSC entry (binary search of column j in row i). */
int culsh_csc_to_csr_map(const CulshData *d, int32_t *csc2csr, void *stream);

/* Online append (replaces the full rebuild of online.py:84-93 extend_ratings):
 * out segment s = old segment s (s < n_old) followed by add segment s, for
 * s < n_total; out_ptr (n_total+1).  Applied to the CSC (segments = columns, the
 * increment's rows sort after the old ones) and to the CSR (segments = rows). */
int culsh_append_segments(int64_t n_old, int64_t n_total, const int64_t *old_ptr, const int32_t *old_idx,
                          const double *old_val, const int64_t *add_ptr, const int32_t *add_idx,
                          const double *add_val, int64_t *out_ptr, int32_t *out_idx, double *out_val,
                          void *stream);

/* csc2csr of the merged views after the two appends above, without a full
 * rebuild: kept entries shift by add_row_ptr[i], added entries are searched.
 * d describes the merged ratings; old_col_ptr/old_map the pre-append CSC. */
int culsh_append_csc2csr(const CulshData *d, int64_t n_old_cols, const int64_t *old_col_ptr,
                         const int32_t *old_map, const int64_t *add_row_ptr, int64_t M_old,
                         int32_t *csc2csr, void *stream);

/* out[s] = sum of val[ptr[s]..ptr[s+1]) for s < n (baseline sums, data.py:289-309;
 * exact, hence order-independent, for integer-valued ratings). */
int culsh_segment_sums(int64_t n, const int64_t *ptr, const double *val, double *out, void *stream);

/* compute_baselines (data.py:289-309) in the reference's summation order for ANY values.
 * pairwise_chunks: out[c] = numpy's pairwise sum (np.add.reduce, 8-accumulator leaves of
 * <= 128, halving splits rounded down to multiples of 8) of x[off[c] .. off[c] + len[c]),
 * each chunk a node of the whole array's split tree with len <= 65,536 (the caller splits
 * the top of the tree the same way and combines the chunk sums).
 * ordered_segment_sums: out[s] = (init ? init[s] : 0.0) + val[order[ptr[s]]] + ... one by one
 * in order (np.add.at's sequential accumulation with entries grouped stably by row or
 * column; order NULL = identity). */
int culsh_pairwise_chunks(const double *x, const int64_t *off, const int64_t *len, int64_t nchunks,
                          double *out, void *stream);
int culsh_ordered_segment_sums(int64_t n, const int64_t *ptr, const int64_t *order, const double *val,
                               const double *init, double *out, void *stream);

/* ------------------------------------------------- DSGD peer ring --- */

/* Ring shift of the moving DSGD block over peer memory (parallel.py:166-227's block hand-
 * over between workers; dsgd.PeerRing).  ring_alloc: this rank's buffer (64 u64 flags +
 * two data slots of slot_bytes) via cudaMalloc, with its CUDA IPC handle (handle_bytes()
 * bytes) for the neighbours; ring_open / ring_close map / unmap a neighbour's buffer.
 * ring_push (after stage s): once the receiver acknowledged slot seq & 1's previous use
 * (seq - 2), copy the n block pieces (ptrs / bytes, at 16-byte-aligned slot offsets offs)
 * into the receiver's slot and release receiver.ready[seq & 1] = seq (system scope).
 * ring_pull: wait on the device for my.ready[seq & 1] >= seq, copy the slot's pieces into
 * ptrs, release sender.ack[seq & 1] = seq.  Stream-ordered, no host synchronisation; a
 * flag wait longer than 20 s sets *status |= 4. */
int culsh_ring_alloc(int64_t slot_bytes, void **buf, void *ipc_handle_out);
int culsh_ring_open(const void *ipc_handle, void **buf);
int culsh_ring_close(void *peer_buf);
int culsh_ring_free(void *buf);
int culsh_ring_handle_bytes(void);
int culsh_ring_push(int n, void *const *ptrs, const int64_t *bytes, const int64_t *offs, void *my_buf,
                    void *peer_buf, int64_t slot_bytes, uint64_t seq, int *status, void *stream);
int culsh_ring_pull(int n, void *const *ptrs, const int64_t *bytes, const int64_t *offs, void *my_buf,
                    void *sender_buf, int64_t slot_bytes, uint64_t seq, int *status, void *stream);

/* ------------------------------------------------------- similarity --- */

/* Exact GSM top-K by the merge route (similarity.py:164-185 _gsm_topk_kernel):
 * target columns j_lo..j_lo+n_rows-1, all N candidates each, statistics by an
 * ascending-row merge in fp64 (similarity.py:57-90), shrunk Pearson with the
 * reference's expression order, ties to the lower index.  entries: (n_rows, K).
 * 1 <= K <= min(128, N-1). */
int culsh_gsm_merge_topk(const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals,
                         int64_t N, int64_t j_lo, int64_t n_rows, int K, double lambda_rho,
                         int32_t *entries, void *stream);

/* Count route, step 1: dense int8 panels xt/rt/qt (N x ld, zero-filled by the
 * caller): 1 / r / r*r at (j, i - row_lo) for every rating with row_lo <= i <
 * row_hi (the caller accumulates the products over row passes).  *status |= 1 if a
 * value is not an integer in [-11, 11] (use the merge route then).  Step 2 is
 * culsh_gsm_stats_tc. */
int culsh_gsm_densify_rows(const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals,
                           int64_t N, int64_t row_lo, int64_t row_hi, int64_t ld, int8_t *xt,
                           int8_t *rt, int8_t *qt, int *status, void *stream);

/* Count route, tiled panels (the layout culsh_gsm_stats_tc reads): for each (128-row
 * block rb of the ld >= N columns, 64-byte block kb of the w rating rows) a 24 KB group
 * [X | R | Q] at ((kb * ld/128 + rb) * 3 + p) * 8192, each 8 KB tile in the tcgen05 K-major
 * 64-byte-swizzle layout (column j row r = j % 128 at r * 64, 16-byte chunk c at
 * c ^ ((r >> 1) & 3)).  densify writes 1 / r / r*r for every rating (i, j) with
 * row_lo <= i < row_hi into a zero-filled 3*ld*w byte array; *status |= 1 if a value is
 * not an integer in [-11, 11] (use the merge route then).  tile_panels converts a plain
 * (3, ld, w) array. */
int culsh_gsm_densify_tiled(const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals,
                            int64_t N, int64_t row_lo, int64_t row_hi, int64_t ld, int64_t w, int8_t *tiles,
                            int *status, void *stream);
int culsh_gsm_tile_panels(const int8_t *plain, int64_t ld, int64_t w, int8_t *tiles, void *stream);

/* Count route, step 2: the four statistic products of the tiled panels:
 * g_xx (+)= X X', g_rx (+)= R X', g_rr (+)= R R', g_qx (+)= Q X' (ld x ld int32,
 * row stride ld; accumulate != 0 adds to the existing values, for row passes), and when
 * non-NULL the transposes g_xr (+)= X R', g_xq (+)= X Q' (the s2 / q2 statistics, so the
 * select kernel reads every statistic row-wise).  One
 * sm_100a kernel: bulk-copy-fed tcgen05.mma kind::i8 with TMEM accumulators, exact int32
 * (similarity.py:57-90 statistics of every pair at once).  ld % 128 == 0, w % 64 == 0. */
int culsh_gsm_stats_tc(const int8_t *tiles, int64_t ld, int64_t w, int accumulate, int32_t *g_xx,
                       int32_t *g_rx, int32_t *g_rr, int32_t *g_qx, int32_t *g_xr, int32_t *g_xq,
                       void *stream);

/* Count route, step 3 (after the int32 products g_xx = X'X, g_rx = R'X,
 * g_rr = R'R, g_qx = Q'X, each N x N with row stride ld): shrunk Pearson of every
 * pair from the exact integer statistics and the per-column top-K, rows
 * j_lo..j_lo+n_rows-1 -> entries (n_rows, K).  With the transposes g_xr / g_xq (from
 * culsh_gsm_stats_tc) every statistic is read row-wise and the selection runs as warp
 * register top-K lists; NULL: strided reads of g_rx / g_qx, per-thread lists.
 * Bit-identical to the merge route either way. */
int culsh_gsm_count_select(const int32_t *g_xx, const int32_t *g_rx, const int32_t *g_rr,
                           const int32_t *g_qx, const int32_t *g_xr, const int32_t *g_xq, int64_t ld,
                           int64_t N, int64_t j_lo, int64_t n_rows, int K, double lambda_rho,
                           int32_t *entries, void *stream);

/* similarity.py:110-135 pearson / shrunk_similarity of one pair:
 * out (device, 3 doubles) = {pearson, shrunk, co-support n}. */
int culsh_pair_similarity(const int64_t *col_ptr, const int32_t *col_rows, const double *col_vals,
                          int64_t j1, int64_t j2, double lambda_rho, double *out, void *stream);

/* ------------------------------------------------------------- ingest --- */

/* data.py:312-346 split_holdout core on HOST memory: perm is the numpy PCG64
 * permutation the caller drew (the reference's stream); entry e is moved to the test
 * side while fewer than n_test are taken and its row and column both keep a training
 * entry.  in_test: nnz bytes (0/1).  Returns the number taken, or a negative error. */
int64_t culsh_split_holdout(const int32_t *entry_rows, const int32_t *entry_cols, int64_t nnz, int64_t M,
                            int64_t N, const int64_t *perm, int64_t n_test, uint8_t *in_test);

/* --------------------------------------------------------------- init --- */

/* factorization.py:196-211 init_params / online.py:187-227 extend_params draws:
 * out[k] = 0.0 + scale * u_{skip+k} for k < n, u_t the t-th double of numpy's PCG64
 * stream seeded to (state, inc) = default_rng(seed).bit_generator.state (128-bit
 * halves), i.e. rng.uniform(0, scale, ...) bit for bit.  fp32 != 0 stores the fp64
 * value rounded to float (the Hogwild model).  Replaces the host numpy draw. */
int culsh_pcg64_uniform(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                        uint64_t skip, int64_t n, double scale, int fp32, void *out, void *stream);

/* Synthetic workload (bench and tests only, not a reference seam): the entries
 * [col_ptr[col_lo], col_ptr[col_hi]) of a random_sparse-shaped matrix
 * (datasets.py:147-164 distribution: distinct uniform rows per column, stars 1..5),
 * column j's rows a keyed permutation of [0, M) -- any column range is generated
 * independently, identically on every rank.  rows/vals are relative to col_ptr[col_lo];
 * rows are NOT sorted within a column. */
int culsh_synth_columns(int64_t M, int64_t col_lo, int64_t col_hi, const int64_t *col_ptr, uint64_t seed,
                        int32_t *rows, double *vals, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* CULSH_H_ */
