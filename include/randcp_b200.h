/*
 * randcp_b200.h -- C ABI of the B200-native leverage-score-sampled ALS hot path.
 *
 * The reference (`randcp`, pure Python/numpy, /root/reference/pkg/src/randcp) has no
 * FFI: its boundary is the Python API called by schedules.py / als.py.  Each entry point
 * below replaces one piece of arithmetic behind that API; the comment on each cites the
 * reference function (file:line) it implements.  The Python package
 * `paper_2210_05105_b200` binds these with ctypes and keeps the reference's names,
 * signatures and exceptions.
 *
 * Conventions
 *   - Plain pointers and sizes only; no torch types.  All `d_*` pointers are device
 *     pointers (cudaMalloc / torch CUDA allocations), `h_*` pointers are host memory.
 *   - `stream` is a cudaStream_t passed as void*; every device call is stream-ordered and
 *     asynchronous.  Nothing allocates: workspaces are caller-provided and sized by the
 *     matching *_ws_bytes() query.
 *   - Matrices are row-major fp64.  Sample index matrices are stored mode-major
 *     (X[m*J + s] = mode-m row of sample s; the reference's X is (J, N), i.e. transposed).
 *   - Return value: RCP_OK or a launch/argument error.  Data-dependent errors (zero-mass
 *     walk, zero sampling probability, asymmetric Gram, non-finite factor) are raised on
 *     the device into `d_status` (one int32, bitwise OR of RCP_ST_* flags) and surfaced
 *     by the host after its next synchronisation, mapped to the reference exceptions:
 *       RCP_ST_DEGENERATE -> DegenerateWalkError   (ref samplers.py:34-35)
 *       RCP_ST_ZERO_PROB  -> ValueError            (ref samplers.py:93-94)
 *       RCP_ST_ASYMMETRIC -> ValueError            (ref linalg.py:92-95)
 *       RCP_ST_ZERO_MASS  -> ValueError            (ref samplers.py:142-143,167-168)
 *       RCP_ST_NONFINITE  -> FloatingPointError    (ref als.py:202-204)
 */
#ifndef RANDCP_B200_H
#define RANDCP_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RCP_OK 0
#define RCP_ERR_ARG 1
#define RCP_ERR_CUDA 2

#define RCP_ST_DEGENERATE 1
#define RCP_ST_ZERO_PROB 2
#define RCP_ST_ASYMMETRIC 4
#define RCP_ST_ZERO_MASS 8
#define RCP_ST_NONFINITE 16
#define RCP_ST_CAPACITY 32
#define RCP_ST_TIMEOUT 64

#define RCP_MAX_RANK 128

/* Stream keys: entry points that draw from a Philox stream take its key by value
 * (key0, key1) and, optionally, `d_key`: a device pointer to the two key words that
 * overrides them when non-NULL, so a captured CUDA graph can replay a round with the
 * next round's keys written into device memory beforehand. */
/* ---------------------------------------------------------------- version / errors */
const char *rcp_version(void);
const char *rcp_last_error(void);
/* Number of SMs of the current device (0 without a device). */
int rcp_device_sms(void);
/* Number of kernels this library has launched in the process (all entry points). */
int64_t rcp_launch_count(void);

/* ------------------------------------------------------------------- random streams
 * Reference: rng.stream(seed, purpose, *context) builds
 *   Generator(Philox(SeedSequence(entropy=seed, spawn_key=(purpose,)+context)))
 * (ref rng.py:26-32).  These reproduce numpy 2.x's SeedSequence key derivation,
 * Philox4x64-10 stream, Generator.random() and Generator.permutation() bit for bit. */

/* key_out[2] = SeedSequence(seed, spawn_key=(purpose, ctx...)).generate_state(2, uint64). */
int rcp_stream_key(uint64_t seed, uint64_t purpose, const uint64_t *h_ctx, int n_ctx,
                   uint64_t *h_key_out);
/* Host: draws [first, first+n) of Generator.random() on that key. */
int rcp_uniform_host(const uint64_t *h_key, int64_t first, int64_t n, double *h_out);
/* Host: Generator.permutation(n) (arange + Fisher-Yates with masked-rejection
 * random_interval on buffered uint32 draws).  Used for the CP-ARLS-LEV SHUFFLE stream
 * (ref samplers.py:183). */
int rcp_permutation_host(const uint64_t *h_key, int64_t n, int64_t *h_out);
/* `count` permutations of the streams h_keys[2c], h_keys[2c+1] into h_outs[c] (n each),
 * spread over `threads` host threads (the CP-ARLS-LEV SHUFFLE streams of a round). */
int rcp_permutations_host(const uint64_t *h_keys, int count, int64_t n, int64_t *const *h_outs,
                          int threads);
/* Device: d_out[i] = draw (first+i) of Generator.random(). */
int rcp_uniform(uint64_t key0, uint64_t key1, int64_t first, int64_t n, double *d_out,
                void *stream);

/* ------------------------------------------------------------- small dense algebra */
/* G = sum_rows (s_r u_r)(s_r u_r)^T for U (n x R); d_scale may be NULL (s_r = 1).
 * Deterministic (fixed CTA partition + ordered reduction).
 * Ref: gram() linalg.py:64-70; sketched Gram (H.w)^T(H.w) schedules.py:104-109. */
size_t rcp_gram_ws_bytes(int64_t n, int R);
int rcp_gram(const double *d_U, const double *d_scale, int64_t n, int R, double *d_G,
             void *d_ws, void *stream);

/* Moore-Penrose inverse of a symmetric PSD R x R matrix with eigenvalue cutoff
 * rel_cutoff * lambda_max (ref pseudo_inverse linalg.py:85-104): symmetry check
 * (RCP_ST_ASYMMETRIC), then a Cholesky inverse when its Frobenius condition bound
 * proves every eigenvalue is above the cutoff, else a parallel cyclic Jacobi
 * eigendecomposition with the reference's cutoff rule.  One CTA.
 * If n_chain > 0, the input is first formed as the Hadamard product of the n_chain
 * R x R matrices d_in[m*R*R] skipping index `skip` (ref hadamard_gram_chain
 * linalg.py:73-82); d_chain_out (nullable) receives that product. */
int rcp_pinv(const double *d_in, int n_chain, int skip, int R, double rel_cutoff,
             double *d_chain_out, double *d_out, int *d_status, void *stream);

/* U_out (n x R) = M (n x R) @ B (R x R); also accumulates per-column sums of squares of
 * U_out into d_colsq (R, caller-zeroed, via ordered per-CTA partials in d_ws) and flags
 * non-finite entries (RCP_ST_NONFINITE).  Ref: _postprocess schedules.py:124-128 and
 * the finite check als.py:202-204. */
size_t rcp_update_ws_bytes(int64_t n, int R);
int rcp_update(const double *d_M, int64_t n, int R, const double *d_B, double *d_U_out,
               double *d_colsq, void *d_ws, int *d_status, void *stream);
/* sigma = sqrt(colsq); U /= (sigma > 0 ? sigma : 1) in place (ref _renormalize
 * als.py:129-138). */
int rcp_renormalize(double *d_U, int64_t n, int R, const double *d_colsq, double *d_sigma,
                    void *stream);

/* ------------------------------------------------------------ CP-ARLS-LEV sampler
 * Ref: arls_lev_build samplers.py:122-135, arls_lev_sample samplers.py:148-191. */
/* d_lev[q] = max(u_q Gp u_q^T, 0); d_dist = d_lev / C (C = sum, ordered), d_cdf =
 * inclusive scan of d_dist normalised by its last element (numpy choice semantics);
 * d_mass[0] = C. */
size_t rcp_arls_build_ws_bytes(int64_t n, int R);
int rcp_arls_build(const double *d_U, int64_t n, int R, const double *d_Gp, double *d_dist,
                   double *d_cdf, double *d_mass, void *d_ws, void *stream);
/* q draws from one rank's distribution with stream key (LOCAL_DRAW): row = row_lo +
 * searchsorted(cdf, u, 'right'); prob = (C_p / W) * dist[row].  Writes into
 * d_rows_out/d_prob_out at [offset, offset+q).  d_total_mass (nullable, device scalar):
 * RCP_ST_ZERO_MASS is raised when it is <= 0 (ref samplers.py:166-168).
 * d_urow_out (nullable): also copies the drawn factor rows U[row - row_lo] (q x R). */
int rcp_arls_draw(const double *d_cdf, const double *d_dist, int64_t n, int64_t row_lo,
                  double mass_ratio, const double *d_total_mass, uint64_t key0, uint64_t key1,
                  const uint64_t *d_key, int64_t q, int64_t offset, int64_t *d_rows_out,
                  double *d_prob_out, const double *d_U, int R, double *d_urow_out, int *d_status,
                  void *stream);
/* Apply the SHUFFLE permutation and fold mode i into the batch:
 * X_i[s] = rows[perm[s]], pmp_i[s] = prob[perm[s]], H[s,:] (*)= row(perm[s]) where
 * row(t) = d_urows[t,:] when d_urows != NULL, else U[rows[t] - u_row_lo, :].
 * d_perm may be NULL (identity).  `first` != 0 assigns H instead of multiplying. */
int rcp_batch_fold(const int64_t *d_perm, const int64_t *d_rows, const double *d_prob,
                   int64_t J, const double *d_U, int64_t u_row_lo, const double *d_urows,
                   int R, int first, int64_t *d_Xi, double *d_pmp_i, double *d_H,
                   void *stream);

/* ------------------------------------------------------------------ STS-CP sampler
 * Ref: sts_build samplers.py:224-288, sts_sample samplers.py:379-468.
 * Device layout: complete binary tree over leaf blocks of `leaf` consecutive rows; level
 * l holds 2^l node Grams, each packed upper-triangular (R(R+1)/2 doubles, row-major),
 * node stride S = R(R+1)/2 rounded up to even (zero pad, 16-byte aligned nodes); node
 * (l, v) lives at offset ((1<<l) - 1 + v) * S.  depth = ceil(log2(n_leaves)). */
int rcp_sts_depth(int64_t n, int leaf);
size_t rcp_sts_tree_doubles(int64_t n, int leaf, int R);
/* Conditioning matrix of constant mode i in a mode-k solve:
 * M = chain_pinv (.) prod_{m>i, m!=k} G_m, left fold in mode order (ref samplers.py:412-415).
 * d_grams: N stacked R x R Grams. */
int rcp_sts_cond(const double *d_chain_pinv, const double *d_grams, int N, int i, int k, int R,
                 double *d_M, void *stream);
/* Shared (rank-level) levels of the walk for P > 1 (ref samplers.py:423-451): node Grams
 * of the padded rank tree, full R x R each, level-major (level l at offset (2^l-1)*R*R);
 * leaf_rank[2^depth] maps tree leaves to ranks (-1 = padding).  Writes owner rank, the
 * rescaled residual and the product of step probabilities; RCP_ST_DEGENERATE on a
 * zero-mass node or a branch into an empty padded subtree.  d_key: as rcp_sts_walk's
 * (non-null: the two key words are read from device memory, for graph-replayed rounds). */
int rcp_sts_rank_walk(const double *d_node_grams, int depth, int P, const int32_t *d_leaf_rank,
                      const double *d_M, const double *d_H, int64_t J, int R, uint64_t key0,
                      uint64_t key1, const uint64_t *d_key, const double *d_override,
                      int32_t *d_owner,
                      double *d_r_out, double *d_pmp_i, int *d_status, void *stream);
/* The rank tree in the local trees' packed layout (complete tree over 2^ceil(log2 P) leaves;
 * leaf v = packed upper triangle of block Gram d_order[v] (d_order NULL: v), zero padding;
 * inner nodes = sums of their children, ref samplers.py:239-275), and the rank-level walk
 * over it grouped by the key of the modes already sampled, like rcp_sts_walk: node masses
 * are evaluated once per distinct (H row, node) instead of once per sample.  Outputs per
 * sample: owner rank (-1 for a degenerate run), rescaled residual, product of the step
 * probabilities.  d_leaf_rank[2^depth] maps tree leaves to ranks (-1 = padding). */
size_t rcp_sts_rank_tree_doubles(int P, int R);
int rcp_sts_rank_tree(const double *d_block_grams, const int64_t *d_order, int P, int R,
                      double *d_tree, void *stream);
size_t rcp_sts_rank_walk_ws_bytes(int64_t J, int P, int R);
int rcp_sts_rank_walk_grouped(const double *d_rank_tree, int P, const int32_t *d_leaf_rank,
                              int R, const double *d_M, const double *d_H_in,
                              const int64_t *d_hkey, int key_bits, int64_t J, uint64_t key0,
                              uint64_t key1, const uint64_t *d_key, const double *d_override,
                              int32_t *d_owner, double *d_r_out, double *d_pmp_i, void *d_ws,
                              size_t ws_bytes, int *d_status, void *stream);
/* The rank-level walk of the first constant mode (every sample's Hadamard row is ones): the
 * 2^(depth+1)-1 node masses are evaluated once per CTA, then every sample descends alone.
 * Same outputs and errors as rcp_sts_rank_walk_grouped; P <= 1024. */
int rcp_sts_rank_walk_ones(const double *d_rank_tree, int P, const int32_t *d_leaf_rank, int R,
                           const double *d_M, int64_t J, uint64_t key0, uint64_t key1,
                           const uint64_t *d_key, const double *d_override, int32_t *d_owner,
                           double *d_r_out, double *d_pmp_i, int *d_status, void *stream);
/* Local search of the first constant mode at P > 1 (all samples share H = ones): samples
 * with d_sel[s] == sel_value invert the CDF of this rank's row masses (rcp_arls_build of
 * the block with the conditioning matrix) at their residual d_rin[s]
 * (ref _leaf_search_batch samplers.py:313-345): d_Xi[s] = row, d_pmp_i[s] *= dist[row],
 * d_resid[s] (nullable) = the residual inside the row's segment.  RCP_ST_DEGENERATE when
 * a sample is routed to a rank without mass. */
int rcp_sts_flat_local(const double *d_cdf, const double *d_dist, int64_t n, int64_t row_lo,
                       const double *d_total_mass, const double *d_rin, const int32_t *d_sel,
                       int32_t sel_value, int64_t J, int64_t *d_Xi, double *d_pmp_i,
                       double *d_resid, int *d_status, void *stream);
/* STS exchange buffers (ref schedules.py:239-247; J x (R + 3) doubles per rank, summed by
 * one all-reduce): pack = [row, step probability, residual, factor row] of the samples
 * this rank owns and zeros elsewhere; unpack = every sample's row, probability and
 * residual, and H[s,:] = row (init) or H[s,:] (.) row. */
int rcp_exchange_pack(const int64_t *d_Xi, const double *d_pmp_i, const double *d_resid,
                      const double *d_U, int64_t n, int64_t row_lo, const int32_t *d_owner,
                      int32_t rank, int64_t J, int R, double *d_buf, void *stream);
int rcp_exchange_unpack(const double *d_buf, int64_t J, int R, int init, int64_t *d_Xi,
                        double *d_pmp_i, double *d_resid, double *d_H, void *stream);
int rcp_sts_build(const double *d_U, int64_t n, int R, int leaf, double *d_tree,
                  void *stream);
/* Walk J samples down the tree of one factor block (rows global [row_lo, row_lo+n)).
 * M = conditioning matrix (R x R, full) for this mode (ref samplers.py:412-415).
 * d_H_in: running Hadamard rows (J x R), NULL = all ones (first constant mode).
 * d_hkey (nullable): per-sample key of the indices already sampled in earlier modes;
 * samples with equal keys must have equal H rows; keys < 2^key_bits - 1 (key_bits in
 * [1, 64], the sort touches only those bits).  Samples are grouped by (key, r) and
 * each group descends as runs, so node masses are evaluated once per distinct
 * (H row, node).  Uniforms: d_override (J doubles) or d_rin (residuals after the
 * rank-level levels) else WALK_UNIFORM draws of key (key0,key1).
 * d_sel (nullable): only samples s with d_sel[s] == sel_value walk (multi-rank owner);
 * their d_pmp_i[s] holds the probability so far and is multiplied, otherwise it is set.
 * Outputs per walked sample: d_Xi[s] (global row), d_pmp_i[s], d_resid[s] (nullable),
 * d_H_out[s,:] = d_H_in[s,:] (.) U[row,:] (or U[row,:] when d_H_in is NULL) when d_H_out is
 * non-NULL (must not alias d_H_in: samples of one group read their common row while others
 * finish).
 * d_ws: rcp_sts_walk_ws_bytes(J, n, leaf, R) (holds this walk's G (.) M node table). */
size_t rcp_sts_walk_ws_bytes(int64_t J, int64_t n, int leaf, int R);
int rcp_sts_walk(const double *d_tree, const double *d_U, int64_t n, int R, int leaf,
                 int64_t row_lo, const double *d_M, const double *d_H_in, const int64_t *d_hkey,
                 int key_bits, int64_t J, uint64_t key0, uint64_t key1, const uint64_t *d_key,
                 const double *d_override,
                 const double *d_rin, const int32_t *d_sel, int32_t sel_value, int64_t *d_Xi,
                 double *d_pmp_i, double *d_resid, double *d_H_out, void *d_ws, size_t ws_bytes,
                 int *d_status,
                 void *stream);
/* The conditioning pass of rcp_sts_walk alone (packed M' tables and G (.) M' for every tree
 * node, written into the walk workspace): it depends only on the tree and M, so it can run
 * on another stream while earlier modes are sampled; rcp_sts_walk_prepared is rcp_sts_walk
 * on a workspace prepared this way (same tree, M, J, n, leaf, R). */
int rcp_sts_walk_gm(const double *d_tree, int64_t n, int R, int leaf, const double *d_M, int64_t J,
                    void *d_ws, size_t ws_bytes, void *stream);
int rcp_sts_walk_prepared(const double *d_tree, const double *d_U, int64_t n, int R, int leaf,
                          int64_t row_lo, const double *d_M, const double *d_H_in,
                          const int64_t *d_hkey, int key_bits, int64_t J, uint64_t key0,
                          uint64_t key1, const uint64_t *d_key, const double *d_override,
                          const double *d_rin, const int32_t *d_sel, int32_t sel_value,
                          int64_t *d_Xi, double *d_pmp_i, double *d_resid, double *d_H_out,
                          void *d_ws, size_t ws_bytes, int *d_status, void *stream);
/* Fold the walked rows: d_out[s,:] = U[X_i[s]-row_lo, :] (init != 0) or
 * d_out[s,:] *= U[X_i[s]-row_lo, :], for samples with d_sel[s] == sel_value (all when
 * d_sel is NULL) whose row lies in this block (ref samplers.py:464, H *= U_i[X_i]). */
int rcp_fold_rows(double *d_out, const double *d_U, int64_t n, int R, int64_t row_lo,
                  const int64_t *d_Xi, int64_t J, int init, const int32_t *d_sel,
                  int32_t sel_value, void *stream);
/* First constant mode of a single-rank walk (all samples share H = ones): the leaf-by-leaf
 * inverse CDF collapses to one inverse CDF over every row.  With row masses, normalised
 * masses and CDF from rcp_arls_build(U, M) (mass = u M u^T, clipped at 0), draw sample s
 * from WALK_UNIFORM draw s: X_i[s] = row_lo + searchsorted(cdf, u, 'right'),
 * pmp_i[s] = mass/total.  Same distribution and inverse-CDF map as the tree walk (ref
 * samplers.py:291-310, 379-468); RCP_ST_DEGENERATE when the total mass is zero. */
int rcp_sts_flat_draw(const double *d_cdf, const double *d_dist, int64_t n, int64_t row_lo,
                      const double *d_total_mass, uint64_t key0, uint64_t key1,
                      const uint64_t *d_key, int64_t J,
                      int64_t *d_Xi, double *d_pmp_i, int *d_status, void *stream);
/* d_out[s] = sum_m X[m*J + s] * strides[m] over modes with nonzero stride (mixed-radix
 * key of a subset of a sample's indices; ref matricization.py:41-54 for the MTTKRP
 * column key, and the STS walk's grouping key). */
int rcp_row_keys(const int64_t *d_X, int N, int64_t J, const int64_t *h_strides,
                 int64_t *d_out, void *stream);
/* d_out[e] = ((p_0[e] + p_1[e]) + p_2[e]) + ... over nparts stacked arrays of len doubles:
 * the rank-ordered sum of replicated contributions (block Grams, column sums of squares;
 * ref grid.py:295-297). */
int rcp_ordered_sum(const double *d_parts, int nparts, int64_t len, double *d_out, void *stream);
/* H[s,:] *= d_urow[s,:] for all s (fold walked rows into the running Hadamard rows). */
int rcp_hadamard_rows(double *d_H, const double *d_urow, int64_t J, int R, int init_ones,
                      void *stream);
/* Sample weights w = 1/sqrt(J * prod_m pmp[m]) (ref sample_weights samplers.py:89-96),
 * also writes prob = prod_m pmp[m] (ref samplers.py:466); RCP_ST_ZERO_PROB if prob<=0. */
int rcp_weights(const double *d_pmp, int N, int64_t J, double *d_prob, double *d_w,
                int *d_status, void *stream);

/* ------------------------------------------------------------- sampled MTTKRP
 * Per-mode sorted store (ref Matricization matricization.py:67-128), device layout:
 *   keys[n_cols]     int64  distinct column keys (off-mode mixed-radix, ascending)
 *   colptr[n_cols+1] int64  nonzeros of column c at [colptr[c], colptr[c+1])
 *   rows[nnz]        int32  local row (global row - row_lo), ascending within a column
 *   vals[nnz]        fp64
 * Downsampled MTTKRP of one mode solve (ref gather_sampled_nonzeros_to_csr
 * mttkrp.py:131-155 + downsampled_mttkrp mttkrp.py:158-189, fused):
 *   out[i,:] = sum_s w_s^2 * T(i, col(s)) * H[s,:]
 * Samples with equal column keys are merged (count * w^2, identical H rows), then the
 * distinct fibers are looked up, transposed to row order and segment-reduced.
 * d_stats (int64[8], accumulated): [0] distinct samples, [1] distinct samples with >=1
 * local nonzero, [2] gathered nonzeros (distinct fibers), [3] gathered nonzeros with
 * multiplicity (the reference's csr.nnz), [4] output rows hit; [5..7] reserved. */
size_t rcp_mttkrp_ws_bytes(int64_t J, int64_t store_nnz, int64_t n_rows, int R);
/* Byte offsets of the internal arrays inside a workspace of ws_bytes (introspection for
 * tests): dkey, dcnt, drep, dlo, dlen, doff, Hs, rcnt, rptr, ed, ev, S, nnz, then the
 * entry capacity; 14 int64 written to h_out. */
int rcp_mttkrp_layout(int64_t J, int64_t n_rows, int R, size_t ws_bytes, int64_t *h_out);
int rcp_sampled_mttkrp(const int64_t *d_keys, const int64_t *d_colptr, int64_t n_cols,
                       const int32_t *d_rows, const double *d_vals, int64_t n_rows,
                       const int64_t *d_X, int N, int64_t J, int k, const int64_t *h_strides,
                       const double *d_H, const double *d_w, int R, double *d_out,
                       int64_t *d_stats, void *d_ws, size_t ws_bytes, int *d_status,
                       void *stream);
/* MTTKRP mode for subsequent rcp_sampled_mttkrp calls (process-wide; initial value from
 * the environment: RCP_MTTKRP_PATH=tiles selects 1):
 *   0  fast: entries transposed to row order, segmented SpMM (fp64 red.add for rows split
 *      across warps; the order of a row's terms varies run to run);
 *   1  deterministic: the sampled fibers' runs per row tile ("pairs") in a canonical order,
 *      expanded stably into row-sorted entries, rows split across the SpMM's chunks summed
 *      in chunk order -- bit-identical results on every run (ref tests/test_mttkrp.py:
 *      60-67,163-172 require bit-identity across worker counts).  Row tiles of 16 rows
 *      (R <= 64) or 8 (R <= 128); above 4096 tiles the pairs are radix-sorted by tile,
 *      which reads their count on the host: such calls inside a CUDA-graph capture run
 *      mode 0.  Requires J < 2^22.
 * Returns the previous mode; a negative argument only queries. */
int rcp_set_mttkrp_mode(int mode);
/* Reference-shaped CSR gather with multiplicity (drop-in for
 * gather_sampled_nonzeros_to_csr): d_counts[s] = fiber length of sample s, and, when
 * d_pos_out != NULL, expanded (row, sample, value) triples in sample order (row-sorting
 * is done by the caller). */
int rcp_fiber_lookup(const int64_t *d_keys, int64_t n_cols, const int64_t *d_colptr,
                     const int64_t *d_X, int N, int64_t J, int k, const int64_t *h_strides,
                     int64_t *d_lo, int64_t *d_counts, void *stream);
int rcp_fiber_expand(const int64_t *d_lo, const int64_t *d_off, int64_t J,
                     const int32_t *d_rows, const double *d_vals, int64_t *d_row_out,
                     int64_t *d_col_out, double *d_val_out, void *stream);
/* CSR SpMM: out[i,:] = sum_{e in row i} val[e] * scale[col[e]] * H[col[e],:]
 * (drop-in for downsampled_mttkrp with scale = w^2; ref mttkrp.py:158-189). */
int rcp_csr_spmm(const int64_t *d_row_ptr, int64_t n_rows, const int64_t *d_col,
                 const double *d_val, const double *d_H, const double *d_scale, int R,
                 double *d_out, void *stream);

/* ---------------------------------------------------------------- exact fit (row F1)
 * Ref compute_fit linalg.py:130-151: fit = 1 - sqrt(max(||T||^2 - 2<T,T_hat> + ||T_hat||^2,
 * 0)) / ||T||.  The three scalars are computed on the device from the mode-k store.
 *   h_U[m]  device pointer of mode m's factor rows (row-major, R columns), first row h_lo[m]
 *           (NULL h_lo = 0); h_U[k] is ignored (d_Uk is the store's own row block).
 *   h_strides  the store's off-mode key strides (ref matricization.py:21-38).
 * Workspace: rcp_fit_ws_bytes(nnz).  Sums are added in a fixed order (reproducible). */
size_t rcp_fit_ws_bytes(int64_t nnz);
/* <T, T_hat> restricted to the store's nonzeros: sum_e v_e sum_r sigma_r U_k[row_e, r]
 * prod_{m != k} U_m[i_m(e), r]  -> d_out[0]. */
int rcp_fit_cross(const int64_t *d_keys, const int64_t *d_colptr, int64_t n_cols,
                  const int32_t *d_rows, const double *d_vals, int64_t nnz, int N, int k,
                  const int64_t *h_dims, const int64_t *h_strides, const double *const *h_U,
                  const int64_t *h_lo, const double *d_Uk, int R, const double *d_sigma,
                  double *d_out, void *d_ws, size_t ws_bytes, void *stream);
/* sum_i v_i^2 -> d_out[0] (ref SparseTensorCOO.norm_squared). */
int rcp_sum_squares(const double *d_v, int64_t n, double *d_out, void *d_ws, size_t ws_bytes,
                    void *stream);
/* sigma^T (G_0 (.) ... (.) G_{N-1}) sigma -> d_out[0]; d_grams N x R x R (ref
 * linalg.py:145-146 with hadamard_gram_chain linalg.py:73-82). */
int rcp_model_norm(const double *d_grams, int N, int R, const double *d_sigma, double *d_out,
                   void *stream);
/* Exact local MTTKRP (drop-in for mttkrp_exact, ref mttkrp.py:65-108): d_out (n_rows x R,
 * local rows) = sum over the store's entries of v * prod_{m != k} U_m[i_m]. */
int rcp_exact_mttkrp(const int64_t *d_keys, const int64_t *d_colptr, int64_t n_cols,
                     const int32_t *d_rows, const double *d_vals, int64_t nnz, int64_t n_rows,
                     int N, int k, const int64_t *h_dims, const int64_t *h_strides,
                     const double *const *h_U, const int64_t *h_lo, int R, double *d_out,
                     void *stream);

/* ---------------------------------------------------------------- device ingest (row F2)
 * Synthetic Zipf tensors generated on the device for the configurations that cannot be
 * built on the host (C4 1.7B, C5 4.7B nonzeros); stands in for load_frostt
 * (ref tensor.py:86-149) with sum_duplicates (tensor.py:72-83) and permute_modes
 * (tensor.py:182-210) semantics.  Draw d uses the splitmix64 stream of synth.zipf_tensor
 * with chunk = d >> chunk_bits and index d & (2^chunk_bits - 1). */
/* d_guide[b] = first i with cdf[i] > b/G (inverse-CDF start table, G entries). */
int rcp_zipf_guide(const double *d_cdf, int64_t n, int64_t G, int32_t *d_guide, void *stream);
/* Draws [d0, d1): per mode a Zipf index by inverse CDF of its cdf (searchsorted right),
 * row-major cell id (u64 bits in int64), value lognormal(0, sigma) (value_kind 0) or a
 * Poisson(3) count (1).  Only cells whose hash partition (top part_bits bits of
 * splitmix(cell)) equals `part` are appended at d_key/d_val[*d_count ...] (capacity cap;
 * overflow raises RCP_ST_CAPACITY). */
int rcp_zipf_draws(int N, const int64_t *h_dims, const double *const *h_cdf,
                   const int32_t *const *h_guide, const int64_t *h_G, uint64_t seed,
                   int chunk_bits, int64_t d0, int64_t d1, int value_kind, double sigma,
                   int part_bits, int64_t part, int64_t *d_key, double *d_val, int64_t *d_count,
                   int64_t cap, int *d_status, void *stream);
/* Stable (key, row) ordering for the per-mode sorted store and the drop-in CSR transpose:
 * d_order = the permutation numpy's lexsort((row, key)) returns (ref matricization.py:56-77),
 * by two LSD radix sorts that carry positions; d_key == NULL orders by d_row alone (the
 * counting-sort transpose of ref mttkrp.py:131-155).  Values must lie in [0, key_max] and
 * [0, row_max].  Workspace: rcp_sort_ws_bytes(n). */
size_t rcp_sort_ws_bytes(int64_t n);
int rcp_order_by_key_row(const int64_t *d_key, const int64_t *d_row, int64_t n, int64_t key_max,
                         int64_t row_max, int64_t *d_order, void *d_ws, size_t ws_bytes,
                         void *stream);
/* d_flag[i] = 1 where sorted cell ids start a new cell. */
int rcp_run_flags(const int64_t *d_sorted, int64_t n, int32_t *d_flag, void *stream);
/* Distinct cells from stably sorted draws: values summed in draw order (ln(1 + sum) when
 * log1p_vals), coordinates decoded and mapped through the per-mode permutations h_perm[m]
 * (device int32 arrays; NULL = identity) into d_idx (n_cells x N int32, row-major). */
int rcp_cells(const int64_t *d_sorted, const double *d_sval, const int64_t *d_starts,
              int64_t n_cells, int64_t n, int N, const int64_t *h_dims,
              const int32_t *const *h_perm, int log1p_vals, int32_t *d_idx, double *d_val,
              void *stream);

#ifdef __cplusplus
}
#endif
#endif /* RANDCP_B200_H */
