/*
 * spand_b200 — C-ABI of the B200-native spaND hot path (sm_100a).
 *
 * Boundary contract (mirrors the reference's Python operators; the host
 * package paper_2007_00789_b200 binds these with ctypes):
 *   - every entry point takes caller-owned DEVICE pointers, plain sizes and a
 *     cudaStream_t passed as void*; nothing here allocates device memory;
 *   - return value: 0 on success, a cudaError_t (>0) if the launch failed,
 *     -1 on a bad argument.  Numerical failures (non-SPD pivots) are reported
 *     through device `info` arrays (LAPACK convention: info = pivot + 1).
 *   - descriptors of batched work are device arrays of int64 rows (layouts
 *     documented per function), so no C struct crosses the boundary.
 *
 * Geometry convention shared by all factorization kernels: every dense
 * matrix is stored column-major at its cluster pair's ORIGINAL size
 * (m0[rc] x m0[cc], ld = m0[rc]); the live part is rows [off[rc], m0[rc]) x
 * cols [off[cc], m0[cc]), where `off` (device int32) grows as sparsification
 * drops fine slots (the reference keeps `dofs[n_fine:]`,
 * /root/reference/pkg/src/spdkit/factorize.py:187-190).  An OPERAND row is 7
 * int64: {ptr, rc, cc, rskip, cskip, rcount, ccount}: the operand starts
 * rskip/cskip past the live start, and is clamped to rcount/ccount when >= 0.
 */
#ifndef SPAND_B200_H
#define SPAND_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int spand_version(void);
int spand_device_sm_count(void);

/* ---- PCG building blocks (replace scipy csr_matvec sparse.py:64-68 and the
 *      NumPy vector algebra of krylov.py:93-131) ---------------------------- */

/* y = A x for CSR A (int32 indices).  If pdot != NULL also writes the
 * per-block partials of x.y into pdot (nblocks = spand_spmv_blocks(n)). */
int spand_spmv_blocks(int n);
int spand_csr_spmv(int n, const int32_t* row_ptr, const int32_t* col_idx,
                   const double* vals, const double* x, double* y,
                   double* pdot, void* stream);

/* deterministic two-stage dot: partials[nb] then out[0] = sum (fixed order) */
int spand_dot_blocks(int n);
int spand_dot(int n, const double* x, const double* y, double* partials,
              double* out, void* stream);
/* sum of nparts partials into out[0] (fixed order) */
int spand_reduce_sum(int nparts, const double* partials, double* out,
                     void* stream);

/* scal[0] = rz, scal[1] = pap -> alpha = rz / pap;  x += alpha p;
 * r -= alpha ap; partials of r.r (spand_dot_blocks(n) entries) */
int spand_pcg_xr(int n, const double* scal, double* x, double* r,
                 const double* p, const double* ap, double* partials,
                 void* stream);
/* beta = scal[2] / scal[0] (rz_new / rz); p = z + beta p */
int spand_pcg_p(int n, const double* scal, const double* z, double* p,
                void* stream);
/* y = x[perm] (gather) and y[perm] = x (scatter) */
int spand_gather(int n, const int32_t* perm, const double* x, double* y,
                 void* stream);
int spand_scatter_perm(int n, const int32_t* perm, const double* x, double* y,
                       void* stream);

/* ---- preconditioner apply (replaces Elimination/Scaling/Orthogonal/
 *      ErrorCorrection.apply_inv/apply_inv_t, schemes.py:102-112,136-140,
 *      162-166,188-192, and Factorization.apply_* factorize.py:269-282) ------
 *
 * A pass is a sequence of phases; a phase is one spand_gemv_tiles launch
 * (products of stored dense payloads with gathered vector pieces, written to
 * scratch) followed by one spand_apply_scatter launch (overwrite or
 * deterministic ordered subtract-accumulate into x).
 *
 * GEMV task row (8 x int64): {M, ld, rows, cols, trans, rot, in_kind, in_ptr}
 *   op = M (trans 0: outputs index rows, the inner index k runs over
 *   columns) or M^T (trans 1: outputs index columns, k runs over rows); M is
 *   column-major; logical column j of M is physical column (j + rot) % cols
 *   (the fine-first column order of the Orthogonal op, schemes.py:291).
 *   Input element k: in_kind 0: x[idx[k]] with idx = (int32*)in_ptr;
 *   in_kind 1: ((double*)in_ptr)[k] (a contiguous piece of x).
 * tile row (8 x int64): {task, ob, oc, kb, kc, out_off, 0, 0}
 *   scratch[out_off + i] = sum_{k in [kb, kb+kc)} op(M)[ob+i, k] * in[k], i < oc <= 64,
 *   kc <= 2048 (larger inner dimensions are split into several tiles whose
 *   partial sums the scatter step adds in a fixed order).
 * nvec right-hand sides: x is (n x nvec) with leading dim ldx and scratch
 * (len x nvec) with leading dim ldscr.
 */
int spand_gemv_tiles(int ntiles, const int64_t* tiles, const int64_t* tasks,
                     const double* x, int64_t ldx, double* scratch,
                     int64_t ldscr, int nvec, void* stream);
/* Warp-granular variant used by the engine-built plans: item rows have the
 * tile layout, but one WARP processes an item (trans 0: oc <= 256 rows x kc
 * columns; trans 1: oc <= 8 columns x kc rows); `grid` CTAs of 8 warps walk
 * the items (grid 0: one warp per item). */
int spand_gemv_items(int nitem, int grid, const int64_t* items, const int64_t* tasks,
                     const double* x, int64_t ldx, double* scratch, int64_t ldscr,
                     int nvec, void* stream);
/* for e in [0, nout): s = sum_{t in [ptr[e], ptr[e+1])} scratch[src[t]]
 * (summed in the stored order: deterministic); mode[e] == 0: x[dst[e]] = s,
 * mode[e] == 1: x[dst[e]] -= s. */
int spand_apply_scatter(int nout, const int64_t* dst, const int64_t* mode,
                        const int64_t* ptr, const int64_t* src, double* x,
                        int64_t ldx, const double* scratch, int64_t ldscr,
                        int nvec, void* stream);
/* Run-structured variant used by the structured (engine-built) plans: the
 * outputs of a phase are contiguous destination runs (whole live cluster
 * ranges in the cluster-contiguous numbering), so one row describes up to
 * 256 outputs.  chunk row (8 x int64): {dst, len <= 256, mode, cb, ce, eoff,
 * idx, 0}: for i < len, x[d] (d = dst + eoff + i, or ((int32*)idx)[eoff + i] when idx
 * != 0) = or -= sum_{c in [cb, ce)} scratch[contrib[c] + eoff + i], in order. */
int spand_apply_runs(int nchunk, const int64_t* chunks, const int64_t* contrib, double* x,
                     int64_t ldx, const double* scratch, int64_t ldscr, int nvec,
                     void* stream);
/* A whole forward or backward pass of a structured plan: for each of the
 * nphase rows of the HOST phase table ph (10 int64: {tasks, ntask, items,
 * nitem, chunks, nchunk, contrib, grid, 0, 0}, offsets in int64 units into
 * the device image), spand_gemv_items then spand_apply_runs on `stream`.
 * Same result as issuing the 2 nphase calls one by one. */
/* One forward or backward pass of the apply as one cooperative launch per
 * group of <= 4 right-hand sides: every phase's work items, a grid barrier,
 * its accumulation chunks, a grid barrier (spand_apply_pass does the same
 * with two launches per phase).  ph: the phase table (10 int64 per phase)
 * in DEVICE memory; bar: 2 uint32 of device scratch (zeroed here). */
int spand_apply_pass_persistent(int nphase, const int64_t* ph, const int64_t* image, double* x,
                                int64_t ldx, double* scratch, int64_t ldscr, int nvec,
                                unsigned* bar, void* stream);
/* The whole apply_m (forward + backward pass) as one persistent launch per
 * group of <= 4 right-hand sides: units (8 int64: {phase, kind, index,
 * first dep, ndeps, counter, counter2, 0}) run in order once their
 * dependency counters ({counter, target} pairs) are reached; ctrs (nctr
 * uint64) are zeroed here before every launch; phases: 8 int64 per phase
 * {tasks, items, chunks, contributions (offsets into image), scratch base}.
 * Schedule: spand_collect_dataflow. */
int spand_apply_dataflow(int64_t nunit, const int64_t* units, const int64_t* deps, int64_t nctr,
                         unsigned long long* ctrs, const int64_t* phases, const int64_t* image,
                         double* x, int64_t ldx, double* scratch, int64_t ldscr, int nvec,
                         void* stream);
/* Nonzero-row bits of column-major panels (the elimination panels of the
 * apply, reference schemes.py:102-112 stores them densely): panels rows
 * {address, ld, rows, cols, first word}; bit i of the panel's words is set
 * iff row i holds a nonzero.  The apply image keeps only row runs. */
int spand_row_bits(int npanel, const int64_t* panels, uint32_t* bits, void* stream);
int spand_apply_pass(int nphase, const int64_t* ph, const int64_t* image, double* x,
                     int64_t ldx, double* scratch, int64_t ldscr, int nvec, void* stream);

/* ---- factorization kernels (replace dense.py:45-183 and the BLAS calls of
 *      schemes.py:199-236, factorize.py:131-220) ---------------------------- */

/* Batched in-place Cholesky (lower) of square operands.  Task row (8 int64):
 * {operand(7), info slot}.  The failing pivot p (0-based, within the operand)
 * is reported as info[slot] = p + piv_off + 1 (LAPACK convention,
 * dense.py:53-55); first_only = 0 overwrites the slot (0 on success),
 * first_only = 1 only records the first failure (blocked factorizations of
 * large blocks, piv_off = the diagonal block's row offset). */
int spand_potrf_batched(int ntask, const int64_t* ops, const int32_t* m0,
                        const int32_t* off, int32_t* info, int piv_off, int first_only,
                        void* stream);
/* Batched lower-triangular inverse: task row = {L operand(7), Linv operand(7)}.
 * Upper triangle of Linv is written with zeros (dense.py:85-93). */
int spand_trtri_batched(int ntask, const int64_t* ops, const int32_t* m0,
                        const int32_t* off, void* stream);
/* Inverse of <= 64x64 lower-triangular tiles (task row = {L operand, X
 * operand}, each clamped to 64x64 with rcount/ccount); X's tile is written
 * in full (zeros above the diagonal).  Used with spand_gemm_grouped for the
 * recursive-doubling trtri of whole levels. */
int spand_trtri_tiles(int ntask, const int64_t* ops, const int32_t* m0,
                      const int32_t* off, void* stream);
/* Batched copy: task row = {src operand(7), dst operand(7), mode}; mode 0:
 * copy the full live rectangle, 1: copy lower triangle + zero upper, 2:
 * write the identity (src ignored). */
int spand_copy_batched(int ntask, const int64_t* ops, const int32_t* m0,
                       const int32_t* off, void* stream);

/* Grouped FP64 GEMM on DMMA tensor cores (mma.sync m8n8k4 f64):
 *   C = beta * C + alpha * sum_{s in segs(target)} A_s * op(B_s)
 * target row (8 int64): {C operand(7), seg_begin}; seg_end = next target's
 * seg_begin (targets array has ntarget+1 rows' worth of seg_begin: the row
 * after the last carries only seg_begin at column 7).
 * segment row (14 int64): {A operand(7), B operand(7)}; A is M x K; B is N x K
 * (bT = 1: op(B) = B^T, "NT") or K x N (bT = 0, "NN").
 * tile (1 int64, packed): target << 32 | (i0 / BM) << 16 | (j0 / BN); the
 * tile shape BM x BN is tri >> 4: 0 64x64, 1 64x16, 2 32x32, 3 16x16,
 * 4 16x64, 5 64x32, 6 32x64 (one shape per launch; the planner launches each
 * logical GEMM once per shape its targets use).
 * lower_only: skip tiles strictly above the diagonal (j0 >= i0 + BM; SYRK use).
 * tri & 7: triangular operands (zero above their diagonal) bound the K range
 * of a tile at (i0, j0): 1 A lower -> k < i0 + BM; 2 B lower and bT = 1 ->
 * k < j0 + BN; 4 B lower and bT = 0 -> k >= j0 (TRSM/TRMM as GEMM at the
 * triangular flop count).
 * compact = 1: a segment is ONE int64 {A block << 32 | B block} indexing the
 * block table btab (rows {ptr, rc, cc}: whole live blocks), the Schur-update
 * form; compact = 0: 14 int64 operand rows (btab unused). */
int spand_gemm_grouped(int ntile, const int64_t* tiles, const int64_t* targets,
                       const int64_t* segs, const int32_t* m0,
                       const int32_t* off, double alpha, double beta, int bT,
                       int lower_only, int tri, const int64_t* btab, int compact,
                       void* stream);
/* The same product with K-chunk masks (bT = 0, compact = 0, one segment per
 * target): kmask[kmoff[t] + c] != 0 when rows 16 c .. 16 c + 15 of target t's
 * B operand hold a nonzero; chunks of zero rows are neither loaded nor
 * multiplied (their products are exact zeros, so the result is bit for bit
 * that of spand_gemm_grouped).  Serves the interface rescale Z_i^-1 B
 * (factorize.py:165-173, schemes.py:235): before its first sparsification a
 * separator is coupled to a neighbour through a few of its rows only.
 * With bT = 1 (the panel TRSM A_ws L_s^-T of eliminate_interior,
 * factorize.py:131-149 / schemes.py:217) the bytes flag 16-row chunks of the
 * A operand instead: a tile whose rows of A are all zero writes its zeros
 * without loading anything.  With compact = 1 (the Schur update) kmoff has
 * one entry per SEGMENT, {A panel's flag offset << 32 | B panel's}: a tile
 * opens only the segments whose A rows (its i range) and B rows (its j
 * range) both hold a nonzero, in their original order.  kmask = NULL: no
 * masks. */
int spand_gemm_grouped_masked(int ntile, const int64_t* tiles, const int64_t* targets,
                              const int64_t* segs, const int32_t* m0,
                              const int32_t* off, double alpha, double beta, int bT,
                              int lower_only, int tri, const int64_t* btab, int compact,
                              const unsigned char* kmask, const int64_t* kmoff,
                              void* stream);
/* Writes the row-chunk masks of a masked launch: the A (which = 0) or B
 * (which = 1) operand of every target's first segment (14-int64 segment
 * rows), one byte per 16 rows. */
int spand_gemm_kmask(int ntarget, const int64_t* targets, const int64_t* segs,
                     const int32_t* m0, const int32_t* off, unsigned char* kmask,
                     const int64_t* kmoff, int which, void* stream);

/* One wave of the batched early-stopping column-pivoted Householder QR of
 * interface panels (restates dense.py:117-222, schemes.py:272-318,
 * factorize.py:175-196): gathers each panel from its blocks, factors it with
 * a co-resident group of CTAs (cooperative launch of `grid` CTAs), writes
 * R's coarse rows (and the kept correction rows) back into the blocks, Q
 * into its buffer, advances off[p] by the fine count and records an event.
 * scheme: 0 first, 1 second-full, 2 second-superfine.  vmax: largest live
 * panel height in the wave (<= 6144).  Row layouts: see rrqr.cu. */
int spand_rrqr_wave(int npanel, int grid, int vmax, const int64_t* panels,
                    const int64_t* nbrs, int32_t* m0, int32_t* off, double eps,
                    int scheme, int64_t* events, void* stream);
int spand_rrqr_cta_count(void);
/* co-resident CTA capacity of one wave launch whose tallest panel has vmax
 * live rows (the cooperative grid must not exceed it) */
int spand_rrqr_capacity(int vmax);
/* The same wave launched as thread-block clusters of cs (2, 4, 8) CTAs:
 * every panel's group is a multiple of cs CTAs starting at a multiple of cs
 * and grid % cs == 0.  Inside the elimination loop each cluster owns the
 * columns c = cluster index (mod clusters in the group) and splits their
 * rows over its CTAs; column dots and the pivot norm are summed over the
 * cluster through distributed shared memory.  Same outputs as
 * spand_rrqr_wave (bitwise-identical decisions; rounding of the updates may
 * differ).  vmax <= spand_rrqr_max_rows_clustered(cs). */
int spand_rrqr_wave_clustered(int npanel, int grid, int vmax, int cs, const int64_t* panels,
                              const int64_t* nbrs, int32_t* m0, int32_t* off, double eps,
                              int scheme, int64_t* events, void* stream);
/* co-resident CTA capacity of a clustered wave (whole clusters of cs) */
int spand_rrqr_cluster_capacity(int vmax, int cs);
int spand_rrqr_max_rows_clustered(int cs);
/* planner: clustered RRQR waves (cs 0/1 = off) for waves whose panels all
 * have >= min_rows live rows and that fit one cluster per panel */
int spand_plan_set_cluster(void* h, int cs, int min_rows);

/* ---- near-kernel preservation (EXTENSION, not in the reference; SURVEY.md
 *      §8a-11; CPU restatement oracle/spand_oracle.py sparsify_panel_nk).
 * U: near-kernel coordinates, column-major (ldu x k, k <= 16) in the
 * cluster-contiguous numbering.  Row layouts: see nearkernel.cu. ---------- */
/* u_p <- Z_p^T u_p for rescaled interfaces; rows {p, Z ptr, ustart} */
int spand_nk_rescale(int ntask, const int64_t* rows, const int32_t* m0, const int32_t* off,
                     double* U, int64_t ldu, int k, int vmax, void* stream);
/* column-pivoted Householder basis of u_p (rank by rtol), u_p <- [0; R_u] */
int spand_nk_basis(int npanel, const int64_t* rows, const int64_t* nbrs, const int32_t* m0,
                   const int32_t* off, double* U, int64_t ldu, int k, double rtol,
                   void* stream);
/* panel W <- [U_perp^T W; U^T W] in the pool blocks (ncols: capacity grid) */
int spand_nk_deflate(int npanel, int64_t ncols, const int64_t* rows, const int64_t* nbrs,
                     const int32_t* m0, const int32_t* off, int vmax, void* stream);
/* Orthogonal op factor [U_perp q2_c, U, U_perp q2_f] from the RRQR's q2 */
int spand_nk_qform(int npanel, int64_t ncols, const int64_t* rows, const int64_t* events,
                   int vmax, void* stream);
int spand_plan_set_nk(void* h, int k);
int spand_plan_set_group_weight(void* h, int w, double exp_m, double exp_n);

/* Final dense block (factorize.py:198-220): assemble the live parts of the
 * remaining clusters (cl[ncl] cluster ids, ascending) into the virtual
 * cluster final_id's m0^2 buffer `dst` (zeroed by the caller), packed at the
 * bottom-right; sets off[final_id].  block rows (4 int64): {index of ci in
 * cl, index of cj in cl, block ptr, 0} for stored blocks (ci <= cj). */
int spand_assemble_final(int ncl, const int64_t* cl, int64_t nblk,
                         const int64_t* blocks, const int32_t* m0,
                         int32_t* off, int32_t final_id, double* dst,
                         void* stream);

/* Nonzero counts of stored payload windows: view rows {ptr, ld, rows, cols};
 * out[i] += count (zeroed by the caller).  (count_nonzero of the reference's
 * nnz properties, schemes.py:114-117,142-144,168-170,194-196.) */
int spand_count_nonzero(int nview, const int64_t* views, unsigned long long* out,
                        void* stream);
/* Total nonzero count of payload windows, load-balanced.  View rows are the
 * collector's {offset (bit 62 set: in fac, else in pool; in doubles), ld,
 * rows, cols}; view v is cut into ceil(cols / max(1, 65536 / max(rows, 1)))
 * column pieces, pstart (nview + 1, device) is the exclusive prefix sum of
 * those counts and npiece = pstart[nview]; the count is ADDED to *total. */
int spand_count_nonzero_pieces(int nview, const int64_t* views, const int64_t* pstart,
                               int64_t npiece, const double* pool, const double* fac,
                               unsigned long long* total, void* stream);

/* Trailing-matrix fingerprint pieces (EliminationState.digest,
 * factorize.py:222-229, taken per level at :347).  Piece rows (6 int64):
 * {block ptr, i, j, first column, columns, record ptr}; each piece ADDS an
 * order-free 64-bit hash of its part of block (i, j)'s live window to
 * record[4] and the piece at column 0 writes record[0..3] = {i, j, live
 * rows, live cols}.  Records are 5 int64, zeroed by the caller. */
int spand_digest_pieces(int npiece, const int64_t* rows, const int32_t* m0,
                        const int32_t* off, void* stream);

/* ---- input side on the device (sparse.py:181-308) ---------- */

/* Row counts (cnt[n], device) of the nd-dimensional (2 or 3) cell-grid
 * finite-volume matrix with dims[nd] cells per axis. */
int spand_fv_counts(int nd, const int64_t* dims, int64_t* cnt, void* stream);
/* Columns / values of that matrix given its row_ptr (device, n + 1):
 * -div(a grad u), a piecewise constant with bv[] per block of `block` cells
 * per axis (C order), harmonic-mean faces, Dirichlet faces adding the cell's
 * coefficient; bitwise equal to the host generator diffusion_fv. */
int spand_fv_fill(int nd, const int64_t* dims, int block, const double* bv,
                  const int64_t* row_ptr, int64_t* col_idx, double* values,
                  void* stream);
/* Jacobi prescale in place on a device CSR (reference jacobi_prescale,
 * sparse.py:290-308): diag, s = 1/sqrt(diag), b *= s (b may be null),
 * a_ij *= s_i s_j; *bad (device int, zeroed) set on a nonpositive diagonal. */
int spand_jacobi_prescale(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                          double* values, double* diag, double* s, double* b, int* bad,
                          void* stream);

/* ---- Matrix Market reader (host, multi-threaded; sparse.py:98-160) ------- */

/* Parse; info[8] = {code, n, nnz, err_entry, bits(mirror value), header
 * end, size line begin, size line end}; code 0 ok, 1 bad header, 2
 * unsupported object/format, 3 not real symmetric, 4 bad size line, 5 not
 * square, 6 file ends early, 7 bad entry line, 8 index out of range, 9
 * duplicate entry, 10 mirror values disagree, 11 cannot open. */
void* spand_mm_read(const char* path, int64_t* info);
int spand_mm_csr(void* h, int64_t* row_ptr, int64_t* col_idx, double* values);
int spand_mm_error_span(void* h, int64_t* span);
int spand_mm_text(void* h, int64_t begin, int64_t end, char* out);
void spand_mm_free(void* h);

/* ---- host-side integer structure (partition.py:118-268) ------------------ */

/* Nested-dissection hierarchy of the graph of a CSR matrix (host memory).
 * dofs_out[n]: cluster dofs concatenated in id order; cptr_out[n+1]: cluster
 * boundaries; depth_out[n]: cluster depths; ncl_out[0]: cluster count. */
int spand_nd_partition(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                       int levels, int64_t* dofs_out, int64_t* cptr_out,
                       int32_t* depth_out, int64_t* ncl_out);

/* Symmetric CSR input validation (sparse.py:40-58), host memory: 0 ok,
 * 1 column out of range, 2 columns not increasing, 3 not symmetric,
 * 4 missing / nonpositive diagonal (first failing property). */
int spand_csr_check(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                    const double* values);

/* ---- native level scheduler (planner.cpp) and collector (collect.cpp) ----
 * Host-side runtime of the factorization: symbolic structure, the launch
 * program, and after the run the operator tables / permutation /
 * diagnostics / apply image.  Layouts are documented in the sources. */
void* spand_plan_create(int ncl, const int64_t* m0, const int32_t* depth, int levels,
                        int skip, int64_t npairs, const int64_t* pairs, int cap_override);
void spand_plan_destroy(void* h);
/* cluster-pair keys of A's nonzeros (ci * ncl + cj, ci <= cj, sorted, unique);
 * out holds nnz(A) entries; returns the count */
int64_t spand_plan_pairs(int ncl, const int64_t* row_ptr, const int64_t* col_idx,
                         const int64_t* cluster_of, const int64_t* cdofs, const int64_t* cptr,
                         int64_t* out);
int spand_plan_set_dofs(void* h, const int64_t* dofs, const int64_t* dptr);
/* pool offsets of A's upper-block entries in CSR order (-1: other triangle) */
int spand_plan_scatter(void* h, const int64_t* row_ptr, const int64_t* col_idx,
                       const int64_t* cluster_of, int64_t* where);
int spand_plan_sizes(void* h, int64_t* out);
int spand_plan_emit(void* h, int64_t pool_base, int64_t fac_base, int64_t temp_base,
                    int64_t ctr_base, int dry);
int spand_plan_program(void* h, int64_t* prog, int64_t* launches);
/* incremental emission (one level per call, then the final block):
 * chunk_sizes[3] = {program length, launch count, workspace used so far};
 * spand_plan_chunk copies the chunk with chunk-relative program offsets. */
int spand_plan_emit_begin(void* h, int64_t pool_base, int64_t fac_base, int64_t temp_base,
                          int64_t ctr_base);
int spand_plan_emit_next(void* h, int64_t* chunk_sizes);
int spand_plan_chunk(void* h, int64_t* prog, int64_t* launches);
int spand_plan_meta(void* h, int64_t* out);
/* Per-level trailing-matrix digests on/off (launch type 11 at every level
 * end); returns the record count, first[nlevels + 1] the per-level record
 * offsets (may be null).  Call with out_base = 0 to size, then with the
 * device address of the zeroed records before emission. */
int64_t spand_plan_set_digest(void* h, int on, int64_t out_base, int64_t* first);
void* spand_collect_create(void* plan, const int64_t* events, int scheme);
void spand_collect_destroy(void* h);
int spand_collect_sizes(void* h, int64_t* out);
int spand_collect_get(void* h, int64_t* ops, int64_t* segs, int64_t* perm, int64_t* diag,
                      int64_t* lsum, int64_t* views, int64_t* fidx);
int spand_collect_fine(void* h, int64_t* out);
int spand_collect_stats(void* h, int64_t* out);
/* bits: the nonzero-row bits of the elimination panels (spand_row_bits over
 * spand_collect_flag_panels; null: every row kept) */
int spand_collect_apply(void* h, int64_t pool_base, int64_t fac_base, int64_t xbuf,
                        int64_t idx_addr, const uint32_t* bits, int64_t* out);
/* out[0] panels, out[1] bit words */
int spand_collect_flag_sizes(void* h, int64_t* out);
/* the dataflow schedule of the apply (after spand_collect_apply): out[4] =
 * units, deps, counters, scratch doubles per right-hand side */
int spand_collect_dataflow_sizes(void* h, int64_t* out);
int spand_collect_dataflow(void* h, int64_t* units, int64_t* deps, int64_t* phases);
/* 5 int64 per panel: {address, ld, rows, cols, first word} */
int spand_collect_flag_panels(void* h, int64_t pool_base, int64_t* out);
int spand_collect_apply_get(void* h, int64_t* image, int64_t* phases);

#ifdef __cplusplus
}
#endif
#endif
