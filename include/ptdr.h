/*
 * ptdr.h -- C ABI of libptdr.so, the B200 (sm_100a) Pauli-decomposition hot path.
 *
 * Operation (Sec. II-A): for A in C^{2^n x 2^n},
 * compute every coefficient of A = sum_P alpha_P P over the 4^n Pauli strings
 * P = sigma_{n-1} (x) ... (x) sigma_0 (l.178), alpha_P = Tr(P A) / 2^n (l.151)
 * = tr(P^* A) / 2^n (P is Hermitian, l.128).
 *
 * Output order ("q order"): q = sum_l code(sigma_l) 4^l with code I=0, X=1, Y=2,
 * Z=3, i.e. ascending text-lexicographic order of the string, leftmost letter
 * (sigma_{n-1}) most significant -- the order of "alpha_II, alpha_IX, alpha_IY, ..."
 * (l.143).  DESIGN.md reading R5.
 *
 * Memory: every pointer argument is a DEVICE pointer (cudaMalloc / torch CUDA
 * tensor memory) unless the function name ends in _host.  The caller owns all
 * memory; the library keeps no global mutable state except a thread-local error
 * string and a per-device cache of launch parameters (SM count, band(s) index tables in
 * pinned host memory), allocates no persistent device memory, and is reentrant given
 * distinct workspaces.  Element type: ptdr_c128 =
 * interleaved (re, im) binary64 (== cuDoubleComplex == torch.complex128), 16-byte
 * aligned.  Streams are passed as `void*` holding a cudaStream_t (NULL = legacy
 * default stream).
 *
 * Errors: functions return ptdr_status and never abort or throw across the ABI.
 *   PTDR_EINVAL       bad n, structure, null / misaligned pointer, world/rank
 *   PTDR_EUNSUPPORTED valid but not implemented combination (e.g. out aliases A)
 *   PTDR_ENOMEM       workspace smaller than ptdr_workspace_bytes(), or a
 *                     temporary allocation in ptdr_decompose / _host failed
 *   PTDR_ECUDA        a CUDA API / launch error; detail in ptdr_last_error().
 *                     Asynchronous faults surface at the caller's next stream sync.
 */
#ifndef PTDR_H_
#define PTDR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double re, im;
} ptdr_c128;

/* Declared structure of A (trusted, not verified: SPEC.md l.202).
 *  GENERAL        dense row-major A[i][j] at offset i*2^n + j                    (l.294)
 *  HERMITIAN      dense storage; only the upper triangle and the real part of the
 *                 diagonal are read; output has Im == 0 exactly (Theorem 2, l.123-136)
 *  REAL_SYMMETRIC dense storage; only Re of the upper triangle + diagonal is read;
 *                 output real, exact zeros where n_Y is odd
 *  DIAGONAL       A = band array d[2^n] (d[i] = A[i][i]); output = the 2^n {I,Z}^n
 *                 coefficients (l.369-389, Table I l.511), ascending z (see below)
 *  TRIDIAGONAL    A = band array [3][2^n]: sub[i]=A[i][i-1] (sub[0] ignored),
 *                 main[i]=A[i][i], sup[i]=A[i][i+1] (sup[2^n-1] ignored); output =
 *                 the (n+1) blocks of 2^n coefficients that can be nonzero
 *                 (Theorem l.404-406, Table I l.513): block b holds the X-mask
 *                 x_b = 2^b - 1 (b = 0: the {I,Z}^n strings; b = n: the {X,Y}^n
 *                 strings), and inside a block coefficients are in ascending
 *                 Z-mask z, which is ascending q order restricted to that block.
 *  ANTI_DIAGONAL  A = a[2^n] with a[i] = A[i][2^n - 1 - i] (the anti-diagonal remark,
 *                 l.391-392: swap I,Z <-> X,Y); output = the 2^n {X,Y}^n coefficients
 *                 (X-mask 2^n - 1), ascending z.
 *  HERMITIAN_TRIDIAGONAL  A = band array [2][2^n]: main[i]=A[i][i], sup[i]=A[i][i+1]
 *                 (sup[2^n-1] ignored); the sub-diagonal is A[i+1][i] = conj(sup[i]) and not
 *                 stored (a real symmetric tridiagonal is the real case; the main diagonal is
 *                 used as given, real for a Hermitian A).  Output exactly as TRIDIAGONAL.
 *                 With S_t the sup samples of segment t and W_t = WHT(S_t), the TRIDIAGONAL
 *                 path's P_t = WHT(S_t + conj S_t) = (2 Re W_t, 0) and M_t = (0, 2 Im W_t):
 *                 one WHT per segment instead of two (Theorem 2, l.123-136: Hermitian
 *                 matrices have real coefficients; l.395-465 for the tridiagonal structure),
 *                 bitwise equal to TRIDIAGONAL on the same matrix.
 * X-mask / Z-mask of a string: bit l of x is set iff sigma_l in {X,Y}; bit l of z
 * is set iff sigma_l in {Y,Z}. */
typedef enum {
  PTDR_GENERAL = 0,
  PTDR_HERMITIAN = 1,
  PTDR_REAL_SYMMETRIC = 2,
  PTDR_DIAGONAL = 3,
  PTDR_TRIDIAGONAL = 4,
  PTDR_ANTI_DIAGONAL = 5,
  PTDR_HERMITIAN_TRIDIAGONAL = 6
} ptdr_structure;

typedef enum {
  PTDR_OK = 0,
  PTDR_EINVAL = 1,
  PTDR_EUNSUPPORTED = 2,
  PTDR_ENOMEM = 3,
  PTDR_ECUDA = 4
} ptdr_status;

/* Supported n: dense structures 1 <= n <= 16; DIAGONAL / TRIDIAGONAL / ANTI_DIAGONAL /
 * HERMITIAN_TRIDIAGONAL 1 <= n <= 28. */
int ptdr_max_n(int structure);

/* Number of ptdr_c128 elements of the input A: 4^n (dense), 2^n (DIAGONAL,
 * ANTI_DIAGONAL), 3*2^n (TRIDIAGONAL), 2*2^n (HERMITIAN_TRIDIAGONAL).  0 if (n, structure)
 * is invalid. */
size_t ptdr_input_count(int n, int structure);

/* Number of ptdr_c128 output coefficients: 4^n, 2^n (DIAGONAL, ANTI_DIAGONAL),
 * (n+1)*2^n (TRIDIAGONAL, HERMITIAN_TRIDIAGONAL).  0 if invalid. */
size_t ptdr_output_count(int n, int structure);

/* Device workspace bytes needed by ptdr_decompose_async for (n, structure) on one
 * GPU (world = 1), or per rank of ptdr_decompose_xshard_async (GENERAL, world > 1) or
 * ptdr_decompose_zshard_async (the band structures, world > 1).
 * Deterministic in its arguments.  (size_t)-1 if invalid. */
size_t ptdr_workspace_bytes(int n, int structure, int world);

/* Synchronous convenience: allocates the workspace with cudaMallocAsync on the
 * default stream, runs, synchronizes, frees.  A, out: device pointers. */
ptdr_status ptdr_decompose(const ptdr_c128* A, int n, int structure, ptdr_c128* out);

/* Asynchronous on `stream`.  A: device, ptdr_input_count(n,structure) elements.
 * out: device, ptdr_output_count elements, must not overlap A.  workspace:
 * device, >= ptdr_workspace_bytes(n, structure, 1) bytes, 256-byte aligned,
 * contents ignored on entry and undefined on exit; it must not be used by
 * another call until this call's work on `stream` has completed. */
ptdr_status ptdr_decompose_async(const ptdr_c128* A, int n, int structure, ptdr_c128* out,
                                 void* workspace, size_t ws_bytes, void* stream);

/* In-place decomposition (BASELINE.json configs[4]: "n=16 ... at 1 GPU in-place"): A (device,
 * dense, 4^n elements) is overwritten with its coefficients in the MATRIX LAYOUT
 *   A[z][z ^ x] = alpha(x, z)   (x, z: X- and Z-mask of the string; a bit permutation of
 *                                the q order, Python helper matrix_index),
 * i.e. each coefficient sits where the element A[z][z ^ x] of its XOR-diagonal was.  The
 * X-masks of a pipeline chunk read and write exactly the same elements, so no second
 * 4^n buffer is needed: n = 16 takes 64 GiB + ptdr_inplace_workspace_bytes (2 GiB) on one
 * GPU.  HERMITIAN / REAL_SYMMETRIC read only their triangle as in ptdr_decompose_async and
 * overwrite the whole matrix.  Values are bitwise those of ptdr_decompose_async.
 * workspace: device, 256-byte aligned, not overlapping A. */
size_t ptdr_inplace_workspace_bytes(int n, int structure); /* (size_t)-1 if invalid */
ptdr_status ptdr_decompose_inplace_async(ptdr_c128* A, int n, int structure, void* workspace,
                                         size_t ws_bytes, void* stream);
/* The same matrix layout out of place: out[z][z ^ x] = alpha(x, z), out must not overlap A;
 * workspace as for ptdr_decompose_inplace_async. */
ptdr_status ptdr_decompose_matrix_layout_async(const ptdr_c128* A, int n, int structure, ptdr_c128* out,
                                               void* workspace, size_t ws_bytes, void* stream);

/* End-to-end from HOST memory: copies A_host to the device, decomposes, copies the
 * result to out_host, synchronizes.  Host buffers may be pageable or pinned
 * (pinned is faster).  Allocates and frees its own device buffers. */
ptdr_status ptdr_decompose_host(const ptdr_c128* A_host, int n, int structure,
                                ptdr_c128* out_host);

/* Selected coefficients of a dense GENERAL-storage matrix: out[k] = coefficient of the string
 * with index qs[k] (q order, < 4^n), evaluated directly by Algorithm 2 (compute_coeff,
 * l.302-313) in O(2^n) per string -- no workspace, no full transform.  A: device
 * [2^n][2^n]; qs: device uint64 [count]; out: device [count].  Indices out of range
 * of q are undefined (not checked on the device). */
ptdr_status ptdr_coefficients_async(const ptdr_c128* A, int n, const uint64_t* qs, uint64_t count,
                                    ptdr_c128* out, void* stream);
/* The same on rank `rank`'s X-mask shard A_local (the input of ptdr_decompose_xshard_async,
 * [2^n][2^n / world]): qs are GLOBAL q indices; a string whose X-mask is not in the shard
 * (x >> (n - log2 world) != rank) yields NaN.  bench.py's multi-GPU result check. */
ptdr_status ptdr_coefficients_xshard_async(const ptdr_c128* A_local, int n, int rank, int world,
                                           const uint64_t* qs, uint64_t count, ptdr_c128* out, void* stream);

/* Batched small matrices (serving many decompositions per launch): A = [batch][2^n][2^n]
 * dense matrices of one structure stored back to back, out = [batch][4^n] coefficient
 * arrays in q order; 1 <= n <= 10 (the whole-vector and direct kernels: no workspace, one
 * launch -- two for HERMITIAN / REAL_SYMMETRIC at n >= 9 -- for the whole batch; batch = 0
 * is a no-op and accepts null pointers).  Each
 * matrix's result is bitwise identical to ptdr_decompose_async on it alone. */
ptdr_status ptdr_decompose_batched_async(const ptdr_c128* A, int n, int structure, uint64_t batch,
                                         ptdr_c128* out, void* stream);

/* Zero padding ("we can use a zero padding to make any size of matrix
 * fit this constraint"): A is an m x m matrix of a dense structure stored row-major with
 * row pitch lda >= m (elements); it is decomposed as the top-left block of a 2^n x 2^n
 * zero matrix, n = max(1, ceil(log2 m)), and out receives the 4^n coefficients in q order.
 * GENERAL matrices on the TMA pipeline (n >= 11) are read in place (out-of-bounds boxes
 * are zero-filled by the TMA unit); everything else is first copied into a zero-padded
 * workspace buffer.  m = 0 (empty) is EINVAL.  workspace >= ptdr_padded_workspace_bytes. */
size_t ptdr_padded_workspace_bytes(uint64_t m, int structure); /* (size_t)-1 if invalid */
ptdr_status ptdr_decompose_padded_async(const ptdr_c128* A, uint64_t m, uint64_t lda,
                                        int structure, ptdr_c128* out, void* workspace,
                                        size_t ws_bytes, void* stream);

/* Multi-GPU, per rank, GENERAL only, after the caller's all-to-all (DESIGN.md
 * "Multi-GPU").  world = 2^g GPUs, R = 2^n / world.  Rank `rank` owns the X-masks
 * x with x >> (n-g) == rank.  A_local: device [2^n][R] row-major with
 * A_local[i][c] = A[i][((i >> (n-g)) ^ rank) * R + c].  out_local: device
 * 4^n / world coefficients: the q-ordered subsequence of rank's strings, i.e.
 * out_local[zt * 4^(n-g) + (q mod 4^(n-g))] for the string (x, z) with
 * zt = z >> (n-g).  Requires n - g >= 4. */
ptdr_status ptdr_decompose_xshard_async(const ptdr_c128* A_local, int n, int rank, int world,
                                        ptdr_c128* out_local, void* workspace, size_t ws_bytes,
                                        void* stream);
/* The same, with the pipeline kernel limited to max_ctas persistent CTAs (0 = one per SM):
 * the SMs left free let a concurrent collective on another stream (the next sub-range's
 * all-to-all) run beside the decomposition instead of after it.
 * Results do not depend on max_ctas. */
ptdr_status ptdr_decompose_xshard_ex_async(const ptdr_c128* A_local, int n, int rank, int world,
                                           ptdr_c128* out_local, void* workspace, size_t ws_bytes,
                                           int max_ctas, void* stream);

/* Matrix-free input ("no need to store the input matrix ... from a
 * function"): the GENERAL matrix of the seeded generator (ptdr_generate_dense_async,
 * variant 0, seed `seed`) is decomposed without being stored -- phase A of the pipeline
 * computes A[i][i ^ x] itself.  world = 1: out_local = all 4^n coefficients in q order;
 * world = 2^g > 1: rank `rank`'s X-mask shard in the layout of ptdr_decompose_xshard_async,
 * with no communication at all (needs n - g >= 11).  Bitwise identical to decomposing the
 * stored matrix.  workspace >= ptdr_generated_workspace_bytes(n, world) ((size_t)-1 if
 * invalid); small n (no pipeline) generates into the workspace first. */
size_t ptdr_generated_workspace_bytes(int n, int world);
ptdr_status ptdr_decompose_generated_async(int n, uint64_t seed, int rank, int world,
                                           ptdr_c128* out_local, void* workspace, size_t ws_bytes,
                                           void* stream);

/* Multi-GPU, per rank, GENERAL, fused exchange ("peer pull"):
 * instead of an all-to-all, the phase-A tiles of rank `rank`'s X-masks are loaded by TMA
 * straight from the row-block shard of the rank that owns the rows, over NVLink.
 * shards: HOST array of `world` device pointers (2, 4 or 8 ranks), shards[r] = rows
 * [r R, (r+1) R) of A, row-major with row pitch 2^n (R = 2^n / world), each readable from
 * this GPU (its own allocation, or a peer's opened with ptdr_ipc_open).  The shards must
 * stay unmodified until the call's work on `stream` completes (and on the peers' side
 * until every rank has finished: the caller synchronises, e.g. with a barrier).
 * out_local: same layout as ptdr_decompose_xshard_async.  workspace: as for
 * ptdr_workspace_bytes(n, GENERAL, world).  Requires n - log2(world) >= 11 (EUNSUPPORTED
 * otherwise).  Bitwise identical to the all-to-all path. */
ptdr_status ptdr_decompose_peer_async(const ptdr_c128* const* shards, int n, int rank, int world,
                                      ptdr_c128* out_local, void* workspace, size_t ws_bytes,
                                      void* stream);
/* CUDA IPC of a shard allocation between the ranks' processes (thin wrappers of
 * cudaIpcGetMemHandle / cudaIpcOpenMemHandle / cudaIpcCloseMemHandle): the handle is an
 * opaque blob of ptdr_ipc_handle_size() bytes naming the whole allocation that contains
 * dev_ptr, and *offset is dev_ptr's byte offset inside it; the peer adds the offset to
 * the pointer ptdr_ipc_open returns.  The caller exchanges handle and offset. */
size_t ptdr_ipc_handle_size(void);
ptdr_status ptdr_ipc_get_handle(const void* dev_ptr, void* handle, uint64_t* offset);
ptdr_status ptdr_ipc_open(const void* handle, void** dev_ptr);
ptdr_status ptdr_ipc_close(void* dev_ptr);

/* Multi-GPU, per rank, the band structures DIAGONAL / TRIDIAGONAL / ANTI_DIAGONAL /
 * HERMITIAN_TRIDIAGONAL (replicated band,
 * z-sharded output, no communication).  Every rank holds the whole band (input layout as
 * for ptdr_decompose_async) and writes the z-slice z in [rank 2^(n-g), (rank+1) 2^(n-g))
 * of every output block, world = 2^g <= 2^n: out_local has ptdr_output_count(n, s) / world
 * elements, block-major, out_local[b * 2^(n-g) + (z - rank 2^(n-g))] = coefficient
 * (block b, z) of ptdr_decompose_async's output.  Results are bitwise identical to the
 * one-GPU path (same WHT schedule).  workspace >= ptdr_workspace_bytes(n, s, world). */
ptdr_status ptdr_decompose_zshard_async(const ptdr_c128* band, int n, int structure, int rank,
                                        int world, ptdr_c128* out_local, void* workspace,
                                        size_t ws_bytes, void* stream);

/* ---- BAND(s): (2s+1)-band matrices (Table I l.500-518) -----------
 * Input diags: device [2s+1][2^n], row d+s holds the d-th diagonal D_d[i] = A[i][i+d],
 * d in [-s, s] (entries with i+d outside [0, 2^n) are ignored).  The coefficients can be
 * nonzero only for the X-masks X_s = {0} U {i ^ (i+d) : 1 <= d <= s}, |X_s| = s n - c(s)
 * (Table I); ptdr_band_xmasks lists them in ascending order, which is the block order of
 * the output: out[b * 2^n + z] = coefficient of the string with X-mask xs[b] and Z-mask z
 * (ascending z = ascending q within the block).  s = 0 is the diagonal, s = 1 the
 * tridiagonal band (same values as DIAGONAL / TRIDIAGONAL).  Valid: 1 <= n <= 28,
 * 0 <= s <= 64, s < 2^n. */
size_t ptdr_band_xmask_count(int n, int s); /* 0 if invalid */
ptdr_status ptdr_band_xmasks(int n, int s, uint64_t* xs_host, size_t cap);
size_t ptdr_band_workspace_bytes(int n, int s); /* (size_t)-1 if invalid */
/* workspace: device, >= ptdr_band_workspace_bytes, 256-byte aligned, disjoint from the
 * operands; out: ptdr_band_xmask_count(n, s) * 2^n elements. */
ptdr_status ptdr_decompose_band_async(const ptdr_c128* diags, int n, int s, ptdr_c128* out,
                                      void* workspace, size_t ws_bytes, void* stream);

/* ---- Decomposition algebra and the inverse transform (Sec. IV-B, l.521-627) ----
 * All coefficient arrays are device complex128 in q order.  A new leftmost qubit makes
 * the output four consecutive blocks of 4^n, one per leading letter I, X, Y, Z. */

/* Inverse transform A = sum_P alpha_P P (l.116-121): dense row-major A [2^n][2^n] from the
 * 4^n q-ordered coefficients.  Same path as the decomposition run backwards (per X-mask:
 * conjugate phase, WHT over z, XOR scatter into rows): n >= 11 is one launch of the dense TMA
 * pipeline whose phase A reads q-order boxes (W^2 consecutive q each) and whose phase B stores
 * the XOR-diagonals into A's rows; smaller n a multi-pass kernel.  workspace >=
 * ptdr_reconstruct_workspace_bytes(n) (the pipeline's scratch, <= 2 GiB + counters, for
 * n >= 11; 16 * 4^n bytes below), 256-byte aligned; coeffs, A, workspace disjoint. */
size_t ptdr_reconstruct_workspace_bytes(int n);
ptdr_status ptdr_reconstruct_async(const ptdr_c128* coeffs, int n, ptdr_c128* A, void* workspace,
                                   size_t ws_bytes, void* stream);
/* Inverse transform from the matrix layout (l.116-121): A[i][i ^ x] = sum_z (-1)^{z.i}
 * (-i)^{popcount(x & z)} M[z][z ^ x], where M[z][z ^ x] = alpha(x, z) is the layout
 * ptdr_decompose_inplace_async / ptdr_decompose_matrix_layout_async write (so
 * reconstruct_matrix_layout(decompose_inplace(A)) = A up to rounding).  M, A: device
 * [2^n][2^n] row-major; A == M runs in place (every XOR-diagonal is read before it is
 * written); any other overlap is PTDR_EUNSUPPORTED.  Sizes with the TMA pipeline (n >= 11)
 * run the forward pipeline with the phase applied on input (one launch, no copy); smaller
 * sizes permute M to q order in the workspace and call the q-order inverse.  workspace:
 * device, >= ptdr_reconstruct_matrix_layout_workspace_bytes(n), 256-byte aligned, disjoint
 * from M and A.  n in 1..16; (size_t)-1 for invalid n. */
size_t ptdr_reconstruct_matrix_layout_workspace_bytes(int n);
ptdr_status ptdr_reconstruct_matrix_layout_async(const ptdr_c128* M, int n, ptdr_c128* A, void* workspace,
                                                 size_t ws_bytes, void* stream);
/* Linear combination (l.570-577): out = mu x + nu y elementwise over `count` coefficients
 * (decomposition of mu A + nu B from those of A and B).  out may alias x or y. */
ptdr_status ptdr_axpby_async(ptdr_c128* out, double mu_re, double mu_im, const ptdr_c128* x,
                             double nu_re, double nu_im, const ptdr_c128* y, size_t count,
                             void* stream);
/* Block diagonal diag(A_0, ..., A_{2^k-1}) (l.524-568; k = 1 is the direct sum A_0 (+) A_1,
 * l.537-540): blocks = [2^k][4^n] coefficient arrays of the A_j (A_j occupies rows and
 * columns [j 2^n, (j+1) 2^n)); out = [4^(n+k)].  The output strings whose k leading letters
 * are in {I, Z} with Z-mask zt carry 2^-k sum_j (-1)^{popcount(j & zt)} alpha_j; all others
 * are 0.  1 <= k <= 4, n + k <= 16. */
ptdr_status ptdr_block_diag_async(const ptdr_c128* blocks, int n, int k, ptdr_c128* out,
                                  void* stream);
/* Hermitian augmentation [[0, A^*], [A, 0]] = X (x) Re A + Y (x) Im A (l.590-627): out =
 * [4^(n+1)] with the X block = Re alpha, the Y block = Im alpha (imaginary parts exactly 0),
 * I and Z blocks 0. */
ptdr_status ptdr_hermitian_augment_async(const ptdr_c128* coeffs, int n, ptdr_c128* out,
                                         void* stream);

/* Seeded counter-based generator (the paper fixes no
 * distribution, "a generic matrix", l.631).  Writes rows [row0, row0+nrows) of the
 * dense variant (0 GENERAL, 1 HERMITIAN, 2 REAL_SYMMETRIC) into A (row-major,
 * nrows x 2^n), entry = Philox4x32-10(counter = global element index) + Box-Muller.
 * Bitwise independent of the row split (any sharding sees the same matrix).
 * fro2_partials (nullable, device, ptdr_fro2_partial_count() doubles, 8-byte aligned):
 * per-block partial sums of |a|^2 over the written elements -- their sum is ||A_rows||_F^2,
 * the right-hand side of Parseval (Theorem 1, l.98-114: sum_P |alpha_P|^2 = ||A||_F^2 / 2^n)
 * without another pass over A.  Deterministic; unused entries are 0. */
size_t ptdr_fro2_partial_count(void);
ptdr_status ptdr_generate_dense_async(int n, uint64_t seed, int variant, uint64_t row0,
                                      uint64_t nrows, ptdr_c128* A, double* fro2_partials, void* stream);

/* Same generator for the band inputs: variant 3 (DIAGONAL) writes d[2^n] into
 * band; variant 4 (TRIDIAGONAL) writes the [3][2^n] sub/main/sup array (sub[0] and
 * sup[2^n-1] written as 0); variant 6 (HERMITIAN_TRIDIAGONAL) writes [main | sup] of the
 * same real symmetric matrix.  fro2_partials: as above, over the matrix's entries (variant 6
 * counts the implied sub-diagonal). */
ptdr_status ptdr_generate_band_async(int n, uint64_t seed, int variant, ptdr_c128* band,
                                     double* fro2_partials, void* stream);

/* Same generator, but writes the send layout of the multi-GPU all-to-all for rank `rank`
 * of `world` (R = 2^n / world), split into `subranges` = K (a power of two) sub-ranges of
 * every rank's X-masks so the exchange of one sub-range can overlap the decomposition of
 * the previous one.  Layout [K][world][K][R'][R'], R' = R / K:
 * element (s, h, t, r', c') = A[(rank K + t) R' + r'][((rank ^ h) K + (t ^ s)) R' + c'].
 * Slice s is one equal-split all-to-all; afterwards rank h holds, as a [2^n][R'] row-major
 * array, exactly the A_local of ptdr_decompose_xshard_async(rank' = h K + s,
 * world' = world K).  K = 1: send[h][r][c] = A[rank R + r][(rank ^ h) R + c].
 * fro2_partials: as above, over the rank's row block. */
ptdr_status ptdr_generate_sendblocks_async(int n, uint64_t seed, int rank, int world, int subranges,
                                           ptdr_c128* send, double* fro2_partials, void* stream);

/* Parseval's left-hand side: partials (device, ptdr_fro2_partial_count() doubles) receive
 * per-block sums of |x_e|^2 over the `count` elements of x (deterministic). */
ptdr_status ptdr_sumsq_async(const ptdr_c128* x, uint64_t count, double* partials, void* stream);

/* ---- Host plans: streaming decomposition of matrices held in HOST memory ----------------
 * A plan owns `depth` (1..4) slots of device buffers for one (n, structure) -- input,
 * output and workspace, ~2 x 16 x 4^n bytes per slot for dense structures -- plus three
 * CUDA streams (host->device copy, kernels, device->host copy).  Every step of the
 * decomposition runs on the device exactly as in ptdr_decompose_async; the plan only
 * orders the copies around it.  Call k uses slot k mod depth: its H2D waits until the
 * slot's previous D2H has finished, its kernels wait for its H2D, its D2H for its kernels.
 * With depth >= 2 the H2D of one call overlaps the D2H of the previous one (full-duplex
 * PCIe), so a sequence of matrices streams at the bidirectional copy rate.
 * Host buffers should be pinned (cudaHostAlloc / torch pin_memory); pageable buffers
 * work but the copies then serialise.  The caller must not modify A_host or read
 * out_host of a call until ptdr_plan_wait() has returned after it.  A plan is used on
 * the device that was current at creation (EINVAL otherwise) and by one host thread at
 * a time.  Errors: EINVAL (bad n / structure / depth / pointer), ENOMEM (device
 * allocation), ECUDA. */
typedef struct ptdr_plan_s* ptdr_plan;
ptdr_status ptdr_plan_create(int n, int structure, int depth, ptdr_plan* plan);
/* Enqueue one decomposition: out_host <- decomposition of A_host (returns immediately). */
ptdr_status ptdr_plan_decompose_host_async(ptdr_plan plan, const ptdr_c128* A_host,
                                           ptdr_c128* out_host);
/* Block until every call enqueued on the plan has completed (copies included). */
ptdr_status ptdr_plan_wait(ptdr_plan plan);
/* Kernel launches enqueued by the plan's most recent call. */
int ptdr_plan_launch_count(ptdr_plan plan);
/* Waits for outstanding work, then frees the plan's buffers and streams (NULL: no-op). */
ptdr_status ptdr_plan_destroy(ptdr_plan plan);

/* Number of kernel launches the last successful call on this host thread enqueued
 * (used by bench.py's gpu_launches count). */
int ptdr_last_launch_count(void);

const char* ptdr_status_string(int status);
const char* ptdr_last_error(void); /* thread-local detail of the last failure */
int ptdr_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PTDR_H_ */
