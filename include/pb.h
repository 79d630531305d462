/* pb.h — C ABI of libpb, the B200-native PolyBench hot path.
 *
 * What the boundary is. The paper (arXiv 2312.13170, /root/reference/PAPER.md)
 * speeds up the SYCL-Bench "polybench" nd-range kernels in which each
 * work-item runs an inner loop over global memory (§VI-C
 * "Loop Internalization", Listings 8-9 at PAPER.md:394-428
 * §VI-B "Detect Reduction"; kernel list PAPER.md:522-526 §VIII). Each entry
 * point below is one of those kernels; its arguments follow the PolyBench/C 4.2
 * problem statement (reading R1 in DESIGN.md), i.e. the same argument order as
 * PolyBench's kernel_<name>(...).
 *
 * Conventions (all entry points):
 *  - Matrices are fp32 IEEE-754, row-major, contiguous (row pitch == #cols).
 *    Vectors are contiguous fp32.
 *  - Every float* / const float* is a DEVICE pointer on the current CUDA device
 *    (cudaPointerGetAttributes must report cudaMemoryTypeDevice), 16-byte
 *    aligned. Every matrix column count must be a multiple of 4 (TMA and
 *    128-bit access stride rule); row counts are unrestricted (>= 1).
 *    Violations -> PB_ERR_UNSUPPORTED (alignment) / PB_ERR_INVALID_ARG.
 *  - Outputs must not overlap inputs or each other (the paper's alias
 *    concern, turned into a checked
 *    precondition) -> PB_ERR_ALIAS. In/out arrays (C of gemm/syrk/syr2k, D of
 *    2mm, x1/x2 of mvt) are read then written in place.
 *  - ws / ws_bytes: caller-owned device workspace, at least
 *    pb_workspace_size(...) bytes, 256-byte aligned; the library allocates
 *    nothing on the call path -> PB_ERR_WORKSPACE if too small.
 *  - stream: a cudaStream_t (NULL = legacy default stream). All work is
 *    enqueued on it; no call synchronises the host. Kernel faults surface at
 *    the caller's next synchronisation.
 *  - Validation happens before anything is enqueued: on any error other than
 *    PB_ERR_CUDA nothing was launched and no output was touched.
 *  - Reentrant; concurrent calls on different streams are independent.
 *  - No C++ exception crosses this ABI; pb_last_error() returns a
 *    thread-local message describing the last failing call.
 *
 * Precision: the dense contractions (gemm/2mm/3mm/syrk/syr2k and the X^T X core
 * of covariance/correlation) run on tcgen05 tensor cores in split 3xTF32
 * (x = hi + lo, acc += hi*hi + hi*lo + lo*hi, fp32 accumulation), the
 * matrix-vector kernels and statistics on CUDA cores in fp32/fp64; every
 * result matches the fp64 oracle within componentwise relative error 1e-4
 * (DESIGN.md "Tolerance").
 */
#ifndef PB_H
#define PB_H
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PB_OK = 0,
  PB_ERR_INVALID_ARG = 1,  /* NULL required pointer, dim <= 0, n < 2 for covariance, host pointer */
  PB_ERR_UNSUPPORTED = 2,  /* pointer not 16-B aligned or a column count not a multiple of 4 */
  PB_ERR_ALIAS = 3,        /* an output range overlaps another argument's range */
  PB_ERR_WORKSPACE = 4,    /* ws NULL / misaligned / smaller than pb_workspace_size */
  PB_ERR_CUDA = 5,         /* a CUDA runtime/driver call or launch failed */
  PB_ERR_NCCL = 6          /* libnccl.so.2 not loadable, or an NCCL call failed */
} pb_status;

typedef struct CUstream_st* pb_stream; /* == cudaStream_t */

const char* pb_status_str(pb_status s);
/* Thread-local detail for the last failing call on this thread ("" if none). */
const char* pb_last_error(void);
/* libpb version string, e.g. "pb 0.1 sm_100a". */
const char* pb_version(void);

/* Workspace bytes needed by `kernel` ("gemm", "2mm", "3mm", "syrk", "syr2k",
 * "covariance", "correlation", "atax", "bicg", "mvt", "gesummv", "conv2d",
 * "conv3d", "fdtd_2d", "gramschmidt") for the dims
 * given in that kernel's argument order (e.g. gemm: {ni, nj, nk}; 2mm:
 * {ni, nj, nk, nl}; 3mm: {ni, nj, nk, nl, nm}; syrk/syr2k: {n, m};
 * covariance/correlation: {m, n}; atax/bicg: {m, n}; mvt/gesummv: {n};
 * conv2d: {ni, nj}; conv3d: {ni, nj, nk}; fdtd_2d: {nx, ny}; gramschmidt: {m, n}).
 * Writes *bytes; PB_ERR_INVALID_ARG on unknown kernel or bad dims. */
pb_status pb_workspace_size(const char* kernel, const long long* dims, int ndims, size_t* bytes);

/* gemm — PAPER.md:394-401 (Listing 8 is alpha=beta=1); PolyBench kernel_gemm.
 *   C[i][j] = beta*C[i][j] + alpha * sum_{k<nk} A[i][k]*B[k][j]
 * C ni x nj (in/out), A ni x nk, B nk x nj. beta == 0 means C is not read
 * (BLAS convention; so NaN/garbage in C is not propagated). Same for the beta
 * of 2mm, syrk, syr2k. */
pb_status pb_gemm(int ni, int nj, int nk, float alpha, float beta, float* C, const float* A,
                  const float* B, void* ws, size_t ws_bytes, pb_stream s);

/* 2mm — PolyBench kernel_2mm (LI applies).
 *   tmp = alpha*A*B;  D = tmp*C + beta*D
 * A ni x nk, B nk x nj, tmp ni x nj (optional output, NULL = not written),
 * C nj x nl, D ni x nl (in/out). */
pb_status pb_2mm(int ni, int nj, int nk, int nl, float alpha, float beta, float* tmp,
                 const float* A, const float* B, const float* C, float* D, void* ws,
                 size_t ws_bytes, pb_stream s);

/* 3mm — PolyBench kernel_3mm.  E = A*B;  F = C*D;  G = E*F
 * A ni x nk, B nk x nj, E ni x nj (out), C nj x nm, D nm x nl, F nj x nl (out),
 * G ni x nl (out). */
pb_status pb_3mm(int ni, int nj, int nk, int nl, int nm, float* E, const float* A, const float* B,
                 float* F, const float* C, const float* D, float* G, void* ws, size_t ws_bytes,
                 pb_stream s);

/* syrk — PolyBench kernel_syrk, LOWER triangle (reading R3):
 *   for j <= i: C[i][j] = beta*C[i][j] + alpha * sum_{k<m} A[i][k]*A[j][k];
 *   strict upper triangle untouched.   C n x n (in/out), A n x m. */
pb_status pb_syrk(int n, int m, float alpha, float beta, float* C, const float* A, void* ws,
                  size_t ws_bytes, pb_stream s);

/* syr2k — PolyBench kernel_syr2k, LOWER triangle (reading R3):
 *   for j <= i: C[i][j] = beta*C[i][j] + alpha*sum_k (A[j][k]*B[i][k] + B[j][k]*A[i][k])
 * C n x n (in/out), A, B n x m. */
pb_status pb_syr2k(int n, int m, float alpha, float beta, float* C, const float* A,
                   const float* B, void* ws, size_t ws_bytes, pb_stream s);

/* Full-matrix forms (SYCL-Bench / PolyBench-GPU, reading R3 and SURVEY.md §8(f)
 * NEXT-2): the same sums for EVERY (i, j), C need not be symmetric:
 *   syrk_full:  C[i][j] = beta*C[i][j] + alpha * sum_k A[i][k]*A[j][k]
 *   syr2k_full: C[i][j] = beta*C[i][j] + alpha * sum_k (A[j][k]*B[i][k] + B[j][k]*A[i][k])
 * Workspace names "syrk_full" / "syr2k_full" with dims {n, m}. */
pb_status pb_syrk_full(int n, int m, float alpha, float beta, float* C, const float* A, void* ws,
                       size_t ws_bytes, pb_stream s);
pb_status pb_syr2k_full(int n, int m, float alpha, float beta, float* C, const float* A,
                        const float* B, void* ws, size_t ws_bytes, pb_stream s);

/* covariance — PolyBench kernel_covariance (reading R4; data NOT mutated, R9):
 *   mean[j] = sum_i data[i][j] / float_n;  X = data - mean
 *   cov[i][j] = cov[j][i] = sum_k X[k][i]*X[k][j] / (float_n - 1)
 * data n x m (n observations of m variables), cov m x m (out, exactly
 * symmetric), mean m (optional out). Requires n >= 2. */
pb_status pb_covariance(int m, int n, float float_n, const float* data, float* cov, float* mean,
                        void* ws, size_t ws_bytes, pb_stream s);

/* correlation — PolyBench kernel_correlation (eps rule R5: stddev <= eps -> 1;
 * diagonal exactly 1.0, R6):
 *   stddev[j] = sqrt(sum_i (data[i][j]-mean[j])^2 / float_n)
 *   X = (data - mean) / (sqrt(float_n)*stddev);  corr[i][j] = sum_k X[k][i]*X[k][j]
 * data n x m, corr m x m (out), mean, stddev m (optional outs). */
pb_status pb_correlation(int m, int n, float float_n, float eps, const float* data, float* corr,
                         float* mean, float* stddev, void* ws, size_t ws_bytes, pb_stream s);

/* Row bands of covariance / correlation (multi-GPU: the data replicated on every
 * rank, output rows [r0, r1) per rank, no exchange; SURVEY.md §8(e) "alternative").
 * cov_blk / corr_blk: (r1 - r0) x m, rows r0.. of the full result (both triangles;
 * corr's diagonal entries in the band are exactly 1). r0 a multiple of 128,
 * 0 <= r0 < r1 <= m. Centring by the exact mean first (the long-column path of
 * reading R18), so the band is symmetric with the other ranks' bands only up to
 * rounding (the single call mirrors; bands cannot). mean / stddev (optional) get
 * all m values. ws: pb_workspace_size("covariance_rows" | "correlation_rows",
 * {m, n, r0, r1}). */
pb_status pb_covariance_rows(int m, int n, float float_n, int r0, int r1, const float* data, float* cov_blk,
                             float* mean, void* ws, size_t ws_bytes, pb_stream s);
pb_status pb_correlation_rows(int m, int n, float float_n, float eps, int r0, int r1, const float* data,
                              float* corr_blk, float* mean, float* stddev, void* ws, size_t ws_bytes, pb_stream s);

/* atax — PolyBench kernel_atax:  tmp = A*x;  y = A^T * tmp
 * A m x n, x n, y n (out), tmp m (optional out). */
pb_status pb_atax(int m, int n, const float* A, const float* x, float* y, float* tmp, void* ws,
                  size_t ws_bytes, pb_stream s);

/* bicg — PolyBench kernel_bicg:  s = A^T * r;  q = A * p
 * A n x m, s m (out), q n (out), p m, r n. */
pb_status pb_bicg(int m, int n, const float* A, float* s_out, float* q, const float* p,
                  const float* r, void* ws, size_t ws_bytes, pb_stream s);

/* mvt — PolyBench kernel_mvt:  x1 += A*y_1;  x2 += A^T*y_2
 * A n x n, x1, x2 n (in/out), y_1, y_2 n. */
pb_status pb_mvt(int n, float* x1, float* x2, const float* y_1, const float* y_2, const float* A,
                 void* ws, size_t ws_bytes, pb_stream s);

/* gesummv — PolyBench kernel_gesummv:
 *   tmp = A*x;  y = alpha*tmp + beta*B*x
 * A, B n x n, x n, y n (out), tmp n (optional out). */
pb_status pb_gesummv(int n, float alpha, float beta, const float* A, const float* B, float* tmp,
                     const float* x, float* y, void* ws, size_t ws_bytes, pb_stream s);

/* ------------------------------------------------------------------------
 * Row-block sharding helpers (multi-GPU, one process per GPU).
 * Rank g owns output rows [begin, end). triangular = 0: uniform; 1: balances
 * the area of a lower triangle (boundaries ~ rows*sqrt(g/G)); 2: balances
 * area + 267 * end (syrk/syr2k: a rank also splits rows [0, end) of its
 * operands; the constant is the measured split-row / triangle-element cost
 * ratio). Boundaries are multiples of `align` (except the last, == rows).
 */
pb_status pb_row_partition(int rows, int nranks, int rank, int triangular, int align, int* begin,
                           int* end);

/* Local (per-shard) pieces the Python distributed layer composes with
 * torch.distributed collectives. Row indices are GLOBAL; C/out pointers point
 * at the first row of the caller's row block.
 *
 * pb_syrk_rows / pb_syr2k_rows: rows [r0, r1) of the lower-triangular update
 *   (r0 must be a multiple of 128); A, B are the FULL n x m inputs, C points
 *   to row r0 of C (rows r1-r0, n columns).
 * pb_matvec_partial: for a row block A_blk (rows x cols):
 *   rowdot[i]  = base_row[i] + sum_j A_blk[i][j]*v[j]   (if v; base_row may be NULL = 0,
 *                                                         may equal rowdot: in place)
 *   colpart[j] = base_col[j] + sum_i A_blk[i][j]*w[i]   (if w; w has `rows` entries;
 *                                                         base_col may be NULL)
 *   this is the local half of bicg/mvt/atax before the reduce-scatter. */
pb_status pb_syrk_rows(int n, int m, int r0, int r1, float alpha, float beta, float* C_blk,
                       const float* A, void* ws, size_t ws_bytes, pb_stream s);
pb_status pb_syr2k_rows(int n, int m, int r0, int r1, float alpha, float beta, float* C_blk,
                        const float* A, const float* B, void* ws, size_t ws_bytes, pb_stream s);
pb_status pb_matvec_partial(int rows, int cols, const float* A_blk, const float* v,
                            const float* base_row, float* rowdot, const float* w,
                            const float* base_col, float* colpart, void* ws, size_t ws_bytes,
                            pb_stream s);
/* pb_gesummv_rows: rows of gesummv for a row block: y_blk = alpha*A_blk*x + beta*B_blk*x,
 *   tmp_blk = A_blk*x (optional); A_blk, B_blk are rows x n, x has n entries. */
pb_status pb_gesummv_rows(int rows, int n, float alpha, float beta, const float* A_blk,
                          const float* B_blk, float* tmp_blk, const float* x, float* y_blk, void* ws,
                          size_t ws_bytes, pb_stream s);
/* workspace for the two helpers above: kernel names "syrk_rows" {n,m,r0,r1},
 * "syr2k_rows" {n,m,r0,r1}, "matvec_partial" {rows, cols}. */

/* ------------------------------------------------------------------------
 * Multi-GPU entry points. One process per
 * GPU; every kernel shards by OUTPUT ROW BLOCKS and has at most one exchange
 * step, run with NCCL (NVLink/NVSwitch) inside libpb:
 *   gemm, 2mm, syrk, syr2k, gesummv   no exchange
 *   3mm                               all-gather of F (overlapped with E = A B
 *                                     on the comm's own stream)
 *   atax, bicg, mvt                   reduce-scatter of the transposed-product
 *                                     partial vector
 * libnccl.so.2 is resolved with dlopen at the first pb_comm_* call (env
 * PB_NCCL_LIB overrides the name), so libpb loads without NCCL; PB_ERR_NCCL if
 * it cannot be loaded or an NCCL call fails (message in pb_last_error()).
 *
 * Partitions (rank g's block = pb_row_partition(rows, nranks, g, tri, align)):
 *   gemm/2mm/3mm rows of ni, and 3mm's rows of F/C (nj): tri 0, align 128
 *   syrk/syr2k rows of C (n): tri 2, align 256
 *   atax/bicg/mvt/gesummv rows of A, and the reduce-scatter destinations
 *   (atax y over n, bicg s over m, mvt x2 over n): tri 0, align 4
 * "_blk" arguments point at the first row (element) of this rank's block and
 * hold exactly its rows; other arrays are full and replicated on every rank.
 * A rank whose block is empty still takes part in the collectives (its _blk
 * pointers may then be NULL). Dims and scalars are GLOBAL and identical on
 * every rank; calls must be issued in the same order on every rank, one
 * stream sequence per comm at a time (NCCL rule). Workspace: kernel name
 * "<k>_dist" with the kernel's dims followed by {nranks, rank}.
 */
typedef struct pb_comm pb_comm;
/* 128 opaque bytes (an ncclUniqueId) created on one rank; the caller sends
 * them to the other ranks out of band (e.g. torch.distributed). */
pb_status pb_comm_unique_id(unsigned char id[128]);
/* Collective over the nranks processes; binds the comm to the current device
 * and creates its side stream. *out owned by the caller until
 * pb_comm_destroy. */
pb_status pb_comm_init(int nranks, int rank, const unsigned char id[128], pb_comm** out);
pb_status pb_comm_destroy(pb_comm* comm);
pb_status pb_comm_size(const pb_comm* comm, int* nranks, int* rank);

/* Peer-memory collectives (the fused path). A pb_peer is one
 * symmetric device buffer per rank (a 4 KiB header + data_bytes), mapped into
 * every other rank's address space with CUDA IPC: NVLink/NVSwitch P2P between
 * GPUs, or one GPU shared by several processes. A collective is two libpb
 * kernels: push (each rank stores its data straight into the destinations'
 * buffers, then release-stores a per-source flag at system scope) and consume
 * (acquire every flag, then sum the slots in rank order — deterministic — or
 * copy the gathered region out, then ack each source so that the next
 * collective may overwrite its slot). Every wait is bounded: on timeout the
 * status word (pb_peer_status) becomes non-zero instead of hanging. The epoch
 * that orders the collectives lives in device memory, so the calls can be
 * captured into a CUDA graph and replayed.
 *   pb_peer_create: allocates the buffer (cudaMalloc, owned by the pb_peer) and
 *     writes this rank's 64-byte IPC handle; at most 8 ranks.
 *   pb_peer_open: handles = nranks x 64 bytes (every rank's handle, in rank
 *     order, gathered out of band); maps the other ranks' buffers.
 *   pb_peer_reduce_scatter: out_blk = this rank's block (partition tri 0,
 *     align 4) of the element-wise sum over ranks of partial[0, total).
 *     Needs data_bytes >= nranks * max block * 4.
 *   pb_peer_all_gather: every rank's row block send_blk (rows partition tri 0,
 *     align 128, cols floats per row) -> the full rows x cols array recv on
 *     every rank (send_blk may point into recv). Needs data_bytes >= rows*cols*4.
 *   pb_comm_attach_peer: the comm's dist entry points then use the peer
 *     collectives instead of NCCL (3mm's all-gather on the comm's side stream).
 *   pb_comm_init_local: a comm without NCCL (collectives only via an attached
 *     peer group), e.g. several processes sharing one GPU.
 * Destroy a peer group only after every rank finished using it (barrier). */
typedef struct pb_peer pb_peer;
pb_status pb_peer_create(int nranks, int rank, size_t data_bytes, pb_peer** out, unsigned char handle[64]);
pb_status pb_peer_open(pb_peer* peer, const unsigned char* handles);
pb_status pb_peer_destroy(pb_peer* peer);
pb_status pb_peer_status(const pb_peer* peer, unsigned* status);
pb_status pb_peer_reduce_scatter(pb_peer* peer, const float* partial, float* out_blk, int total, pb_stream s);
pb_status pb_peer_all_gather(pb_peer* peer, const float* send_blk, float* recv, int rows, int cols,
                             pb_stream s);
pb_status pb_comm_attach_peer(pb_comm* comm, pb_peer* peer);
pb_status pb_comm_init_local(int nranks, int rank, pb_comm** out);

/* C_blk = beta*C_blk + alpha*A_blk*B.  A_blk rows x nk, B nk x nj, C_blk rows x nj. */
pb_status pb_gemm_dist(pb_comm* comm, int ni, int nj, int nk, float alpha, float beta, float* C_blk,
                       const float* A_blk, const float* B, void* ws, size_t ws_bytes, pb_stream s);
/* tmp_blk = alpha*A_blk*B (optional out);  D_blk = tmp_blk*C + beta*D_blk. */
pb_status pb_2mm_dist(pb_comm* comm, int ni, int nj, int nk, int nl, float alpha, float beta,
                      float* tmp_blk, const float* A_blk, const float* B, const float* C, float* D_blk,
                      void* ws, size_t ws_bytes, pb_stream s);
/* F[rows' of nj] = C_blk*D, all-gathered into the FULL F (nj x nl) on every
 * rank; E_blk = A_blk*B;  G_blk = E_blk*F.  C_blk holds this rank's rows of C
 * (partition of nj). */
pb_status pb_3mm_dist(pb_comm* comm, int ni, int nj, int nk, int nl, int nm, float* E_blk,
                      const float* A_blk, const float* B, float* F, const float* C_blk,
                      const float* D, float* G_blk, void* ws, size_t ws_bytes, pb_stream s);
/* Lower-triangle rows of this rank (tri partition); A (and B) FULL n x m. */
pb_status pb_syrk_dist(pb_comm* comm, int n, int m, float alpha, float beta, float* C_blk,
                       const float* A, void* ws, size_t ws_bytes, pb_stream s);
pb_status pb_syr2k_dist(pb_comm* comm, int n, int m, float alpha, float beta, float* C_blk,
                        const float* A, const float* B, void* ws, size_t ws_bytes, pb_stream s);
/* tmp_blk = A_blk*x (optional out); y = sum over ranks of A_blk^T tmp_blk,
 * reduce-scattered: y_blk = this rank's block of y (partition of n). */
pb_status pb_atax_dist(pb_comm* comm, int m, int n, const float* A_blk, const float* x, float* y_blk,
                       float* tmp_blk, void* ws, size_t ws_bytes, pb_stream s);
/* A n x m by rows: q_blk = A_blk*p;  s = A^T r reduce-scattered into s_blk
 * (partition of m); r_blk = this rank's rows of r. */
pb_status pb_bicg_dist(pb_comm* comm, int m, int n, const float* A_blk, float* s_blk, float* q_blk,
                       const float* p, const float* r_blk, void* ws, size_t ws_bytes, pb_stream s);
/* x1_blk += A_blk*y_1;  x2 += A^T y_2 with x2_blk / y_2_blk this rank's blocks
 * (same partition as A's rows). */
pb_status pb_mvt_dist(pb_comm* comm, int n, float* x1_blk, float* x2_blk, const float* y_1,
                      const float* y_2_blk, const float* A_blk, void* ws, size_t ws_bytes,
                      pb_stream s);
/* y_blk = alpha*A_blk*x + beta*B_blk*x; tmp_blk = A_blk*x (optional). */
pb_status pb_gesummv_dist(pb_comm* comm, int n, float alpha, float beta, const float* A_blk,
                          const float* B_blk, float* tmp_blk, const float* x, float* y_blk, void* ws,
                          size_t ws_bytes, pb_stream s);

/* Covariance / correlation with the OBSERVATIONS split over ranks (SURVEY.md §8(e) /
 * S17; BASELINE north_star: "an allreduce of column sums for covariance/correlation";
 * definitions as pb_covariance / pb_correlation, PolyBench/C 4.2, readings R4-R6, R17).
 * data_blk = this rank's observations: rows block(n, nranks, rank, tri 0, align 32) of
 * data (n x m), i.e. (o1 - o0) x m. Steps: fp64 column sums S1, S2 of the block ->
 * all-gather of every rank's sums, added in rank order on every rank (the allreduce; all
 * ranks hold the same bits) -> mean = S1 / float_n, stddev from (S2 - 2 mean S1 + n mean^2)
 * / float_n with the eps rule -> the centred (correlation: normalised) block, transposed ->
 * its partial Gram on tcgen05 (pb_syrk_full, 3xTF32, full square) -> reduce-scatter of the
 * m x m sum into row bands -> 1/(float_n - 1) (covariance) or diagonal := 1 (correlation).
 * cov_blk / corr_blk: rows block(m, nranks, rank, tri 0, align 32) of the result (r1 - r0
 * rows of m floats). mean / stddev: optional, FULL m vectors, written on every rank.
 * The two triangles of the result are computed by different tiles and summed over ranks:
 * symmetric to rounding, not bitwise (the single-GPU call mirrors, bitwise).
 * Errors as pb_covariance; m % 4 == 0; workspace "covariance_dist" / "correlation_dist"
 * {m, n, nranks, rank}. */
pb_status pb_covariance_dist(pb_comm* comm, int m, int n, float float_n, const float* data_blk,
                             float* cov_blk, float* mean, void* ws, size_t ws_bytes, pb_stream s);
pb_status pb_correlation_dist(pb_comm* comm, int m, int n, float float_n, float eps,
                              const float* data_blk, float* corr_blk, float* mean, float* stddev,
                              void* ws, size_t ws_bytes, pb_stream s);

/* ------------------------------------------------------------------------
 * Paper ablation: the GEMM of PAPER.md Listing 8
 * (variant 0: one thread per C[i][j], k-loop over global memory, C updated in
 * global memory each iteration) and its loop-internalised form, Listing 9
 * (variant 1: M x M local tiles, two barriers per tile step, M = 16);
 * variant 2 = Listing 9 plus detect-reduction (register accumulator,
 * PAPER.md Listing 5). All plain fp32 SIMT with pb_gemm's semantics.
 * Variant 3 = the production 3xTF32 tcgen05 path (== pb_gemm).
 */
pb_status pb_gemm_variant(int variant, int ni, int nj, int nk, float alpha, float beta, float* C,
                          const float* A, const float* B, void* ws, size_t ws_bytes, pb_stream s);

/* ------------------------------------------------------------------------
 * SYCL-Bench polybench stencils. PAPER.md:524 (§VIII
 * "Evaluation") lists "2D Convolution", "3D Convolution" and "FDTD2D" among the
 * polybench benchmarks it measures, at problem size 1024 (3D Convolution,
 * FDTD2D) and 4096 (2D Convolution); it gives no bodies, so the definitions are
 * readings R19-R21 in DESIGN.md. All arrays row-major fp32 device memory,
 * 16-byte aligned, innermost extent a multiple of 4.
 *
 * conv2d (R19) — 3x3 weighted stencil (cross-correlation) over the interior:
 *   B[i][j] = sum_{di,dj in -1..1} w[(di+1)*3 + (dj+1)] * A[i+di][j+dj]
 *   for 1 <= i <= ni-2, 1 <= j <= nj-2. Border entries of B are not written.
 * A, B ni x nj (B out; must not overlap A). w: HOST pointer to 9 floats, read
 * during the call (copied into the kernel parameters; the caller may reuse it on
 * return). The SYCL-Bench / PolyBench-GPU kernel is w = {0.2, 0.5, -0.8,
 * -0.3, 0.6, -0.9, 0.4, 0.7, 0.1}. No workspace. ni or nj < 3: nothing to do. */
pb_status pb_conv2d(int ni, int nj, const float* w, const float* A, float* B, pb_stream s);

/* conv3d (R20) — 3x3x3 weighted stencil over the interior of ni x nj x nk
 * (k fastest):
 *   B[i][j][k] = sum_{di,dj,dk in -1..1} w[(di+1)*9 + (dj+1)*3 + (dk+1)] * A[i+di][j+dj][k+dk]
 *   for 1 <= i <= ni-2, 1 <= j <= nj-2, 1 <= k <= nk-2; border entries not written.
 * w: HOST pointer to 27 floats (the PolyBench-GPU 3DConvolution is 11 nonzero
 * taps: its 15 source terms with equal offsets added, R20). Requires
 * nk % 4 == 0, ni*nj <= 2^31. No workspace. */
pb_status pb_conv3d(int ni, int nj, int nk, const float* w, const float* A, float* B, pb_stream s);

/* fdtd_2d (R21) — PolyBench/C 4.2 kernel_fdtd_2d, argument order as there:
 *   for t < tmax:  ey[0][j] = fict[t];
 *                  ey[i][j] -= 0.5f*(hz[i][j] - hz[i-1][j])         (i >= 1)
 *                  ex[i][j] -= 0.5f*(hz[i][j] - hz[i][j-1])         (j >= 1)
 *                  hz[i][j] -= 0.7f*(ex[i][j+1] - ex[i][j] + ey[i+1][j] - ey[i][j])
 *                                                                   (i < nx-1, j < ny-1)
 * ex, ey, hz nx x ny (in/out, distinct), fict tmax floats (device; may be NULL
 * when tmax == 0). Every update is evaluated with the statement's fp32
 * operations in C order (no contraction), so the result is bitwise that of the
 * sequential PolyBench sweeps in fp32. ws: pb_workspace_size("fdtd_2d",
 * {nx, ny}) bytes. When every 64 x 128 tile fits on the GPU at once (nx * ny up to
 * ~148 tiles), one persistent cooperative launch (state in shared memory, 8 steps
 * per neighbour exchange through the workspace); otherwise one launch per time
 * step with the fields ping-ponging through the workspace (+3 device copies when
 * tmax is odd). */
pb_status pb_fdtd_2d(int tmax, int nx, int ny, float* ex, float* ey, float* hz, const float* fict, void* ws,
                     size_t ws_bytes, pb_stream s);

/* Stencil ablation (as pb_gemm_variant for GEMM): variant 0 = the SYCL-Bench kernel
 * shape - one thread per output point, every tap a global load, no staging;
 * variant 1 = pb_conv2d / pb_conv3d. Same arguments and semantics. */
pb_status pb_conv2d_variant(int variant, int ni, int nj, const float* w, const float* A, float* B, pb_stream s);
pb_status pb_conv3d_variant(int variant, int ni, int nj, int nk, const float* w, const float* A, float* B,
                            pb_stream s);

/* gramschmidt (R22) — PolyBench/C 4.2 kernel_gramschmidt (the SYCL-Bench
 * "Gramschmidt" of PAPER.md:524; PAPER.md:551 notes its candidate loop sits in a
 * divergent region). Modified Gram-Schmidt, for k < n:
 *   R[k][k] = sqrt(sum_i A[i][k]^2);  Q[i][k] = A[i][k] / R[k][k];
 *   for j > k:  R[k][j] = sum_i Q[i][k]*A[i][j];  A[i][j] -= Q[i][k]*R[k][j]
 * A m x n (in/out: on return column j holds R[j][j]*Q[:,j], as in PolyBench),
 * R n x n (out; entries below the diagonal are not written), Q m x n (out). All
 * distinct. Computed in fp64 (state and reductions), rounded to fp32 once.
 * Linearly dependent columns give Inf/NaN (division by R[k][k] = 0), as in
 * PolyBench. ws: pb_workspace_size("gramschmidt", {m, n}) bytes. One persistent
 * cooperative kernel (one CTA per SM) plus three transposes; the co-residency
 * of the persistent kernel needs m * ceil(n / #SMs) * 8 <= 200 KiB for the
 * shared-memory path, else its columns stay in the (L2-resident) workspace. */
pb_status pb_gramschmidt(int m, int n, float* A, float* R, float* Q, void* ws, size_t ws_bytes, pb_stream s);

/* Gramschmidt ablation: variant 0 = the PolyBench-GPU / SYCL-Bench kernel shape (three
 * launches per column: a single-thread norm, the column normalisation, one thread per
 * trailing column looping over the rows; fp64 working arrays, same results within
 * R22); variant 1 = pb_gramschmidt. Same arguments and workspace. */
pb_status pb_gramschmidt_variant(int variant, int m, int n, float* A, float* R, float* Q, void* ws, size_t ws_bytes,
                                 pb_stream s);

/* Number of kernels launched by the last successful pb_* call on this thread. */
int pb_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* PB_H */
