/*
 * gls.h -- C ABI of libgls.so: the B200 hot path of HP-GWAS / OOC-HP-GWAS
 * (Fabregat, Aulchenko, Bientinesi; arXiv 1210.7325).
 *
 * The library solves the sequence of generalized least-squares problems
 *
 *     b_i := (X_i^T M^{-1} X_i)^{-1} X_i^T M^{-1} y,      1 <= i <= m          (Eq. (1))
 *
 * with X_i = (X_L | X_Ri): X_L (n x pL) shared by all problems, X_Ri (n x pR) per problem
 * (PAPER.md:53-54).  M is n x n SPD, X_i full rank, n > p = pL + pR, 1 <= p <= 20
 * (PAPER.md:44-51).
 *
 *   gls_create       -- Alg. 5 lines 1, 2, 4, 5, 6: potrf of M, the shared
 *                       transforms X~_L = L^{-1} X_L, y~ = L^{-1} y, S_TL = X~_L^T X~_L,
 *                       b_T = X~_L^T y~.  Done once, on the GPU.
 *   gls_solve_block  -- Alg. 5 line 3 + lines 7-11 on one block of problems (PAPER.md:314,
 *                       318-322; Alg. 8 lines 9-14): the blocked triangular
 *                       solve of the block's X_R columns fused with the per-problem assembly of
 *                       S_i, b_i (Fig. 1) and the p x p SPD solve.  The whitened
 *                       X~_R is never written to memory.  A host-resident X_R block is streamed
 *                       to the device with double buffering (Alg. 8).
 *
 * All matrices are column-major FP64: element (r, c) of an n x k matrix is at r + c*n (leading
 * dimension = n, no padding).  Problem i of a block uses columns [i*pR, (i+1)*pR) of X_R.
 * Result record i is b_out[i*p .. i*p+p-1]: the pL coefficients of X_L first, then the pR
 * coefficients of X_Ri, following the column order of X_i = (X_L | X_Ri) (reading A3).
 *
 * Pointers may be host or CUDA device pointers (detected with cudaPointerGetAttributes; host
 * memory may be pinned or pageable -- pinned is required for copy/compute overlap).
 *
 * Errors are return codes; nothing is thrown across the ABI.  One context belongs to one CUDA
 * device (the device current at gls_create) and must be used by one host thread at a time.
 */
#ifndef GLS_H_
#define GLS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gls_ctx gls_ctx; /* opaque */

enum {
  GLS_OK = 0,
  GLS_ERR_ARG = 1,     /* NULL pointer where one is required, bad flag value                 */
  GLS_ERR_DIM = 2,     /* dimensions violate n > p, pL >= 0, pR >= 1, p <= 20, m_blk >= 1     */
  GLS_ERR_NOT_SPD = 3, /* M is not SPD: a Cholesky pivot d_j <= 2^-52 * max_k M_kk (reading A5)*/
  GLS_ERR_CUDA = 4,    /* a CUDA runtime/driver call failed; see gls_last_error               */
  GLS_ERR_OOM = 5,     /* device or pinned-host allocation failed                             */
  GLS_ERR_STATE = 6    /* context is in a failed state or not yet committed (adopt mode)      */
};

/* gls_create -- factor M and prepare the shared state (Alg. 5 lines 1,2,4,5,6).
 *   n, pL, pR : dimensions; GLS_ERR_DIM unless n > pL+pR, pL >= 0, pR >= 1, pL+pR <= 20.
 *   M         : n x n, column-major; only the lower triangle (r >= c) is read.
 *   X_L       : n x pL column-major; may be NULL iff pL == 0.
 *   y         : n observations.
 *   out       : receives the context.
 * Ownership: M, X_L, y are copied; the caller may free them on return.  The context owns all
 * device memory it allocates (about 1.6*n^2*8 bytes transiently, 0.5*n^2*8 bytes resident).
 * On GLS_ERR_NOT_SPD (and on any CUDA failure after the dims were validated) *out is set to a
 * context in the failed state: only gls_failed_pivot, gls_last_error and gls_destroy are valid
 * on it.  On GLS_ERR_ARG / GLS_ERR_DIM *out is set to NULL. */
int gls_create(int64_t n, int32_t pL, int32_t pR, const double* M, const double* X_L,
               const double* y, gls_ctx** out);

/* gls_create_async -- gls_create without waiting for the factorisation (Alg. 8 lines 1-5 overlapped
 * with the first async_read of line 7; §4.3 notes that the first block's load is
 * otherwise not overlapped with computation).  Same arguments and the same
 * resulting state, bit for bit.  Every step is enqueued on the context's stream and the call returns
 * before it runs, so a following gls_solve_block* call can start streaming its host X_R block while
 * M is still being factored (its H2D copies do not depend on the setup; its kernels do).
 * Ownership: M, X_L, y are BORROWED until the first synchronising call on the context (a synchronous
 * solve, gls_sync, gls_read_timing, gls_read_stream_report, gls_path_counts, gls_shared_view*,
 * gls_destroy): the host copies read them in stream order.  Host pointers should be pinned.
 * Errors: argument / dimension / allocation errors are returned here as by gls_create.  A non-SPD M
 * is reported by the first synchronising call, which returns GLS_ERR_NOT_SPD (once) and puts the
 * context in the failed state (gls_failed_pivot then holds the index); the b_out of solves enqueued
 * before that call are undefined and must be discarded. */
int gls_create_async(int64_t n, int32_t pL, int32_t pR, const double* M, const double* X_L,
                     const double* y, gls_ctx** out);

/* gls_solve_block -- solve m_blk consecutive problems (Alg. 5 line 3 and lines 7-11; Alg. 8 l.9-14).
 *   X_R   : n x (m_blk*pR) column-major, NOT modified (reading A9: the in-place X_R := L^{-1} X_R of
 *           the paper is never materialised).  Device pointer: read in place.  Host pointer:
 *           streamed through two device staging buffers (Alg. 8 double buffering).
 *   m_blk : number of problems in the block, >= 1.
 *   b_out : m_blk x p, record i at b_out + i*p (host or device).  A RankDeficient problem
 *           (a pivot of its p x p Cholesky <= 1e-10 * S_jj, reading A4) gets a quiet-NaN record;
 *           the other problems are unaffected.
 * Path (GLS_PATH_AUTO): per problem, on the device -- see gls_set_path.  Workspaces (kept by the
 * context, from its stream-ordered pool): two int8 copies of up to 8 waves of X_R columns, one int per
 * problem of the block, and up to 512 MB for the FP64 fallback's gathered columns.
 * Synchronous: returns after b_out is written. */
int gls_solve_block(gls_ctx* ctx, const double* X_R, int64_t m_blk, double* b_out);

/* gls_solve_block_ex -- as gls_solve_block, plus
 *   status_out : NULL, or m_blk int32 (host or device): 0 = OK, 1 = RankDeficient.
 *   async      : 0 = return after b_out/status_out are written; 1 = return after enqueueing
 *                on the context stream (device X_R) or after the last host chunk is enqueued
 *                (host X_R); X_R, b_out and status_out stay borrowed until gls_sync. */
int gls_solve_block_ex(gls_ctx* ctx, const double* X_R, int64_t m_blk, double* b_out,
                       int32_t* status_out, int async);

/* gls_sync -- wait until every enqueued solve of this context has completed. */
int gls_sync(gls_ctx* ctx);

/* gls_set_stream -- run the compute kernels on `stream` (a cudaStream_t of the context's device,
 * e.g. torch.cuda.current_stream().cuda_stream); NULL restores the context's own stream. */
int gls_set_stream(gls_ctx* ctx, void* stream);

/* gls_set_block_cols -- columns per host->device chunk for host-resident X_R (the paper's block
 * size); rounded to whole problems.  Default: 64 * (number of SMs) columns. */
int gls_set_block_cols(gls_ctx* ctx, int64_t cols);

/* gls_destroy -- free everything (NULL is a no-op).  Waits for outstanding work first.  The
 * context's CUDA streams and events go back, idle, to a per-device cache that the next context on
 * that device takes them from (creating and destroying them per context stalled the host for tens of
 * ms now and then; GLS_RES_CACHE=0 turns the cache off). */
void gls_destroy(gls_ctx* ctx);

/* Diagnostics. */
int64_t gls_failed_pivot(const gls_ctx* ctx);  /* 0-based failing pivot of M after NOT_SPD, else -1 */
const char* gls_last_error(const gls_ctx* ctx); /* owned by ctx; "" when no error                  */
const char* gls_error_string(int code);         /* static text for any return code                 */

/* Multi-GPU replicate-then-shard.  The root rank calls
 * gls_create; every other rank calls gls_create_adopt (allocates the shared state, computes
 * nothing), receives the root's buffers listed by gls_shared_view (e.g. an NCCL broadcast over
 * NVLink), then calls gls_commit_shared.  Afterwards all ranks are bitwise identical.
 *   gls_shared_view: ptrs[k] (device pointers, owned by ctx), bytes[k]; *count = number of
 *   buffers (<= 8).  Valid on a committed context (root) and on an adopt-mode context. */
int gls_create_adopt(int64_t n, int32_t pL, int32_t pR, gls_ctx** out);
int gls_shared_view(gls_ctx* ctx, void** ptrs, int64_t* bytes, int32_t* count);
int gls_commit_shared(gls_ctx* ctx);
/* Int8-only replication: gls_create_adopt_int8 allocates only the int8 path's shared state (no packed T
 * for the FP64 kernel -- n^2 * 4 bytes less per GPU, never broadcast); the root lists the matching
 * buffers with gls_shared_view_ex(ctx, GLS_SHARE_INT8_ONLY, ...).  An int8-only context solves genotype
 * codes (gls_solve_block_i8) and integer-valued double X_R (converted on the device; a block holding any
 * other value fails with GLS_ERR_ARG and the call synchronises); gls_set_path(GLS_PATH_FP64) on it is
 * GLS_ERR_STATE.  GLS_ERR_DIM when n > 131071. */
enum { GLS_SHARE_INT8_ONLY = 1 };
int gls_create_adopt_int8(int64_t n, int32_t pL, int32_t pR, gls_ctx** out);
int gls_shared_view_ex(gls_ctx* ctx, int32_t flags, void** ptrs, int64_t* bytes, int32_t* count);

/* Number of kernel launches this context issued so far (evidence counter for bench.py). */
int64_t gls_kernel_launches(const gls_ctx* ctx);

/* Arithmetic path of the trsm (Alg. 5 line 3).  Both give FP64-accurate b.
 *   GLS_PATH_AUTO (default): problems whose pR columns of X_R hold only integers in [-128, 127]
 *     (SNP genotypes) run on the int8 tensor cores with T = L^{-1} split into seven
 *     base-256 digits per element (exact int32 digit products, one rounding of T to 55 bits per
 *     row, reading A15); every other problem runs on the FP64 tensor pipe.  Decided per problem, on
 *     the device (no host synchronisation), so a problem's bits depend only on its own values --
 *     never on its neighbours or the block partition.  Only for n <= 131071.
 *   GLS_PATH_FP64: every block on the FP64 tensor pipe (DMMA).
 * The environment variable GLS_PATH=fp64 sets the default of new contexts. */
enum { GLS_PATH_AUTO = 0, GLS_PATH_FP64 = 1 };
int gls_set_path(gls_ctx* ctx, int32_t path);  /* GLS_ERR_ARG for an unknown path */
/* Evidence: how many int8 and FP64 hot-kernel launches did their work so far (synchronises). */
int gls_path_counts(gls_ctx* ctx, int64_t* int8_launches, int64_t* fp64_launches);

/* gls_solve_block_i8 -- as gls_solve_block_ex, with X_R given as genotype codes: G is n x
 * (m_blk*pR) int8, column-major with leading dimension ldg >= n (element (r, c) at G[r + c*ldg]),
 * each value the exact integer X_R entry (e.g. minor-allele counts 0/1/2).  Always the int8 path
 * (GLS_ERR_DIM when n > 131071).  Device G with ldg % 16 == 0 and a 16-byte aligned base is read
 * in place (no conversion pass); host G is streamed with double buffering (Alg. 8) at one byte
 * per genotype.  Ownership and errors as gls_solve_block_ex; GLS_ERR_ARG if ldg < n. */
int gls_solve_block_i8(gls_ctx* ctx, const int8_t* G, int64_t ldg, int64_t m_blk, double* b_out,
                       int32_t* status_out, int async);

/* Diagnostics for the benchmark: when enabled, every hot-kernel launch (and every int8 conversion
 * pass) is bracketed by CUDA events on the stream it runs on.  gls_read_timing synchronises,
 * returns the summed device milliseconds per kind since the last read, the number of timed
 * launches, and resets. */
int gls_set_timing(gls_ctx* ctx, int32_t enable);
int gls_read_timing(gls_ctx* ctx, double* ms_int8, double* ms_fp64, double* ms_conv, int64_t* launches);

/* Overlap accounting of the host -> HBM stream (Alg. 8; fig:double-buff,
 * PAPER.md:698-704).  When enabled, every host chunk of gls_solve_block[_ex|_i8] with a host X_R is
 * bracketed by CUDA timing events: its H2D copy (h2d stream), its compute (recorded on the compute
 * stream after the two waits of Alg. 8 -- "wait(current X_blk)" and "wait(previous b_blk)" -- have
 * cleared, up to the end of its kernels) and its D2H copy.  gls_read_stream_report synchronises,
 * summarises every chunk since the last read (in issue order), and resets:
 *   wall_ms          first chunk's H2D start -> last event
 *   h2d/compute/d2h  summed busy time of each engine
 *   first_load_ms    the part of the first copy the compute stream waited for: from the later of
 *                    the copy's start and the end of the compute stream's earlier work (e.g. an
 *                    asynchronous gls_create, which hides it) to the first chunk's compute
 *                    (§4.3 warm-up block)
 *   exposed_h2d_ms   compute-stream idle time between chunks while the next X block was still in
 *                    flight (wait(current X_blk) exposed)
 *   exposed_other_ms the rest of the idle time between chunks (wait(previous b_blk), host gaps)
 *   tail_ms          after the last compute (the final D2H)
 * Perfect overlap (the paper's claim) means exposed_h2d_ms + exposed_other_ms ~ 0
 * when compute is the slower engine. */
typedef struct {
  int64_t chunks, h2d_bytes, d2h_bytes;
  double wall_ms, h2d_ms, compute_ms, d2h_ms, first_load_ms, exposed_h2d_ms, exposed_other_ms, tail_ms;
} gls_stream_report;
int gls_set_stream_report(gls_ctx* ctx, int32_t enable);
int gls_read_stream_report(gls_ctx* ctx, gls_stream_report* rep);

/* gls_get_dims -- n, pL, pR of a context (any state but NULL). */
int gls_get_dims(const gls_ctx* ctx, int64_t* n, int32_t* pL, int32_t* pR);

/* gls_release_cached_memory -- return the device memory that destroyed contexts left cached in the
 * current device's stream-ordered pool (up to GLS_POOL_KEEP_BYTES, default 32 GiB, is kept so that
 * create/destroy cycles do not remap pages) to the driver, e.g. before a large allocation by another
 * allocator.  Synchronises the device.  Returns GLS_OK or GLS_ERR_CUDA. */
int gls_release_cached_memory(void);

/* ---- Out-of-core from secondary storage (§4; NEXT-1 / NEXT-4 of SURVEY §8(f)).
 * gls_solve_file streams the X_R of m problems from a file, in blocks of problems, and writes the b
 * records (m x p doubles, record i at byte 8 p i) and optionally the int32 statuses to files.
 *   xr_path, xr_offset : X_R as stored: m*pR columns of n elements, column-major from byte xr_offset;
 *                        elem_bytes 8 = FP64 (gls_solve_block_ex), 1 = int8 genotype codes
 *                        (gls_solve_block_i8)
 *   block_groups       : problems per block (the paper's block size)
 *   warmup_groups      : 0, or a smaller first block (§4.3: "initiate the computation with a small
 *                        block size ... and increase it after a few iterations")
 *   mode               : GLS_OOC_SYNC  -- Alg. 7, blocking read / solve / blocking write per block;
 *                        GLS_OOC_ASYNC -- Alg. 8, two pinned host workspaces (fig:workspaces), a reader
 *                        thread prefetching the next block and a writer thread storing the previous b,
 *                        at most one read and one write in flight.
 *   rep (nullable)     : wall, compute, read-wait and write-wait seconds measured at the algorithms' wait
 *                        points (Alg. 8 lines 8 and 16; Alg. 7 lines 7 and 14), the first block's load,
 *                        blocks and bytes moved.
 * Results are bitwise identical between the two modes and to gls_solve_block on the same values (same
 * kernels, block-partition independent; the int8-or-FP64 choice is made per problem, reading A16).
 * Synchronous: returns when every b is on the file.
 * Errors: GLS_ERR_ARG (bad argument, unreadable/short X_R file, failed write), GLS_ERR_DIM, GLS_ERR_OOM
 * (pinned workspaces), and any error of the solve calls. */
enum { GLS_OOC_SYNC = 0, GLS_OOC_ASYNC = 1 };
typedef struct {
  double wall_s, compute_s, read_wait_s, write_wait_s, first_load_s;
  int64_t blocks, bytes_read, bytes_written;
} gls_ooc_report;
int gls_solve_file(gls_ctx* ctx, const char* xr_path, int64_t xr_offset, int32_t elem_bytes, int64_t m,
                   const char* b_path, const char* status_path, int64_t block_groups, int64_t warmup_groups,
                   int32_t mode, gls_ooc_report* rep);

/* gls_select_block_size -- §4.3's block-size condition: the largest block (problems)
 * whose two workspaces (X_R + b + status, elem_bytes per X_R element) fit in mem_limit_bytes, and
 * *io_bound = 0 if at that size time(compute) >= 1.1 (time(load) + time(store)) with the given
 * rates (compute in problems/s, I/O in bytes/s, io_latency_s per request), else *io_bound = 1.
 * Returns -1 on bad arguments or when not even one problem fits. Pure host arithmetic. */
int64_t gls_select_block_size(int64_t n, int32_t p, int32_t pR, int32_t elem_bytes, int64_t mem_limit_bytes,
                              double compute_groups_per_s, double io_bytes_per_s, double io_latency_s,
                              int32_t* io_bound);

/* ---- GenABEL's gwfgls (Alg. 6) on the B200 kernels: a rung of the algorithm
 * ladder (NEXT-2 of SURVEY §8(f)) kept for Table II's cost comparison, not the hot
 * path.  It follows the listing: M^{-1} explicitly (line 1; here T^T T with T = L^{-1} from this
 * library's potrf + inverse), W_L = M^{-1} X_L (line 2), then per problem w = M^{-1} x_R (line 3:
 * GLS_GWFGLS_GEMV = one gemv per column as listed, GLS_GWFGLS_GEMM = the block's gemvs as one GEMM),
 * S_i = W^T X_i with all p x p entries (line 4), W^T y (line 5) and an LU solve with partial pivoting
 * (line 6; a zero or non-finite pivot => NaN record, status 1).
 *   gls_gwfgls_create: as gls_create (M, X_L, y host or device, copied; GLS_ERR_NOT_SPD if potrf fails).
 *   gls_gwfgls_solve:  X_R (n x m_blk pR, column-major) and b_out (m_blk x p) / status_out (nullable)
 *                      are DEVICE pointers; synchronous.  Errors: GLS_ERR_ARG, GLS_ERR_DIM, GLS_ERR_CUDA. */
typedef struct gls_gwfgls gls_gwfgls;
enum { GLS_GWFGLS_GEMV = 0, GLS_GWFGLS_GEMM = 1 };
int gls_gwfgls_create(int64_t n, int32_t pL, int32_t pR, const double* M, const double* X_L, const double* y,
                      gls_gwfgls** out);
int gls_gwfgls_solve(gls_gwfgls* g, const double* X_R, int64_t m_blk, double* b_out, int32_t* status_out,
                     int32_t mode);
int64_t gls_gwfgls_launches(const gls_gwfgls* g);
void gls_gwfgls_destroy(gls_gwfgls* g);

/* ---- Distributed create: M beyond one GPU (NEXT-3 of SURVEY §8(f); §6).
 * G ranks (one per GPU) each hold the column blocks j (width nb, a multiple of 128) with j % G == rank
 * of M and of T = L^{-1}, and run a right-looking blocked Cholesky fused with the forward substitution
 * that forms T, one panel per block column, then build the int8 path's shared state from the
 * distributed T.  The library computes; the caller moves data between the steps (e.g. torch.distributed
 * over NCCL; paper_1210_7325_b200/multi.py dist_create runs the whole protocol):
 *   for k in 0..K-1:  owner (k % G): gls_dist_step(FACTOR, k)  (GLS_ERR_NOT_SPD: pivot in
 *                                    gls_dist_failed_pivot; every rank must stop)
 *                     broadcast the GLS_DIST_PANEL buffer of k from the owner
 *                     all: gls_dist_step(UPDATE, k)
 *   all: gls_dist_step(PARTIALS);  W = sum over ranks (in rank order) of every rank's GLS_DIST_WPART,
 *        written to GLS_DIST_W;  GLS_DIST_ROWMAX all-reduced with MAX
 *   all: gls_dist_step(PACK);      GLS_DIST_VMAX all-reduced with MAX
 *   all: gls_dist_step(PACK2);     GLS_DIST_T8 and GLS_DIST_V8 all-reduced with SUM (bytes; each byte has
 *                                  exactly one nonzero contributor)
 *   all: gls_dist_finish -> an int8-only context (see gls_create_adopt_int8), identical on every rank.
 * gls_dist_create: M (n x n column-major, host or device; each rank copies its own column blocks),
 * X_L, y as gls_create; GLS_ERR_ARG unless 0 <= rank < nranks and nb is a positive multiple of 128;
 * GLS_ERR_DIM unless the gls_create conditions hold and n <= 131071.  Device memory per rank:
 * 2 n (n / G) 8 bytes for the local blocks of M and T (+ a n x nb panel), plus the int8 state.
 * gls_dist_buffer: device pointer and byte size of a buffer (k: block index for GLS_DIST_PANEL).
 * Every step synchronises.  gls_dist_finish hands the context to the caller (destroy it with
 * gls_destroy); gls_dist_destroy frees the rest. */
typedef struct gls_dist gls_dist;
enum { GLS_DIST_FACTOR = 0, GLS_DIST_UPDATE = 1, GLS_DIST_PARTIALS = 2, GLS_DIST_PACK = 3, GLS_DIST_PACK2 = 4 };
enum { GLS_DIST_PANEL = 0, GLS_DIST_WPART = 1, GLS_DIST_W = 2, GLS_DIST_ROWMAX = 3, GLS_DIST_VMAX = 4,
       GLS_DIST_T8 = 5, GLS_DIST_V8 = 6 };
int gls_dist_create(int64_t n, int32_t pL, int32_t pR, int64_t nb, int32_t nranks, int32_t rank, const double* M,
                    const double* X_L, const double* y, gls_dist** out);
int gls_dist_info(const gls_dist* d, int64_t* nb, int64_t* nblocks, int64_t* nloc);
int gls_dist_buffer(gls_dist* d, int32_t which, int64_t k, void** ptr, int64_t* bytes);
int gls_dist_step(gls_dist* d, int32_t phase, int64_t k);
int gls_dist_finish(gls_dist* d, gls_ctx** out);
int64_t gls_dist_failed_pivot(const gls_dist* d);
int64_t gls_dist_launches(const gls_dist* d);
void gls_dist_destroy(gls_dist* d);

#ifdef __cplusplus
}
#endif

#endif /* GLS_H_ */
