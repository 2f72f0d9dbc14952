/*
 * mcr.h -- C ABI of the B200-native reachability solver (libmcr.so, sm_100a).
 *
 * Drop-in boundary for the solve path of the reference package `mcreach`
 * (/root/reference/pkg/src/mcreach). Every entry point takes plain pointers and sizes;
 * no C++ or torch type crosses it. Host-pointer entry points copy inputs to the device and
 * the result back (what a Python/ctypes caller uses); `*_device` entry points take device
 * pointers on the handle's GPU (inputs already resident in HBM).
 *
 * Reference interface each entry point replaces (file:line in /root/reference/pkg/src/mcreach):
 *   mcr_matrix_create   CsrMatrix + its cached scipy handle      sparse.py:71-98
 *                       diagonal() / _jacobi_diagonal()          sparse.py:194-198, solvers.py:277-282
 *                       without_diagonal() (built lazily)        sparse.py:227-231
 *   mcr_matvec          matvec(a, x)                             sparse.py:184-191
 *   mcr_residual_inf    residual_inf_norm(m, x, b)               solvers.py:123-133
 *   mcr_jacobi          jacobi_solve(m, b, config)               solvers.py:194-230
 *   mcr_bicgstab        bicgstab_solve(m, b, config)             solvers.py:399-426, 450-491
 *   status codes        ZeroDiagonal / NotConverged / Breakdown  solvers.py:43-78
 *
 * Thread safety: calls on one handle are serialised by a per-handle mutex; different handles
 * may be used concurrently. The library owns all device memory of a handle.
 */
#ifndef MCR_H
#define MCR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define MCR_API __attribute__((visibility("default")))
#else
#define MCR_API
#endif

/* Return codes (the Python wrapper maps them onto the reference's exceptions). */
enum {
    MCR_OK = 0,                /* converged; outputs filled                                  */
    MCR_NOT_CONVERGED = 1,     /* NotConverged: outputs hold the last iterate                */
    MCR_BREAKDOWN = 2,         /* Breakdown: outputs hold the snapshot before that iteration */
    MCR_ZERO_DIAGONAL = 3,     /* ZeroDiagonal: report->zero_diagonal_index                  */
    MCR_DIMENSION = 4,         /* malformed CSR / mismatched sizes                           */
    MCR_CUDA_ERROR = 5,        /* CUDA failure; see mcr_last_error()                         */
    MCR_INVALID_ARGUMENT = 6,
    MCR_UNSUPPORTED_INPUT = 7  /* text readers: outside the fast subset (mcr_text_reason())  */
};

/* Breakdown.which of the reference (solvers.py:465-480). */
enum { MCR_BD_NONE = 0, MCR_BD_Y_PREV_W = 1, MCR_BD_Q_V = 2, MCR_BD_T_T = 3 };

/* Device storage selection for mcr_matrix_create. AUTO picks dense 32-row slabs when the
 * matrix is at least 2/3 full and n >= 1024; the band-staged two-pass layout (STAGED) when
 * the gathered vector is far larger than L2 (8 * n >= 80 MB, rows of at most 2048 entries,
 * fewer than 2^31 entries); otherwise CSR, laid out as SELL-32-sigma when the caller asks for
 * it (coalesced thread-per-row streaming) and as CSR tiles staged by TMA bulk copies otherwise
 * (the default). SELL / TILES / STAGED force one layout (STAGED falls back to TILES when the
 * matrix is not eligible). Tiled systems whose tiles all fit on the GPU at once (<= 2 tiles
 * per SM) solve in ONE cooperative launch (grid barriers between sweeps); TILES_STREAM opts
 * out of that. mcr_matrix_info reports the layout in use (DENSE, SELL, TILES or STAGED). */
enum {
    MCR_STORAGE_AUTO = 0,
    MCR_STORAGE_CSR = 1,
    MCR_STORAGE_DENSE = 2,
    MCR_STORAGE_SELL = 3,
    MCR_STORAGE_TILES = 4,
    MCR_STORAGE_TILES_STREAM = 5, /* tiles, but never the single-launch small-system solvers */
    MCR_STORAGE_STAGED = 6        /* column bands: products pass + row-sum pass (staged.cuh) */
};

typedef struct mcr_matrix mcr_matrix;

/* Outcome of one solve; field meaning follows SolveResult (solvers.py:112-120). */
typedef struct mcr_report {
    int64_t iterations;          /* sweeps / iterations (breakdown: the breakdown iteration) */
    int32_t converged;
    int32_t breakdown_which;     /* MCR_BD_*                                                 */
    int64_t breakdown_iteration;
    int64_t zero_diagonal_index; /* first row without a non-zero stored diagonal, else -1   */
    double residual_inf;         /* max|b - M x| with the full M                             */
    double device_seconds;       /* CUDA-event time: iteration loop + final residual         */
    int64_t kernel_launches;     /* kernels launched by this call                            */
} mcr_report;

typedef struct mcr_matrix_info {
    int64_t n;
    int64_t nnz;
    int32_t storage;             /* MCR_STORAGE_DENSE, _SELL, _TILES or _STAGED               */
    int32_t device;
    int64_t tiles;               /* CSR row tiles                                           */
    int64_t max_row_nnz;
    int64_t first_zero_diagonal; /* -1 when every row has a non-zero diagonal               */
    int64_t device_bytes;        /* bytes of device memory held by the handle               */
    int64_t n_global;            /* rows of the whole system (== n unless a row shard)       */
    int64_t row0;                /* first global row held (0 unless a row shard)            */
    int32_t world;               /* ranks the system is sharded over (1 = whole system)     */
    int32_t rank;
} mcr_matrix_info;

/* Library version (major*10000 + minor*100 + patch). */
MCR_API int mcr_version(void);

/* Number of visible CUDA devices (0 on a machine without a GPU). */
MCR_API int mcr_device_count(int* count);

/* Upload an n x n CSR matrix (host arrays, int64 row starts and columns, float64 values,
 * rows sorted by column) to `device`. The caller keeps ownership of the host arrays. */
MCR_API int mcr_matrix_create(int64_t n, const int64_t* rstart, const int64_t* col,
                              const double* nonzero, int device, int storage,
                              mcr_matrix** out);
MCR_API void mcr_matrix_destroy(mcr_matrix* m);
MCR_API int mcr_matrix_info_get(const mcr_matrix* m, mcr_matrix_info* info);

/* Inner products of BiCGStab. SEQUENTIAL = the reference's strictly left-to-right
 * _dot_ascending (solvers.py:136-141), bit-identical to the reference, computed in parallel by
 * k_xdot (csrc/xdot.cuh: binade runs + candidate tables, checked, with exact fallbacks);
 * SERIAL = the same bits from one dependent add per element on one CTA (slow; cross-check);
 * TREE = deterministic fixed-shape trees fused into the producing kernels (not the
 * reference's order: iteration counts may differ). Jacobi, SpMV and the residual are
 * bit-identical in every mode. */
enum { MCR_DOTS_TREE = 0, MCR_DOTS_SEQUENTIAL = 1, MCR_DOTS_SERIAL = 2 };
MCR_API int mcr_set_dot_mode(mcr_matrix* m, int mode);

/* parallel_dot_products (solvers.py:98, 384-396): with nblocks > 1 every inner product is the
 * sum, in ascending block order starting from 0.0, of the reference-order dots of the
 * _row_blocks(n, nblocks) row blocks (solvers.py:159-168). 1 = off. */
MCR_API int mcr_set_dot_blocks(mcr_matrix* m, int nblocks);

/* Stand-alone reference-order dot on `device` (host arrays): out[0] = the dot (the blocks'
 * dots summed in ascending order from 0.0 when nblocks > 1), out[1 + b] = block b's dot
 * (np.cumsum(u * v)[-1] of the block, 0.0 when empty). stats (may be NULL): fallback counters,
 * filled only when the library runs with MCR_XDOT_STATS=1. Replaces _dot_ascending
 * (solvers.py:136-141) and _ParOps.dot (solvers.py:384-396). */
/* Diagnostics: the fallback counters of a handle's reference-order dots (MCR_XDOT_STATS=1
 * runs only; zeros otherwise), `count` entries. */
MCR_API int mcr_xdot_stats(mcr_matrix* m, uint64_t* out, int count);

MCR_API int mcr_xdot(int device, int64_t n, const double* u, const double* v, int nblocks,
                     double* out, uint64_t* stats);
/* Same, then `reps` more launches on the device-resident inputs; *ms = mean ms per launch. */
MCR_API int mcr_xdot_bench(int device, int64_t n, const double* u, const double* v, int nblocks,
                           int reps, double* out, double* ms, uint64_t* stats);

/* The same dot by the one-CTA path of the small whole-solve BiCGStab kernel (n <= 8192): k = 1
 * (out[0] = u0.v0) or 2 (out[1] = u1.v1 too, both in one launch). Test / diagnostics entry. */
MCR_API int mcr_xdot_cta(int device, int64_t n, const double* u0, const double* v0, const double* u1,
                         const double* v1, int k, double* out);

/* Use `stream` (a cudaStream_t on the handle's device, or NULL for the handle's own stream)
 * for every later call on this handle. */
MCR_API int mcr_set_stream(mcr_matrix* m, void* stream);

/* y = M x, each row summed in ascending column order, no FMA (bit-identical to scipy). */
MCR_API int mcr_matvec(mcr_matrix* m, const double* x, double* y);
MCR_API int mcr_matvec_device(mcr_matrix* m, const double* d_x, double* d_y);

/* max|b - M x| (NaN-propagating, like numpy max). */
MCR_API int mcr_residual_inf(mcr_matrix* m, const double* x, const double* b, double* out);

/* Jacobi: x' = (b - R x) / diag(M) from the frozen previous iterate; stop when
 * max|x' - x| <= tol (the count includes the certifying sweep). x0 may be NULL (zeros). */
MCR_API int mcr_jacobi(mcr_matrix* m, const double* b, const double* x0, double tol,
                       int64_t max_iterations, double* x_out, mcr_report* report);
MCR_API int mcr_jacobi_device(mcr_matrix* m, const double* d_b, const double* d_x0,
                              double tol, int64_t max_iterations, double* d_x_out,
                              mcr_report* report);

/* Un-preconditioned BiCGStab with shadow vector q = r0; converged when max|s| <= tol
 * (tested before the final x/r update, which is still applied). */
MCR_API int mcr_bicgstab(mcr_matrix* m, const double* b, const double* x0, double tol,
                         int64_t max_iterations, double* x_out, mcr_report* report);
MCR_API int mcr_bicgstab_device(mcr_matrix* m, const double* d_b, const double* d_x0,
                                double tol, int64_t max_iterations, double* d_x_out,
                                mcr_report* report);

/* ---------------------------------------------------------------------------------------
 * Row-sharded solves over 1..N GPUs (the reference's row-block parallel
 * solvers jacobi_solve_parallel / bicgstab_solve_parallel, solvers.py:159-168, 233-274,
 * 314-396, with worker threads replaced by GPUs). Rank r of `world` holds the contiguous rows
 * [r*c, min(n, (r+1)*c)), c = ceil(n / world) (mcr_shard_rows), as a local CSR whose column
 * indices stay global. mcr_jacobi / mcr_bicgstab (and the _device variants) on a shard take
 * and return this rank's slice of b, x0 and x; every rank must call the same solve with the
 * same tolerance and iteration limit, and every rank gets the same iterations, residual and
 * status. Jacobi iterates are bit-identical to the one-GPU (and reference) iterates.
 * ------------------------------------------------------------------------------------- */
#define MCR_COMM_ID_BYTES 128
typedef struct mcr_comm mcr_comm;

/* Contiguous row range of `rank`. */
MCR_API int mcr_shard_rows(int64_t n_global, int world, int rank, int64_t* row0, int64_t* rows);
/* NCCL bootstrap: rank 0 creates the id, the caller distributes it to every rank. */
MCR_API int mcr_comm_unique_id(void* id);
/* One process (or thread) per GPU; NCCL is loaded at run time (libnccl.so.2). */
MCR_API int mcr_comm_create_nccl(const void* id, int world, int rank, int device, mcr_comm** out);
/* `world` ranks of ONE process, each driven by its own host thread (devices[r], or device 0
 * for all when devices is NULL): collectives become peer copies ordered by CUDA events. Fills
 * out[0..world-1]. */
MCR_API int mcr_comm_create_local(int world, const int* devices, mcr_comm** out);
MCR_API void mcr_comm_destroy(mcr_comm* comm);
MCR_API int mcr_comm_info(const mcr_comm* comm, int* world, int* rank, int* device);
/* Upload this rank's rows (local rstart, GLOBAL columns) of an n_global x n_global system. */
MCR_API int mcr_shard_create(mcr_comm* comm, int64_t n_global, int64_t row0, int64_t rows,
                             const int64_t* rstart, const int64_t* col, const double* nonzero,
                             mcr_matrix** out);

/* Fused exchange for a row shard (collective: every rank calls it, before its first solve):
 * the full vectors that SpMVs gather (Jacobi iterates, BiCGStab p and s) move to an
 * IPC-exportable allocation mapped into every peer (cudaIpc* across processes, plain pointers
 * within one); the kernels that produce those vectors store each own-row value into every
 * peer's copy as they compute it, so the allgather rides NVLink inside the producer instead
 * of following it, and the per-sweep collective shrinks to the SEND_SLOTS exchange. */
MCR_API int mcr_shard_enable_p2p(mcr_matrix* shard);

/* ---------------------------------------------------------------------------------------
 * Synthetic systems built directly in HBM (config C5: n = 2e8 does not fit the reference's
 * host generator). Family of generate_dd_matrix / generate_rhs (generator.py:100-132):
 * strictly diagonally dominant, row i has k_i ~ Poisson(mean_offdiag) (capped at 64 and n-1)
 * distinct off-diagonal columns uniform over the other n-1, values U{lo..hi}, diagonal =
 * row sum + U{1..hi}; b_i ~ U{1..10}. Every row draws from its own counter-based stream keyed
 * by (seed, global row), so the matrix is identical for any sharding. comm == NULL: the whole
 * system on `device`; else this rank's rows on the communicator's device. The CPU oracle
 * restates the generator bit for bit (orc_generate).
 * ------------------------------------------------------------------------------------- */
MCR_API int mcr_generate(mcr_comm* comm, int device, int64_t n_global, double mean_offdiag,
                         int lo, int hi, uint64_t seed, int storage, mcr_matrix** out);
/* This handle's rows of the right-hand side into device memory d_b. */
MCR_API int mcr_generate_rhs(const mcr_matrix* m, uint64_t seed, double* d_b);
/* Copy the handle's CSR back to host arrays (local rstart[n+1], global col[nnz] as int64,
 * nonzero[nnz]); any pointer may be NULL. */
MCR_API int mcr_matrix_export(mcr_matrix* m, int64_t* rstart, int64_t* col, double* nonzero);

/* The reference's input generator on the device, drawing numpy's default_rng(seed) stream:
 * generate_dd_matrix (S/generator.py:100-124, off-diagonal codes by _sample_off_diagonal
 * :77-97) with `count` = target_nnz - n off-diagonal entries and values in [lo, hi] -- the same
 * arrays as the reference, directly into a device handle. pcg = {state >> 64, state & (2^64-1),
 * inc >> 64, inc & (2^64-1)} of numpy's PCG64(seed) (the Python wrapper computes it). */
MCR_API int mcr_refgen_matrix(int device, int64_t n, int64_t count, int64_t lo, int64_t hi,
                              const uint64_t* pcg, int storage, mcr_matrix** out);
/* default_rng(seed).integers(lo, hi, size=n, endpoint=True) as doubles into host `out`
 * (generate_rhs, S/generator.py:127-132: lo = 1, hi = 10). */
MCR_API int mcr_refgen_integers(int device, int64_t n, int64_t lo, int64_t hi, const uint64_t* pcg,
                                double* out);
/* default_rng(seed).integers(0, range, size=n) into host `out` (range >= 2): the bounded draw of
 * either width, rejections included. Test / diagnostics entry. */
MCR_API int mcr_refgen_u64(int device, int64_t n, uint64_t range, const uint64_t* pcg, uint64_t* out);

/* ---------------------------------------------------------------------------------------
 * Reachability of a Markov chain: the caller side of the solve,
 * build_system + reachability_probabilities (markov.py:152-293), on the device.
 *   mcr_chain_create  uploads the transitions (CSR, rows sorted by target) and the goal states,
 *                     partitions the states with two backward closures (prob 0 / prob 1 /
 *                     uncertain), and assembles M = I - A over the uncertain states (ascending)
 *                     and rhs = one-step goal probability -- bit-identical to the reference.
 *   mcr_chain_export  host copies: classes[n] (0 = prob zero, 1 = prob one, 2 = uncertain),
 *                     uncertain[k], M (k+1 / m / m) and rhs[k]; any pointer may be NULL.
 *   mcr_chain_matrix  the solve-ready handle of M (owned by the chain: do not destroy).
 *   mcr_chain_solve   method 0 Jacobi / 1 BiCGStab (dots 1 = reference-order inner products)
 *                     on M x = rhs from x0[k] (NULL: zeros); on success x_out[n] = 1 on
 *                     prob-one states, 0 on prob-zero
 *                     states, clip(x, 0, 1) on the uncertain ones. xs_out[k] receives the
 *                     reduced solution (also on NotConverged / Breakdown). Status as mcr_jacobi.
 * ------------------------------------------------------------------------------------- */
typedef struct mcr_chain mcr_chain;
MCR_API int mcr_chain_create(int64_t n, const int64_t* rstart, const int64_t* col,
                             const double* prob, const int64_t* goals, int64_t ngoals, int device,
                             mcr_chain** out);
MCR_API void mcr_chain_destroy(mcr_chain* chain);
MCR_API int mcr_chain_info(const mcr_chain* chain, int64_t* uncertain, int64_t* prob_one,
                           int64_t* prob_zero, int64_t* m_nnz);
MCR_API int mcr_chain_export(mcr_chain* chain, int8_t* classes, int64_t* uncertain,
                             int64_t* m_rstart, int64_t* m_col, double* m_nonzero, double* rhs);
MCR_API int mcr_chain_matrix(mcr_chain* chain, mcr_matrix** out);
MCR_API int mcr_chain_solve(mcr_chain* chain, int method, int dots, double tol,
                            int64_t max_iterations, const double* x0, double* x_out,
                            double* xs_out, mcr_report* report);

/* ---------------------------------------------------------------------------------------
 * Text formats (formats.py read_matrix / read_vector / read_dtmc):
 * multithreaded readers (threads <= 0: all cores) returning the reference's result --
 * matrices in csr_from_triplets order with explicit zeros dropped, chains validated as by
 * validate(), values parsed exactly like Python's float(). Files outside the well-formed
 * plain-decimal subset (any error, duplicate, failed check, inf/nan, underscores, non-ASCII)
 * return MCR_UNSUPPORTED_INPUT; mcr_text_reason() says why and the caller defers to the
 * reference reader for its exact error. Results: mcr_text_info (n, stored entries m, initial
 * state, goal count) then mcr_text_export (rstart[n+1], col[m], values[m] -- or values[n] of a
 * vector -- and sorted unique goals[ngoals]).
 * ------------------------------------------------------------------------------------- */
typedef struct mcr_text mcr_text;
MCR_API int mcr_read_matrix(const char* path, int threads, mcr_text** out);
MCR_API int mcr_read_vector(const char* path, int threads, mcr_text** out);
MCR_API int mcr_read_dtmc(const char* path, int threads, mcr_text** out);
MCR_API int mcr_text_info(const mcr_text* text, int64_t* n, int64_t* m, int64_t* initial,
                          int64_t* ngoals);
MCR_API int mcr_text_export(const mcr_text* text, int64_t* rstart, int64_t* col, double* values,
                            int64_t* goals);
MCR_API void mcr_text_destroy(mcr_text* text);
MCR_API const char* mcr_text_reason(void);

/* Message of the last failing call on this thread ("" if none). */
MCR_API const char* mcr_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* MCR_H */
