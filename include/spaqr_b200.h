/*
 * spaqr_b200 — C ABI of the B200 implementation of the spaQR hot path.
 *
 * The reference (proj/include/spaqr/, C++20 + Eigen, single-threaded CPU) has
 * no FFI or plugin layer; its drop-in boundary is the C++ API
 *   Pipeline::Pipeline           proj/include/spaqr/pipeline.h:39-44
 *   spaqr_factorize(A,h,owner)   proj/include/spaqr/factorize.h:51-53
 *   Factorization::w_solve/...   proj/include/spaqr/transforms.h:66-69
 *   cgls(A, W, b, u, opt, w)     proj/include/spaqr/solve.h:30-31
 *   csne_solve(...)              proj/include/spaqr/solve.h:39-41
 *   block_householder_qr, apply_reflectors_left_t, truncated_cpqr,
 *   tri_solve_upper              proj/include/spaqr/dense_kernels.h:24-54
 * Each entry point below replaces one of those (cited per function).  Plain
 * pointers and sizes only; host arrays unless a name says "_dev".
 *
 * Conventions: matrices are FP64 column-major; indices are int32; A is CSC
 * (colptr n+1, rowind nnz, vals nnz).  Status codes: SPQR_OK, SPQR_E_SINGULAR
 * (singular front; *err_cluster names it, as SingularFrontError, types.h:24-31),
 * SPQR_E_SHAPE (std::invalid_argument), SPQR_E_CUDA, SPQR_E_OTHER.  One host
 * thread per handle.
 */
#ifndef SPAQR_B200_H
#define SPAQR_B200_H

#ifdef __cplusplus
extern "C" {
#endif

enum { SPQR_OK = 0, SPQR_E_SINGULAR = 1, SPQR_E_SHAPE = 2, SPQR_E_CUDA = 3, SPQR_E_OTHER = 4 };
enum { SPQR_SOLVER_SPAQR = 0, SPQR_SOLVER_DIRECT = 1, SPQR_SOLVER_DIAG = 2 };
enum { SPQR_W_APPLY = 0, SPQR_W_SOLVE = 1, SPQR_WT_APPLY = 2, SPQR_WT_SOLVE = 3 };
/* Factorization::q_apply_t / q_apply (transforms.h:70-71; transforms.cpp:113-127): y (length M)
 * <- Q^T y / Q y, for factorizations made with store_q (factorize.h:16). */
enum { SPQR_Q_APPLY_T = 4, SPQR_Q_APPLY = 5 };

typedef struct spqr_pipeline spqr_pipeline;

/* FactorizeObserver / EngineView (factorize.h:31-43): the engine state after each phase,
 * materialised on the host (tests, diagnostics).  Front f (cluster front_cluster[f]) has rows
 * rows[rows_ptr[f] .. rows_ptr[f+1]) and key blocks keys[keys_ptr[f] .. keys_ptr[f+1])
 * (ascending), block b being key_width[b] columns of nrows values (column-major) at
 * values + block_off[b].  cols: the active columns of every cluster.  The GPU engine
 * eliminates a stage in dependency waves: one "eliminate" notification per wave, whose
 * clusters are wave[0..nwave) (detail = wave[0]); other phases: "scale", "sparsify_rows",
 * "sparsify_cols", "merge" (detail -1). */
typedef struct {
    int nfronts;
    const int* front_cluster;
    const int* rows_ptr;
    const int* rows;
    const int* keys_ptr;
    const int* keys;
    const int* key_width;
    const long long* block_off;
    const double* values;
    int nclusters;
    const int* cols_ptr;
    const int* cols;
    int nwave;
    const int* wave;
    long long pivots, dropped, trailing;
} spqr_engine_view;
typedef void (*spqr_observer_fn)(void* user, const char* phase, int stage, int detail, const spqr_engine_view* view);

/* Library / device probes. */
const char* spqr_version(void);
int spqr_device_count(void);

/* Pipeline::Pipeline (pipeline.cpp:19-62): scale columns, nested dissection
 * (geometric when coords != NULL, imported when parts != NULL), interfaces,
 * ordering, row matching/assignment on the host; spaqr_factorize
 * (factorize.cpp:795-804) on the GPU.  levels <= 0 picks default_num_levels. */
int spqr_pipeline_create(int m, int n, const int* colptr, const int* rowind, const double* vals,
                         const double* coords, int dim, const int* parts, int levels, double eps,
                         int skip_levels, int solver, int device, spqr_pipeline** out, char* err, int errlen,
                         int* err_cluster);
/* Same with an observer called after every engine phase (Pipeline's obs, pipeline.h:39-41). */
int spqr_pipeline_create_observed(int m, int n, const int* colptr, const int* rowind, const double* vals,
                                  const double* coords, int dim, const int* parts, int levels, double eps,
                                  int skip_levels, int solver, int device, spqr_observer_fn obs, void* obs_user,
                                  spqr_pipeline** out, char* err, int errlen, int* err_cluster);
/* Same with FactorizeOptions::store_q (factorize.h:16; pipeline.h:18): the engine also keeps Q
 * (transforms.h:34-37,57) for SPQR_Q_APPLY_T / SPQR_Q_APPLY. */
int spqr_pipeline_create_ex(int m, int n, const int* colptr, const int* rowind, const double* vals,
                            const double* coords, int dim, const int* parts, int levels, double eps, int skip_levels,
                            int solver, int store_q, int ranks, int device, spqr_observer_fn obs, void* obs_user,
                            spqr_pipeline** out, char* err, int errlen, int* err_cluster);
void spqr_pipeline_destroy(spqr_pipeline* p);
/* |Q| (number of RowReflect factors), or -1 when the factorization keeps no Q. */
long long spqr_pipeline_nq(const spqr_pipeline* p);

/* ---- subtree split across GPUs ------------------------------ */
/* The ownership of a G = 2^g GPU split, on the host only: the pipeline's partition of A
 * (pipeline.cpp:36-53), then the owner rank of every cluster — the subtree below the top g
 * separator levels holding its tree node; top-g separator pieces at granularity k > g go to the
 * lowest subtree they border, coarser pieces to rank 0.  Call with NULL arrays to get
 * *nclusters / *ntree first.  No GPU needed. */
int spqr_rank_plan(int m, int n, const int* colptr, const int* rowind, const double* vals, const double* coords,
                   int dim, const int* parts, int levels, int nranks, int* nclusters, int* ntree, int* owner,
                   int* cluster_node, int* cluster_level, int* tree_parent, int* tree_level, char* err, int errlen);
/* A pipeline created with ranks = G > 1 accounted, per stage, the flops each rank would own
 * (flops[stage * G + rank]) and the bytes crossing ranks by phase (cross[stage * 4 + phase]:
 * stack rows, R to holders, sparsify_cols holder blocks, merges).  Returns G (0 when not
 * accounted); *nstages stages; owner (nclusters) optional. */
int spqr_pipeline_rank_stats(const spqr_pipeline* p, int* nstages, double* flops, double* cross, int* owner);

/* A factorization across nranks = 2^g processes (one per GPU), the Pipeline of every rank
 * built from the same A: each rank partitions A (identically) and keeps only its own subtree
 * (spqr_rank_plan owners) plus the top-g separator pieces; through every stage before the first
 * scale_all it eliminates its subtree's clusters, and after each such stage the ranks exchange
 * the eliminated clusters and the top-separator fronts they touched (each rank re-merges them as
 * the sequential engine leaves them); after the last one ranks > 0 send rank 0 their subtree —
 * fronts, W factors, pivot / trailing rows — and rank 0 runs the remaining stages.  Metadata
 * goes through the caller's blocking byte transport, values device to device (CUDA IPC).  Rank 0's pipeline is the factorization (identical to spqr_pipeline_create's); the
 * other ranks' pipelines hold none (solve returns an error).  Transport callbacks return 0 on
 * success. */
typedef int (*spqr_send_fn)(void* user, int dst, const void* buf, long long n);
typedef int (*spqr_recv_fn)(void* user, int src, void* buf, long long n);
int spqr_pipeline_create_dist(int m, int n, const int* colptr, const int* rowind, const double* vals,
                              const double* coords, int dim, const int* parts, int levels, double eps, int skip_levels,
                              int device, int rank, int nranks, spqr_send_fn send, spqr_recv_fn recv, void* user,
                              spqr_pipeline** out, char* err, int errlen, int* err_cluster);
/* out3: 1 if this rank's part went to rank 0 (no factorization here), seconds in the
 * exchanges, bytes exchanged (host transport sent + received, values read over peer memory). */
void spqr_pipeline_dist_info(const spqr_pipeline* p, double* out3);

/* info[16]: M, N, L, nclusters, nW, n_dropped, n_trailing, n_stages, nnz_w, nnz(A), W sweep levels,
 *           engine launches, engine syncs, h2d bytes, d2h bytes, solve-plan launches per sweep pair */
void spqr_pipeline_info(const spqr_pipeline* p, long long* info);
/* times[24]: t_partition, t_factorize, t_upload, qr_device_ms, qr_flops, qr_bytes, cpqr_flops,
 *            cpqr_bytes, qr_launches, factorize_event_ms, solve_event_ms, solve_launches,
 *            elimination_waves, cpqr_redundant_bytes, cpqr_redundant_flops, sweep_device_ms (last
 *            solve), sweeps (last solve), sweep_algorithmic_bytes (one sweep), solve_plan_build_s,
 *            w_solve levels, wt_solve levels (rest 0) */
void spqr_pipeline_times(const spqr_pipeline* p, double* times);
/* Device time (CUDA events on the engine stream), algorithmic HBM bytes and launch
 * counts per kernel family: assemble, stats, front_qr, trsm, cpqr, scatter (6 each). */
void spqr_pipeline_kernel_stats(const spqr_pipeline* p, double* ms, double* bytes, long long* launches);

/* Pipeline::solve (pipeline.cpp:70-80) -> cgls (solve.cpp:24-76) on the device, or
 * Pipeline::solve_direct (:82-92) -> csne_solve (solve.cpp:78-108) when direct != 0.
 * b: M, x: N (original column order and scaling).  hist needs maxit+2 (direct: refine+1) slots.
 * tol <= 0 / maxit <= 0 use the pipeline defaults (1e-12 / 500). */
int spqr_pipeline_solve(spqr_pipeline* p, int direct, const double* b, double* x, double tol, int maxit,
                        int* iters, int* converged, double* hist, int* nhist, double* t_solve, char* err,
                        int errlen);

/* Factorization::w_apply / w_solve / wt_apply / wt_solve (transforms.cpp:40-111),
 * applied on the device to a host vector z of length N (permuted coordinates); modes
 * SPQR_Q_APPLY_T / SPQR_Q_APPLY act on a vector of length M (store_q pipelines only). */
int spqr_pipeline_apply(spqr_pipeline* p, int mode, double* z);

/* Structure getters (reference-facing results for parity checks). */
void spqr_pipeline_perm(const spqr_pipeline* p, int* perm);          /* N: perm[new] = old */
void spqr_pipeline_owner(const spqr_pipeline* p, int* owner);        /* M: row -> finest cluster */
void spqr_pipeline_weights(const spqr_pipeline* p, double* w);       /* N */
/* pivot_row: N; dropped: n_dropped; trailing: n_trailing (info[5], info[6]) */
void spqr_pipeline_rows(const spqr_pipeline* p, int* pivot_row, int* dropped, int* trailing);
/* The SeparatorTree (partition.h:14-27): returns the node count; parent[ntree] and the root
 * when non-NULL.  finest_of_col: N.  scaled: the scaled, permuted A (Pipeline::scaled,
 * pipeline.h:62) as CSC (colptr N+1, rowind / vals nnz(A) = info[9]). */
int spqr_pipeline_tree(const spqr_pipeline* p, int* parent, int* root);
void spqr_pipeline_finest(const spqr_pipeline* p, int* finest_of_col);
void spqr_pipeline_scaled(const spqr_pipeline* p, int* colptr, int* rowind, double* vals);
/* cluster: tree_node, level, parent, stage, interior, ncols */
void spqr_pipeline_cluster(const spqr_pipeline* p, int c, int* info6);
void spqr_pipeline_cluster_cols(const spqr_pipeline* p, int c, int* cols);
/* StageStats (transforms.h:40-47): out5 = stage, nfronts, top_rows, top_cols, nnz_w; t5 = phase times */
void spqr_pipeline_stage(const spqr_pipeline* p, int s, long long* out5, double* t5);
void spqr_pipeline_stage_fronts(const spqr_pipeline* p, int s, int* front_cols, double* front_aspect);
/* W factor i: out4 = kind (0 TriangularScale, 1 ColumnRotation), |cols|, |coupled| or k, batch */
void spqr_pipeline_wfactor(const spqr_pipeline* p, int i, int* out4);
/* kind 0: cols, R (c x c), coupled, C (c x k).  kind 1: cols, V (c x k), tau, sign. */
int spqr_pipeline_wfactor_data(const spqr_pipeline* p, int i, int* cols, double* a, int* coupled, double* b,
                               double* c);
/* save_factorization (proj/src/transforms.cpp:206-240; declared transforms.h:75): write the
 * factorization (M, N, eps, pivot/dropped/trailing rows, W in chronological order) as an
 * SPQRFW01 file readable by the reference's load_factorization (transforms.cpp:242-289).
 * Returns SPQR_OK, or an error code with the message in err. */
int spqr_pipeline_save(const spqr_pipeline* p, const char* path, char* err, int errlen);

/* ---- engine- and solver-level entry points ------------------------------------------ */
/* A factorization handle: W resident on one GPU (transforms.h:53-72). */
typedef struct spqr_factorization spqr_factorization;

/* spaqr_factorize(A, h, row_owner, opt) (factorize.h:51-53; factorize.cpp:795-804) on a
 * caller-supplied hierarchy.  A: m x n CSC, already column-scaled and permuted (the engine's
 * input, pipeline.cpp:47-53).  The ClusterHierarchy (partition.h:54-75) as flat arrays:
 * cluster_info[5*c] = tree_node, level, parent, stage, interior; cluster c's (permuted) columns
 * cluster_cols[cluster_colptr[c] .. cluster_colptr[c+1]); finest_of_col[n]; the SeparatorTree
 * nodes' parents tree_parent[ntree] and its root.  row_owner[m]: a stage-(L+1) cluster per row.
 * obs (may be NULL): the FactorizeObserver (factorize.h:40-43), see spqr_engine_view.
 * Errors: m < n or inconsistent hierarchy / owner arrays -> SPQR_E_SHAPE (std::invalid_argument);
 * SingularFrontError -> SPQR_E_SINGULAR with *err_cluster. */
int spqr_factorize(int m, int n, const int* colptr, const int* rowind, const double* vals, int num_levels,
                   int nclusters, const int* cluster_info, const int* cluster_colptr, const int* cluster_cols,
                   const int* finest_of_col, int ntree, const int* tree_parent, int tree_root, const int* row_owner,
                   double eps, int skip_levels, int device, spqr_observer_fn obs, void* obs_user,
                   spqr_factorization** out, char* err, int errlen, int* err_cluster);
/* Same with FactorizeOptions::store_q (factorize.h:16). */
int spqr_factorize_ex(int m, int n, const int* colptr, const int* rowind, const double* vals, int num_levels,
                      int nclusters, const int* cluster_info, const int* cluster_colptr, const int* cluster_cols,
                      const int* finest_of_col, int ntree, const int* tree_parent, int tree_root, const int* row_owner,
                      double eps, int skip_levels, int store_q, int device, spqr_observer_fn obs, void* obs_user,
                      spqr_factorization** out, char* err, int errlen, int* err_cluster);
void spqr_factorization_destroy(spqr_factorization* f);
long long spqr_factorization_nq(const spqr_factorization* f);
/* info[8]: M, N, nW, nnz_w, n_dropped, n_trailing, n_stages, w_solve sweep levels */
void spqr_factorization_info(const spqr_factorization* f, long long* info);
void spqr_factorization_rows(const spqr_factorization* f, int* pivot_row, int* dropped, int* trailing);
/* StageStats s (transforms.h:40-47): out5 = stage, nfronts, top_rows, top_cols, nnz_w */
int spqr_factorization_stage(const spqr_factorization* f, int s, long long* out5);
int spqr_factorization_stage_fronts(const spqr_factorization* f, int s, int* front_cols);
/* Factorization::w_apply / w_solve / wt_apply / wt_solve (transforms.h:66-69) on host z (N);
 * SPQR_Q_APPLY_T / SPQR_Q_APPLY (transforms.h:70-71) on host y (M) when the factorization has Q. */
int spqr_factorization_apply(spqr_factorization* f, int mode, double* z);
/* save_factorization / load_factorization (transforms.h:75-76; transforms.cpp:206-289): SPQRFW01
 * files; a loaded factorization solves on the GPU (factor once, solve many).  Q sections
 * (store_q) are written and read back. */
int spqr_factorization_save(const spqr_factorization* f, const char* path, char* err, int errlen);
int spqr_factorization_load(const char* path, int device, spqr_factorization** out, char* err, int errlen);
/* cgls(A, W, b, u, opt, weights) (solve.h:30-31; solve.cpp:24-76) on the GPU: A m x n CSC in W's
 * column coordinates, W may be NULL (plain CGLS), weights (n) may be NULL; u (n) out;
 * tol <= 0 / maxit <= 0 take 1e-12 / 500.  hist needs maxit + 2 slots.  device is used when W is
 * NULL (else W's device). */
int spqr_cgls(int m, int n, const int* colptr, const int* rowind, const double* vals, spqr_factorization* W,
              const double* b, double* u, double tol, int maxit, const double* weights, int device, int* iters,
              int* converged, double* hist, int* nhist, double* t_solve, char* err, int errlen);

/* ---- dense kernels (dense_kernels.h:24-54), batched, one launch each ---- */
/* block_householder_qr + apply_reflectors_left_t fused: for each of nb problems
 * (m x ntot, column-major, packed back to back in a), QR of the first n columns
 * and H^T on the remaining ntot-n.  On exit: R (nonnegative diagonal) in the
 * upper triangle, reflectors (unit diagonal implicit) below, H^T X to the right.
 * info[b] = -1 ok, else the first zero/denormal pivot. */
int spqr_qr_apply_batched(int nb, int m, int n, int ntot, double* a, double* tau, double* sign, int* info);
/* Same on device pointers, in place; runs on the legacy default stream (0) and synchronises
 * before returning.  *ms = device time of the launches (CUDA events around them);
 * d_info[b] = -1 ok, else the first zero/denormal pivot (as the host entry point). */
int spqr_qr_apply_batched_dev(int nb, int m, int n, int ntot, double* d_a, double* d_tau, double* d_sign,
                              int* d_info, float* ms);
/* truncated_cpqr (dense_kernels.cpp:124-232) for nb m x n problems.  Outputs per
 * problem b (kmax = min(m,n)): rank[b], r11[b], perm[b*kmax..], R[b*kmax*n..]
 * (rank x n, ld = kmax, original column order), V[b*m*kmax..] (ld = m), tau, sign. */
int spqr_cpqr_batched(int nb, int m, int n, const double* a, double eps, int* rank, double* r11, int* perm,
                      double* R, double* V, double* tau, double* sign);
/* Same on device data, in place (R rows over the leading rank rows of each problem), ranks to
 * d_rank; *ms = device time of the launches (the C5 microbenchmark's CPQR leg). */
int spqr_cpqr_batched_dev(int nb, int m, int n, double* d_a, double eps, int* d_rank, float* ms);
/* tri_solve_upper(R, B, Right, false) (dense_kernels.cpp:242-257): B (nrows x n) <- B R^{-1}
 * for nb problems packed back to back; R (n x n) per problem. */
int spqr_trsm_right_batched(int nb, int nrows, int n, double* b, const double* r);

#ifdef __cplusplus
}
#endif
#endif /* SPAQR_B200_H */
