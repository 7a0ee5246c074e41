/*
 * hecsolve_c.h -- the C-ABI boundary of the B200 HEC triangular-solve path.
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 * Every entry point returns a status code; on failure the message (and, for
 * zero pivots, the row/block) is kept in thread-local storage.
 *
 *   HEC_OK          0
 *   HEC_EINVAL      1  std::invalid_argument in the reference
 *   HEC_ERANGE      2  std::out_of_range
 *   HEC_ERUNTIME    3  std::runtime_error / CUDA failure / no device
 *   HEC_EZEROPIVOT  4  hec::ZeroPivotError(row, block)
 *   HEC_EOVERFLOW   5  std::overflow_error
 *
 * Section 1 (hec_tri_*, hec_precond_*, hec_spmv_*, hec_gmres_*) is the device
 * path: each entry replaces one reference call site (cited per function).
 * Section 2 (hec_csr_*, hec_prep_*, hec_ilu*, hec_bp_*) exposes the host setup
 * (bit-identical to the reference) so non-C++ hosts and the test-suite can
 * drive the whole path through this one library.
 */
#ifndef HECSOLVE_C_H
#define HECSOLVE_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    HEC_OK = 0,
    HEC_EINVAL = 1,
    HEC_ERANGE = 2,
    HEC_ERUNTIME = 3,
    HEC_EZEROPIVOT = 4,
    HEC_EOVERFLOW = 5
};

const char* hec_last_error(void);
int hec_last_error_row(void);
int hec_last_error_block(void);
/* library version string ("hecsolve-b200 <semver> sm_100a") */
const char* hec_version(void);
/* 1 if a CUDA device is usable by this process, else 0 (never fails). */
int hec_device_available(void);

/* ===================== Section 1: device path ========================== */

/* Solve strategies (hec_tri_options.strategy). */
enum {
    HEC_STRATEGY_AUTO = 0,
    HEC_STRATEGY_LEVELS = 1,    /* one launch per level, captured in a CUDA graph  */
    HEC_STRATEGY_PIPELINE = 2   /* persistent CTA-owned chunk pipeline (default)   */
};

typedef struct {
    int strategy;      /* HEC_STRATEGY_*                                        */
    int ctas;          /* persistent CTAs for PIPELINE; 0 = auto (cost model)   */
    int threads;       /* threads per CTA; 0 = auto                             */
    int reserved[5];
} hec_tri_options;

typedef struct {
    int n;
    int nlev;
    int strategy;        /* strategy actually used                              */
    int ctas;
    int threads;
    int chunks;          /* (CTA, level) work units                             */
    long long nnz;       /* stored entries incl. diagonal (nnz_T)               */
    long long device_bytes;
    double alg_bytes;    /* 12 nnz_T + 20 n                   */
    double predicted_us; /* cost-model critical path of one solve               */
    /* PIPELINE layout actually built (diagnostics; -1 / 0 for LEVELS) */
    int layout;          /* 0 slabs, 1 z-pencils (recognised grid), 2 strips,     */
                         /* 3 mirror of the L layout (U of an ILU pair),          */
                         /* 4 columns (7-point grid: one lane per grid column),   */
                         /* 5 columns, mirror of the L layout                     */
    int group, groups, rows_per_lane; /* solver shape G x K x RPL               */
    int width;           /* sliced-ELL width W of the device blob                */
    int ring, halo_ring, inflight;    /* shared-memory rings, descriptor slots  */
    long long wave_len;  /* entries of the wave-ordered vectors: bp holds        */
                         /* wave_len + 2, xw wave_len (n, except the column      */
                         /* layout, whose slots include padding)                 */
} hec_tri_info;

typedef struct hec_tri* hec_tri_t;

/*
 * Upload a prepared triangle. The arguments are the fields of the reference's
 * hec::PreparedTriangular (proj/include/hecsolve/triangular.hpp:18-24):
 * n, reversal_applied, schedule.{nlev, level_starts[nlev+1], inv_perm[n]},
 * hec.ell.{width, col_indices[width*n], values[width*n]} (column-major),
 * hec.csr.{row_offsets[n+1], col_indices, values} (diagonal last per row).
 * Replaces the data the reference reads in solve() (proj/src/triangular.cpp:96-103).
 */
int hec_tri_create(int n, int reversal_applied, int nlev, const int* level_starts,
                   const int* inv_perm, int ell_width, const int* ell_cols,
                   const double* ell_vals, const int* csr_row_offsets, const int* csr_cols,
                   const double* csr_vals, const hec_tri_options* options, hec_tri_t* out);

/*
 * x = T^-1 b in the original ordering, device pointers, enqueued on `stream`
 * (cudaStream_t; NULL = legacy default stream). Bitwise equal to the
 * reference's hec::solve (proj/src/triangular.cpp:90-135) for any worker count.
 * b and x must not alias. Concurrent solves on different streams are allowed:
 * each stream gets its own workspace (tickets, epoch, mailboxes). A CUDA graph
 * captured on a stream keeps that stream's workspace, so a replay must not
 * overlap another solve enqueued on the capture stream, nor a replay of another
 * graph captured on the same stream (serialise them, or capture on distinct
 * streams).
 */
int hec_tri_solve(hec_tri_t t, const double* b_dev, double* x_dev, void* stream);

/*
 * hec_tri_solve split in its two device passes: hec_tri_permute_in writes the
 * right-hand side in the layout's private row order (the reference's
 * permute-in, proj/src/triangular.cpp:110-111, into the order the persistent
 * kernel consumes: CTA, chunk, row), then the solve from bp. That order is
 * OPAQUE: only hec_tri_permute_in produces a valid bp. bp must hold
 * info.wave_len + 2 doubles (hec_tri_query) and be 16-byte aligned (the kernel moves it with bulk copies);
 * otherwise HEC_EINVAL.
 */
int hec_tri_permute_in(hec_tri_t t, const double* b_dev, double* bp_dev, void* stream);
int hec_tri_solve_ordered(hec_tri_t t, const double* bp_dev, double* x_dev, void* stream);
/* hec_tri_solve_ordered in two halves: the solve leaves x in the layout's wave
 * order (xw[p], p = wave position; the solution order for the level strategy),
 * hec_tri_permute_out gathers x[o] = xw[wpos[o]] (the reference's permute-out,
 * proj/src/triangular.cpp:131-132). A consumer that can read the wave order
 * directly (the U solve of an ILU apply) skips the second pass. */
int hec_tri_solve_wave(hec_tri_t t, const double* bp_dev, double* xw_dev, void* stream); /* bp: as above; xw: wave_len */
int hec_tri_permute_out(hec_tri_t t, const double* xw_dev, double* x_dev, void* stream);

/* Same with host vectors (H2D, solve, D2H; synchronous). Drop-in for hec::solve. */
int hec_tri_solve_host(hec_tri_t t, const double* b, double* x);

int hec_tri_query(hec_tri_t t, hec_tri_info* info);
int hec_tri_destroy(hec_tri_t t);

/* Diagnostics (PIPELINE strategy): same as hec_tri_solve, and additionally
 * writes 64 uint64 per chunk into trace_dev (device, info.chunks * 64,
 * zero-initialised): %globaltimer ns at [0] blob copy issued, [1] waiter sees
 * the blob, [2] foreign values staged, [3] chunk ready; for solver warp w:
 * [8+3w] ready seen, [9+3w] source warps done, [10+3w] segment done.
 * cta_chunk0 (host, ctas + 1) receives the chunk range of every CTA. Either
 * pointer may be NULL. */
int hec_tri_solve_traced(hec_tri_t t, const double* b_dev, double* x_dev, void* stream,
                         unsigned long long* trace_dev, int* cta_chunk0);

/*
 * L+U pair with optional RAS gather/scatter: x = scatter(U^-1 L^-1 gather(r)).
 * n_ext rows of the concatenated block ordering; gather[k] = global row feeding
 * concatenated row k; owned[k] != 0 where part(k) owns that row (restriction).
 * gather == NULL means the identity (n_ext == n, every row owned).
 * The L and U arguments are the prepared fields as in hec_tri_create.
 * Replaces hec::apply (proj/src/precond.cpp:119-145).
 */
typedef struct hec_precond* hec_precond_t;
int hec_precond_create(int n, int n_ext, const int* gather, const char* owned,
                       /* L */ int l_nlev, const int* l_level_starts, const int* l_inv_perm,
                       int l_ell_width, const int* l_ell_cols, const double* l_ell_vals,
                       const int* l_csr_row_offsets, const int* l_csr_cols,
                       const double* l_csr_vals,
                       /* U (reversal applied) */ int u_nlev, const int* u_level_starts,
                       const int* u_inv_perm, int u_ell_width, const int* u_ell_cols,
                       const double* u_ell_vals, const int* u_csr_row_offsets,
                       const int* u_csr_cols, const double* u_csr_vals,
                       const hec_tri_options* options, hec_precond_t* out);
/*
 * Local form for one RAS subdomain of a distributed vector (the multi-GPU
 * layer): the input vector has n_in entries and factor row k reads
 * r[gather[k]]; the output has n_out entries and factor row k writes
 * x[out_index[k]] unless out_index[k] < 0 (rows the subdomain does not own).
 * Replaces one block of hec::apply (proj/src/precond.cpp:125-143). Identity
 * maps (n_in == n_out == n_ext, gather[k] == out_index[k] == k: one subdomain
 * holding the whole vector) build the same object as hec_precond_create
 * without maps.
 */
int hec_precond_create_local(int n_in, int n_out, int n_ext, const int* gather, const int* out_index,
                             /* L */ int l_nlev, const int* l_level_starts, const int* l_inv_perm,
                             int l_ell_width, const int* l_ell_cols, const double* l_ell_vals,
                             const int* l_csr_row_offsets, const int* l_csr_cols,
                             const double* l_csr_vals,
                             /* U (reversal applied) */ int u_nlev, const int* u_level_starts,
                             const int* u_inv_perm, int u_ell_width, const int* u_ell_cols,
                             const double* u_ell_vals, const int* u_csr_row_offsets,
                             const int* u_csr_cols, const double* u_csr_vals,
                             const hec_tri_options* options, hec_precond_t* out);
int hec_precond_apply(hec_precond_t m, const double* r_dev, double* x_dev, void* stream);
/* Host vectors (pinned for full PCIe speed). Square preconditioners of at least
 * 2^21 rows copy in slices: each input slice is permuted while the next is in
 * flight and each output slice copied back while the next is permuted
 * (HEC_HOST_SLICES overrides the count, 1 = one copy each way). */
int hec_precond_apply_host(hec_precond_t m, const double* r, double* x);
int hec_precond_query(hec_precond_t m, hec_tri_info* l_info, hec_tri_info* u_info);
int hec_precond_destroy(hec_precond_t m);

/* HEC SpMV on the device: y = A x over column-major ELL slots (256-byte
 * aligned columns, vectorised coalesced loads) plus a CSR remainder staged
 * through shared memory per warp.
 * hec_spmv_create: from CSR, split as hec_from_csr(a, false, automatic) with
 *   padding skipped -- row sums in storage order, bitwise equal to spmv_csr
 *   (proj/src/csr.cpp:43-57).
 * hec_spmv_create_hec: from a reference HecMatrix's fields (hec.hpp:13-46:
 *   ell.{width, col_indices[width*n_rows], values} column-major, csr.{row_offsets,
 *   col_indices, values}); bitwise equal to spmv_hec (proj/src/hec.cpp:88-108),
 *   padding slots multiplied as the reference does.
 * hec_spmv_residual: y = b - A x with A x summed as above (gmres.cpp:19-24). */
typedef struct hec_spmv* hec_spmv_t;
int hec_spmv_create(int n_rows, int n_cols, const int* row_offsets, const int* cols,
                    const double* vals, hec_spmv_t* out);
int hec_spmv_create_hec(int n_rows, int n_cols, int ell_width, const int* ell_cols,
                        const double* ell_vals, const int* csr_row_offsets, const int* csr_cols,
                        const double* csr_vals, hec_spmv_t* out);
int hec_spmv_run(hec_spmv_t a, const double* x_dev, double* y_dev, void* stream);
int hec_spmv_residual(hec_spmv_t a, const double* b_dev, const double* x_dev, double* y_dev,
                      void* stream);
int hec_spmv_run_host(hec_spmv_t a, const double* x, double* y);
int hec_spmv_destroy(hec_spmv_t a);

/* Restarted right-preconditioned GMRES(m) on the device (proj/src/gmres.cpp:28-137).
 * m may be NULL. x (host, n) receives the solution. inner_residuals (host) may be
 * NULL; otherwise it receives up to inner_capacity estimates. */
typedef struct {
    int restart;
    int max_iters;
    double rel_tol;
    double abs_tol;
} hec_gmres_config;

typedef struct {
    int converged;
    int iterations;
    double final_relative_residual;
    double solve_seconds;
    int n_inner;
} hec_gmres_report;

int hec_gmres_solve(hec_spmv_t a, hec_precond_t m, const double* b, const hec_gmres_config* cfg,
                    double* x, hec_gmres_report* report, double* inner_residuals,
                    int inner_capacity);

/*
 * Fused Krylov vector kernels of the device GMRES (proj/src/gmres.cpp:63-80,
 * 120-124), exposed for drivers that reduce across GPUs themselves (RAS).
 * All scalars are device pointers; dots use a fixed-shape reduction.
 */
typedef struct hec_krylov* hec_krylov_t;
int hec_krylov_create(int n, hec_krylov_t* out);
/* w -= (*h_prev) * v_prev (skipped if v_prev == NULL); *out = dot(w, v_next) */
int hec_krylov_mgs(hec_krylov_t k, double* w, const double* v_prev, const double* h_prev,
                   const double* v_next, double* out, void* stream);
int hec_krylov_scale(hec_krylov_t k, double* y, const double* x, const double* s, void* stream); /* y = x / *s */
int hec_krylov_combine(hec_krylov_t k, int j, double* xc, const double* V, long long ldv,
                       const double* y, void* stream);                                  /* xc = sum_i<j y_i V_i */
int hec_krylov_add(hec_krylov_t k, double* x, const double* d, void* stream);           /* x += d */
int hec_krylov_sqrt(hec_krylov_t k, const double* in, double* out, void* stream);       /* *out = sqrt(*in) */
int hec_krylov_destroy(hec_krylov_t k);

/* ===================== Section 2: host setup ============================= */

typedef struct hec_csr* hec_csr_t;   /* owns a hec::CsrMatrix */

int hec_csr_create(int n_rows, int n_cols, const int* row_offsets, const int* cols,
                   const double* vals, hec_csr_t* out);
int hec_csr_from_triples(int n_rows, int n_cols, long long count, const int* rows,
                         const int* cols, const double* vals, hec_csr_t* out);
/* Borrowed views, valid until hec_csr_destroy. */
int hec_csr_view(hec_csr_t a, int* n_rows, int* n_cols, long long* nnz,
                 const int** row_offsets, const int** cols, const double** vals);
int hec_csr_destroy(hec_csr_t a);
/* hec::spmv_csr (csr.hpp:35-36): y = A x on the device (host vectors). */
int hec_csr_spmv_host(hec_csr_t a, const double* x, double* y, int workers);

/* hec::hec_from_csr (hec.hpp:48, hec.cpp:28-86) and hec::spmv_hec (hec.hpp:52-53,
 * on the device). width_mode 0 = automatic (median), 1 = fixed `width`. */
typedef struct hec_hec* hec_hec_t;   /* owns a hec::HecMatrix */
typedef struct {
    int n_rows, n_cols, ell_width;
    const int* ell_cols;       /* [ell_width * n_rows], slot k of row i at k*n_rows+i */
    const double* ell_vals;
    const int* csr_row_offsets; /* [n_rows + 1] */
    const int* csr_cols;
    const double* csr_vals;
    long long csr_nnz;
} hec_hec_view;
int hec_hec_from_csr(hec_csr_t a, int triangular, int width_mode, int width, hec_hec_t* out);
int hec_hec_view_get(hec_hec_t h, hec_hec_view* v);
int hec_hec_spmv_host(hec_hec_t h, const double* x, double* y, int workers);
int hec_hec_destroy(hec_hec_t h);

int hec_gen_poisson7(int nx, int ny, int nz, hec_csr_t* out);
int hec_gen_poisson27(int nx, int ny, int nz, hec_csr_t* out);
int hec_gen_reservoir7(int nx, int ny, int nz, double sigma, double kz_ratio, uint64_t seed,
                       hec_csr_t* out);
int hec_permute_symmetric(hec_csr_t a, const int* perm, hec_csr_t* out);
/* principal submatrix on the ascending row set rows[count] (reference
 * precond.cpp:13-34, extract_block) */
int hec_csr_submatrix(hec_csr_t a, const int* rows, int count, hec_csr_t* out);

/* hec::partition_graph + hec::extend_overlap (reference partition.cpp:28-107):
 * part_of[n]; extended part p = ext_rows[ext_offsets[p] .. ext_offsets[p+1]),
 * ascending. Borrowed views valid until hec_partition_destroy. */
typedef struct hec_partition* hec_partition_t;
int hec_partition_create(hec_csr_t a, int parts, int overlap, hec_partition_t* out);
int hec_partition_view(hec_partition_t p, int* n, int* parts, const int** part_of,
                       const int** ext_offsets, const int** ext_rows);
int hec_partition_destroy(hec_partition_t p);
int hec_random_ordering(int n, uint64_t seed, int* perm);
int hec_rcm_ordering(hec_csr_t a, int* perm);

int hec_ilu0(hec_csr_t a, hec_csr_t* l, hec_csr_t* u);
int hec_ilu_k(hec_csr_t a, int k, hec_csr_t* l, hec_csr_t* u);
int hec_ilut(hec_csr_t a, int p, double tol, hec_csr_t* l, hec_csr_t* u);

/* hec::PreparedTriangular. width_mode: 0 automatic, 1 fixed(width). */
typedef struct hec_prep* hec_prep_t;
int hec_prepare(hec_csr_t t, int upper, int width_mode, int width, hec_prep_t* out);
typedef struct {
    int kind;            /* 0 lower, 1 upper */
    int n;
    int reversal_applied;
    int nlev;
    const int* level_of;
    const int* perm;
    const int* inv_perm;
    const int* level_starts;
    int ell_width;
    const int* ell_cols;
    const double* ell_vals;
    const int* csr_row_offsets;
    const int* csr_cols;
    const double* csr_vals;
    long long csr_nnz;
} hec_prep_view;
int hec_prep_view_get(hec_prep_t p, hec_prep_view* v);
/* hec::solve on the prepared object (device mirror cached inside it). */
int hec_prep_solve_host(hec_prep_t p, const double* b, double* x);
/* the device triangle backing p (owned by p; do not destroy) */
int hec_prep_device(hec_prep_t p, hec_tri_t* t);
int hec_serial_solve(hec_csr_t t, int upper, const double* b, double* x);
int hec_prep_destroy(hec_prep_t p);

/* hec::BlockPreconditioner. kind: 0 bilu0, 1 bilut, 2 ras, 3 biluk. */
typedef struct hec_bp* hec_bp_t;
int hec_bp_build(hec_csr_t a, int kind, int blocks, int overlap, int ilut_p, double ilut_tol,
                 int width_mode, int width, int fill_level, hec_bp_t* out);
int hec_bp_dims(hec_bp_t m, int* n, int* n_parts, int* n_ext);
/* part_of[n], offsets[n_parts+1], ext_rows[n_ext] (concatenated), owned[n_ext] */
int hec_bp_maps(hec_bp_t m, int* part_of, int* offsets, int* ext_rows, char* owned);
int hec_bp_prepared(hec_bp_t m, hec_prep_t* l, hec_prep_t* u); /* borrowed */
int hec_bp_apply_host(hec_bp_t m, const double* r, double* x);
int hec_bp_device(hec_bp_t m, hec_precond_t* d); /* borrowed */
int hec_bp_destroy(hec_bp_t m);

/* hec::gmres through the C++ drop-in (device inside). m may be NULL. */
int hec_gmres_host(hec_csr_t a, const double* b, hec_bp_t m, const hec_gmres_config* cfg,
                   double* x, hec_gmres_report* report, double* inner_residuals,
                   int inner_capacity);

/* ===================== Section 3: multi-GPU RAS ======================== */
/*
 * Restricted Additive Schwarz with one subdomain per process / GPU
 * (reference proj/src/precond.cpp:74-145 build_preconditioner(ras) + apply,
 * proj/src/partition.cpp:28-107, proj/src/gmres.cpp:28-137 with the
 * preconditioner). Rank g of `world` owns part g of partition_graph(A, world)
 * and keeps local vectors [own | halo]; its block is extract_block(A, ext_g)
 * factored with ILU(0) / ILUT / ILU(k) and solved by this library's kernels.
 * Every call marked "collective" must be made by all ranks.
 */
typedef struct hec_ras_plan* hec_ras_plan_t;
/* Host plan of one rank (no device, no communication; deterministic on every rank). */
int hec_ras_plan_create(hec_csr_t a, int world, int rank, int overlap, hec_ras_plan_t* out);
/* Borrowed views, valid until the plan (or the hec_ras_t owning it) is destroyed:
 * own[n_own] and ext[n_ext] ascending global rows, halo[n_halo] by (owner, row),
 * send_offsets / recv_offsets [world + 1] (peer p's segments), send_idx[n_send]
 * (own positions sent, in the peer's halo order), gather / out_index [n_ext]
 * (block row -> local [own | halo] index; -> own position or -1). */
typedef struct {
    int n, rank, world, overlap, n_own, n_halo, n_ext, n_send;
    const int* own;
    const int* halo;
    const int* ext;
    const int* send_offsets;
    const int* send_idx;
    const int* recv_offsets;
    const int* gather;
    const int* out_index;
    const int* part_of; /* [n] */
} hec_ras_plan_view;
int hec_ras_plan_view_get(hec_ras_plan_t p, hec_ras_plan_view* v);
int hec_ras_plan_destroy(hec_ras_plan_t p);

/* Communication between the ranks. */
enum { HEC_COMM_NONE = 0, HEC_COMM_NCCL = 1, HEC_COMM_CALLBACKS = 2 };
typedef struct {
    void* ctx;
    /* in place sum over ranks of count doubles (host buffer); return 0 on success */
    int (*allreduce_sum)(void* ctx, double* buf, int count);
    /* halo exchange: send[send_offsets[p] ..) goes to peer p, recv[recv_offsets[p] ..)
     * comes from p (offsets of the rank's plan); return 0 on success */
    int (*exchange)(void* ctx, const double* send, int send_count, double* recv, int recv_count);
} hec_comm_callbacks;
typedef struct {
    int kind;                      /* HEC_COMM_*                                        */
    int rank, world;
    const unsigned char* nccl_id;  /* HEC_COMM_NCCL: 128 bytes from hec_nccl_unique_id   */
    hec_comm_callbacks callbacks;  /* HEC_COMM_CALLBACKS                                 */
} hec_comm_spec;
/* NCCL (opened at first use; a process that already loaded libnccl shares it). */
int hec_nccl_unique_id(unsigned char id[128]);
int hec_nccl_version(void); /* 0 if libnccl cannot be opened */

typedef struct hec_ras* hec_ras_t;
/* Collective. local_kind: 0 ilu0 (ras / bilu0), 1 ilut(ilut_p, ilut_tol), 3 ilu_k(fill_level).
 * The communicator spans `comm->world` ranks (HEC_COMM_NONE: world 1). */
int hec_ras_create(hec_csr_t a, int overlap, int local_kind, int ilut_p, double ilut_tol, int fill_level,
                   const hec_comm_spec* comm, hec_ras_t* out);
int hec_ras_get_plan(hec_ras_t r, hec_ras_plan_t* plan); /* borrowed */
/* Collective: z_own = M^-1 r_own (halo exchange, local L and U solves, restricted
 * scatter): rank g's rows of the reference's apply(ras, world blocks), bitwise. */
int hec_ras_apply(hec_ras_t r, const double* r_own_dev, double* z_own_dev, void* stream);
int hec_ras_apply_host(hec_ras_t r, const double* r_own, double* z_own);
/* Collective: RAS-preconditioned GMRES(m) on the owned rows (host vectors, n_own).
 * Two all-reduces and two halo exchanges per iteration (CGS2). */
int hec_ras_gmres(hec_ras_t r, const double* b_own, const hec_gmres_config* cfg, double* x_own,
                  hec_gmres_report* report, double* inner_residuals, int inner_capacity);
/* Same with device vectors, enqueued on `stream` (returns when done). */
int hec_ras_gmres_device(hec_ras_t r, const double* b_own_dev, const hec_gmres_config* cfg, double* x_own_dev,
                         hec_gmres_report* report, double* inner_residuals, int inner_capacity, void* stream);
/* counters of the last hec_ras_gmres*: all-reduces, halo exchanges, our kernel launches */
int hec_ras_stats(hec_ras_t r, long long* allreduces, long long* exchanges, long long* launches);
int hec_ras_destroy(hec_ras_t r);

#ifdef __cplusplus
}
#endif

#endif /* HECSOLVE_C_H */
