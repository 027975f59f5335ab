/*
 * spg/capi.h — the drop-in C ABI of the B200 SpGEMM hot path.
 *
 * Plain C: status codes, opaque handles, host pointers and sizes only (no CUDA
 * or torch types in any signature). Host pointers are borrowed for the duration
 * of a call and never retained. Device matrices are owned by their context until
 * spg_csr_free. No function throws.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/proj/include/spgsim/…). The C++ drop-in library
 * (include/spgsim/ headers, paper_2603_21444_b200/host/) is a thin layer over this
 * ABI that re-throws the matching spgsim::Error subclass.
 *
 * Device CSR layout: rowptr int64[nrows+1], colind int32[nnz]
 * (columns < 2^31), values float64[nnz]; canonical form exactly as csr.hpp:12-17
 * (strictly increasing columns per row, explicit zeros kept).
 */
#ifndef SPG_CAPI_H
#define SPG_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One code per spgsim::Error subclass (errors.hpp:9-58) plus device failures. */
typedef enum spg_status {
    SPG_OK = 0,
    SPG_ERROR = 1,                /* spgsim::Error                     */
    SPG_DIMENSION_ERROR = 2,      /* spgsim::DimensionError            */
    SPG_PARAMETER_ERROR = 3,      /* spgsim::ParameterError            */
    SPG_GRID_ERROR = 4,           /* spgsim::GridError                 */
    SPG_INCOMPLETE_TILE_SET = 5,  /* spgsim::IncompleteTileSet         */
    SPG_ROUTING_ERROR = 6,        /* spgsim::RoutingError              */
    SPG_SCHEDULE_ERROR = 7,       /* spgsim::ScheduleError             */
    SPG_DEADLOCK_ERROR = 8,       /* spgsim::DeadlockError             */
    SPG_CUDA_ERROR = 20,
    SPG_OOM = 21,
    SPG_NO_DEVICE = 22
} spg_status;

/* Message of the last failing call on this thread (never NULL). */
const char* spg_last_error(void);

/* Library version string (for logs). */
const char* spg_version(void);

/* ---------------------------------------------------------------- context */
typedef struct spg_ctx spg_ctx;
typedef struct spg_csr spg_csr;

/* Number of usable CUDA devices (0 when there is no driver / device). */
spg_status spg_device_count(int* count);

/* Binds a context to CUDA device `device` (stream, stream-ordered memory pool,
 * kernel timers). Fails with SPG_NO_DEVICE when no device / driver is usable:
 * there is no CPU fallback. */
spg_status spg_init(int device, spg_ctx** out);
spg_status spg_finalize(spg_ctx* ctx);
/* The context's CUDA stream as an opaque pointer (a cudaStream_t), so callers
 * can time on the stream the kernels are launched on. */
void* spg_ctx_stream(spg_ctx* ctx);
spg_status spg_ctx_synchronize(spg_ctx* ctx);
int spg_ctx_device(const spg_ctx* ctx);

/* Kernel timing (CUDA events around each launch on the context stream).
 * spg_timing_enable(ctx, 1) starts recording; spg_timing_read synchronizes and
 * returns, per kernel name, the number of launches and total milliseconds.
 * names_out receives up to `cap` NUL-separated names. Returns entry count. */
spg_status spg_timing_enable(spg_ctx* ctx, int on);
spg_status spg_timing_reset(spg_ctx* ctx);
int spg_timing_read(spg_ctx* ctx, char* names_out, size_t names_cap, int64_t* launches, double* ms, int cap);

/* ------------------------------------------------------------- device CSR */
/* Upload a host CSR (replaces constructing spgsim::CsrMatrix, csr.hpp:18-35).
 * colind_width is 4 (int32) or 8 (int64; narrowed on the host — fails with
 * SPG_PARAMETER_ERROR if a column does not fit). The input must be canonical
 * only as far as the kernels need (rowptr monotone, columns sorted per row);
 * spg_csr_check validates fully. */
spg_status spg_csr_upload(spg_ctx* ctx, int64_t nrows, int64_t ncols, const int64_t* rowptr,
                          const void* colind, int colind_width, const double* values, spg_csr** out);
/* Allocate an empty (all-zero rows) device matrix: CsrMatrix::zeros (csr.cpp:11-17). */
spg_status spg_csr_zeros(spg_ctx* ctx, int64_t nrows, int64_t ncols, spg_csr** out);
spg_status spg_csr_shape(const spg_csr* m, int64_t* nrows, int64_t* ncols, int64_t* nnz);
/* Download into caller-allocated arrays sized from spg_csr_shape. Any pointer
 * may be NULL to skip that array. colind_width 4 or 8. */
/* Refills an existing device matrix from host arrays of the SAME shape and nnz
 * (int32 colind), keeping its device buffers (and any IPC export) in place.
 * The end-to-end benchmark's per-step upload of resident tiles. */
spg_status spg_csr_upload_into(spg_ctx* ctx, spg_csr* m, const int64_t* rowptr, const int32_t* colind,
                               const double* values);
spg_status spg_csr_download(spg_ctx* ctx, const spg_csr* m, int64_t* rowptr, void* colind, int colind_width,
                            double* values);
/* Device-side canonical check (csr.cpp:30-50): SPG_OK or SPG_ERROR with a
 * message naming the first violated invariant. */
spg_status spg_csr_check(spg_ctx* ctx, const spg_csr* m);
/* result_checksum (report.cpp:11-26) computed on the device: nnz and the
 * order-independent 64-bit hash of (row, col, llround(v*1e9)) — identical to
 * the reference's, so a C that never leaves HBM can be compared with it. */
spg_status spg_result_checksum(spg_ctx* ctx, const spg_csr* m, int64_t* nnz, uint64_t* hash);
spg_status spg_csr_free(spg_csr* m);
/* Raw device pointers of a handle (rowptr int64*, colind int32*, values double*). */
spg_status spg_csr_device_ptrs(const spg_csr* m, void** rowptr, void** colind, void** values);

/* --------------------------------------------------------- local kernels */
/* C = A*B (csr.hpp:64 spgemm_local, csr.cpp:132-165): SPG_DIMENSION_ERROR when
 * a.ncols != b.nrows. Pattern bit-identical to the reference; values summed per
 * output entry in ascending inner index with separate multiply and add, i.e.
 * bit-identical to the reference as well. */
spg_status spg_spgemm(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, spg_csr** c);
/* Σ_i Σ_{k∈A_i} nnz(B_k): the products (flops/2) of A*B, computed on device. */
spg_status spg_spgemm_products(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, int64_t* products);
/* C = A + B (csr.hpp:67 spgeam, csr.cpp:167-196): union pattern, values a+b. */
spg_status spg_spgeam(spg_ctx* ctx, const spg_csr* a, const spg_csr* b, spg_csr** c);
/* In-place accumulate: *acc = spgeam(*acc, x) (the partial-C merge of
 * algorithms.cpp:91); *acc may be replaced by a new handle. */
spg_status spg_spgeam_inplace(spg_ctx* ctx, spg_csr** acc, const spg_csr* x);
/* Vertical concatenation (csr.hpp:107 vconcat, csr.cpp:348-363). Slices may live
 * on other devices (peer copies over NVLink). n == 0 gives a 0x0 matrix. */
spg_status spg_vconcat(spg_ctx* ctx, const spg_csr* const* slices, int n, spg_csr** out);
/* Sub-block [r0,r1) x [c0,c1) with local indices (the per-tile effect of
 * partition, partition.cpp:161-222). */
spg_status spg_csr_extract(spg_ctx* ctx, const spg_csr* m, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                           spg_csr** out);
/* Copy a handle (possibly from another device) into this context. */
spg_status spg_csr_copy(spg_ctx* ctx, const spg_csr* m, spg_csr** out);

/* Device tile store. Schemes as spgsim::Scheme (partition.hpp:10). */
typedef enum spg_scheme { SPG_SCHEME_TRIDENT = 0, SPG_SCHEME_GRID2D = 1, SPG_SCHEME_ROWS1D = 2 } spg_scheme;
/* The tile rectangles of make_tile_map (partition.cpp:95-159): rects_out
 * receives procs x {row_begin, row_end, col_begin, col_end}. SPG_GRID_ERROR as
 * the reference (trident: P % lambda, P/lambda a perfect square; grid2d: P a
 * perfect square). */
spg_status spg_tile_rects(int64_t nrows, int64_t ncols, int scheme, int procs, int gpus_per_node,
                          int64_t* rects_out);
/* Device partition (partition.cpp:161-222): the global matrix m, resident on
 * its context's device, split into the procs tiles of make_tile_map with local
 * indices. Tile r is built on ctxs[r % nctx] by kernels that read m in place
 * (NVLink peer loads when m lives on another device): one pass over m, no host
 * round trip. tiles_out receives procs handles. */
spg_status spg_partition(spg_ctx* const* ctxs, int nctx, const spg_csr* m, int scheme, int procs, int gpus_per_node,
                         spg_csr** tiles_out);
/* Device reassemble (partition.cpp:224-261): the global nrows x ncols matrix
 * from the procs tiles of that map (rank order, on any devices, read in place),
 * built on ctx. SPG_INCOMPLETE_TILE_SET when the tile count or a tile's shape
 * does not match the map. Bit-identical inverse of spg_partition. */
spg_status spg_reassemble(spg_ctx* ctx, const spg_csr* const* tiles, int ntiles, int64_t nrows, int64_t ncols,
                          int scheme, int procs, int gpus_per_node, spg_csr** out);

/* Host-buffer convenience for the drop-in path: upload A and B, multiply,
 * keep C on the device (query with spg_csr_shape, fetch with spg_csr_download).
 * When B's host arrays are A's (C = A*A) the matrix is uploaded once. */
spg_status spg_spgemm_host(spg_ctx* ctx, int64_t a_nrows, int64_t a_ncols, const int64_t* a_rowptr,
                           const void* a_colind, const double* a_values, int64_t b_nrows, int64_t b_ncols,
                           const int64_t* b_rowptr, const void* b_colind, const double* b_values,
                           int colind_width, spg_csr** c);

/* Host-to-host local multiply, the whole of spgemm_local (csr.cpp:132-165:
 * host CSR in, host CSR out). A and B are uploaded (once when B is A), A is
 * multiplied in `batches` row batches (<= 0: 8) cut at equal shares of A's
 * entries, and each batch's columns/values are copied into the caller's
 * arrays while the next batch is multiplied. At most two batch products are
 * alive on the device at a time, so batches also bound the device memory C
 * needs. (Config 2 on one B200: 8 batches 250-267 ms per call against 283-290
 * ms for spg_spgemm_host + spg_csr_download; 32 batches 556 ms.) c_rowptr has a_nrows+1 slots,
 * c_colind/c_values room for c_cap entries (colind 4- or 8-byte per
 * colind_width, which also gives the width of A's and B's colind). *c_nnz
 * receives nnz(C); when it exceeds c_cap the call returns SPG_PARAMETER_ERROR
 * and the arrays are left unspecified (retry with c_cap >= *c_nnz). Host
 * arrays should be pinned (spg_host_register) for the copies to overlap. */
spg_status spg_spgemm_host_to_host(spg_ctx* ctx, int64_t a_nrows, int64_t a_ncols, const int64_t* a_rowptr,
                                   const void* a_colind, const double* a_values, int64_t b_nrows, int64_t b_ncols,
                                   const int64_t* b_rowptr, const void* b_colind, const double* b_values,
                                   int colind_width, int batches, int64_t c_cap, int64_t* c_rowptr,
                                   void* c_colind, double* c_values, int64_t* c_nnz);

/* MCL post-step on device (csr.cpp:224-249): column_normalize then prune. */
spg_status spg_column_normalize(spg_ctx* ctx, spg_csr* m);
spg_status spg_prune(spg_ctx* ctx, const spg_csr* m, double threshold, spg_csr** out);
/* In-place v = pow(v, exponent) (csr.hpp:80 elementwise_power, csr.cpp:251-255);
 * exponent 2 is the correctly rounded square. */
spg_status spg_elementwise_power(spg_ctx* ctx, spg_csr* m, double exponent);
/* The MCL iteration post-step after the expansion (apps.cpp:79-82):
 * *out = column_normalize(elementwise_power(prune(column_normalize(c), prune_threshold), inflation)).
 * The first normalize, the prune and the power are one fused pass over c
 * (c is not modified); SPG_PARAMETER_ERROR on a negative threshold. */
spg_status spg_mcl_poststep(spg_ctx* ctx, const spg_csr* c, double prune_threshold, double inflation, spg_csr** out);

/* --------------------------------------------------- distributed drivers */
/* Ledger cell, mirrors LedgerCell (netmodel.hpp:53-63). */
typedef struct spg_ledger_cell {
    uint64_t messages;
    uint64_t nnz;
    uint64_t bytes;
} spg_ledger_cell;

/* Trident grid (partition.hpp:18-35): q = sqrt(P/lambda), SPG_GRID_ERROR when
 * P % lambda != 0 or P/lambda is not a perfect square. */
spg_status spg_trident_grid(int procs, int gpus_per_node, int* q);

/* Single-process trident_spgemm (algorithms.cpp:24-101) over the contexts in
 * `ctxs` (one per GPU; logical ranks are mapped rank -> ctxs[rank % nctx]).
 * a_tiles / b_tiles: the trident partition of A and B (rank order), each tile
 * living on its rank's device. Exchange: GI pulls of A_{i,s,k}, B_{s,j,k} from
 * their owners + LI allgather of B_{s,j,.} inside the virtual node, all as
 * device-to-device copies over NVLink; the local multiply and the partial-C
 * merge run on each rank's device. c_tiles_out receives P handles.
 * ledger_out (optional): P*2*2 cells [rank][0 sent,1 received][0 LI,1 GI].
 * timeline_out (optional): P*q*4 doubles [rank][round][fetch_ms, allgather_ms,
 * multiply_ms, merge_ms] measured with CUDA events. */
spg_status spg_trident_spgemm(spg_ctx* const* ctxs, int nctx, const spg_csr* const* a_tiles,
                              const spg_csr* const* b_tiles, int procs, int gpus_per_node, int index_width,
                              int value_width, spg_csr** c_tiles_out, spg_ledger_cell* ledger_out,
                              double* timeline_out);

/* One exchange timeline event, mirrors TimelineEvent (engine.hpp:25-38).
 * type: 0 enqueue-request, 1 serve-request, 2 transfer-complete,
 * 3 allgather-complete, 4 compute-complete (EventType, engine.hpp:15-21);
 * operand: 0 A, 1 B; link: 0 SELF, 1 LI, 2 GI (LinkClass, netmodel.hpp:11).
 * src/dst/round/operand/link/nnz/bytes follow the reference engine's
 * bookkeeping (engine.cpp:228-302); t_start/t_end are MEASURED seconds from the
 * rank's start (CUDA events on its device), not the modeled alpha-beta clock.
 * allgather-complete: src = node id, dst = -1, times over the node's members. */
typedef struct spg_event {
    int32_t type, src, dst, round, operand, link;
    double t_start, t_end;
    int64_t nnz, bytes;
} spg_event;

/* spg_trident_spgemm with the measured exchange record. The ledger is built
 * from the tiles each rank actually consumed (one log entry per pull or
 * in-place read of another rank's tile, with its rows and nnz), booked along
 * the reference's routes: A and the rank's own B slice index from their
 * owners (GI/LI by node), the other slices of B_{s,j} as the node's LI
 * allgather (engine.cpp:228-302). node_start_delay (optional, n_delays
 * entries, seconds): virtual node n's ranks start their pulls after that delay
 * on the device (the reference's skew knob, engine.cpp:217-221).
 * events_out (optional): up to events_cap events; *n_events (optional)
 * receives how many were produced (SPG_PARAMETER_ERROR if more than events_cap;
 * C, ledger and timeline are still complete then).
 * xfer_out (optional): P*4 doubles per rank [device bytes pulled, pull ms
 * (first pull start to last pull end), tiles pulled, tiles read in place]. */
spg_status spg_trident_spgemm_ex(spg_ctx* const* ctxs, int nctx, const spg_csr* const* a_tiles,
                                 const spg_csr* const* b_tiles, int procs, int gpus_per_node, int index_width,
                                 int value_width, const double* node_start_delay, int n_delays,
                                 spg_csr** c_tiles_out, spg_ledger_cell* ledger_out, double* timeline_out,
                                 spg_event* events_out, int events_cap, int* n_events, double* xfer_out);

/* Single-process Sparse SUMMA (algorithms.cpp:103-174) on a sqrt(P) x sqrt(P)
 * grid2d partition; ledger as above (node_of = rank / gpus_per_node). */
spg_status spg_summa_spgemm(spg_ctx* const* ctxs, int nctx, const spg_csr* const* a_tiles,
                            const spg_csr* const* b_tiles, int procs, int gpus_per_node, int index_width,
                            int value_width, spg_csr** c_tiles_out, spg_ledger_cell* ledger_out,
                            double* timeline_out);
/* spg_summa_spgemm with the measured exchange record (events as the
 * reference's summa_spgemm emits them: transfer-complete per remote tile,
 * compute-complete per rank and round; algorithms.cpp:133-166). */
spg_status spg_summa_spgemm_ex(spg_ctx* const* ctxs, int nctx, const spg_csr* const* a_tiles,
                               const spg_csr* const* b_tiles, int procs, int gpus_per_node, int index_width,
                               int value_width, spg_csr** c_tiles_out, spg_ledger_cell* ledger_out,
                               double* timeline_out, spg_event* events_out, int events_cap, int* n_events,
                               double* xfer_out);

/* Single-process sparsity-aware 1D driver (algorithms.cpp:176-269) on a
 * rows1d partition of A and B (tile r on ctxs[r % nctx]). Rank p pulls exactly
 * the B rows named by the distinct columns of its A block from their owners
 * (read in place over NVLink), builds the reference's gathered K x n operand
 * and multiplies. ledger_out as above (one request + one transfer per (rank,
 * owner) with needed rows; node_of = rank / gpus_per_node); timeline_out: P*4
 * doubles [exchange_ms, exposed_ms, multiply_ms, 0]. */
spg_status spg_oned_spgemm(spg_ctx* const* ctxs, int nctx, const spg_csr* const* a_tiles,
                           const spg_csr* const* b_tiles, int procs, int gpus_per_node, int index_width,
                           int value_width, spg_csr** c_tiles_out, spg_ledger_cell* ledger_out,
                           double* timeline_out);

/* ------------------------------------------------------ host memory pinning */
/* Page-lock caller host memory (cudaHostRegister) so uploads/downloads of that
 * buffer run at full host-link bandwidth; unregister before freeing it. */
spg_status spg_host_register(void* ptr, size_t bytes);
spg_status spg_host_unregister(void* ptr);

/* ------------------------------- one process per GPU: CUDA IPC tile exchange */
/* Copy a matrix into IPC-exportable device memory (plain cudaMalloc blocks). */
spg_status spg_csr_make_shareable(spg_ctx* ctx, const spg_csr* m, spg_csr** out);
/* Serialize a shareable matrix into 256 opaque bytes (IPC handles + shape). */
spg_status spg_csr_ipc_export(const spg_csr* m, char* out256);
/* Map a peer process's exported matrix read-only into this context (NVLink
 * peer memory). spg_csr_free on the view unmaps it. */
spg_status spg_csr_ipc_open(spg_ctx* ctx, const char* in256, spg_csr** out);
/* The trident rounds of ONE rank (algorithms.cpp:53-92) in a one-process-per-GPU
 * job: a_views / b_views hold every rank's tile as seen from this process (its
 * own tiles and IPC views of the peers'), pulled over NVLink round by round,
 * double-buffered against the multiply. c_out receives this rank's C tile.
 * timeline_out (optional): q*4 doubles as in spg_trident_spgemm. */
spg_status spg_trident_rank(spg_ctx* ctx, int rank, int procs, int gpus_per_node, const spg_csr* const* a_views,
                            const spg_csr* const* b_views, spg_csr** c_out, double* timeline_out);

#ifdef __cplusplus
}
#endif

#endif /* SPG_CAPI_H */
