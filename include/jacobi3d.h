/*
 * jacobi3d.h -- C ABI of the B200-native Jacobi3D hot path (arXiv 2202.11819).
 *
 * The method (Sec. 3-4):
 *   a global fp64 grid is split into equal cuboid blocks
 *   ("chares"), ODF blocks per GPU ("Overdecomposition
 *   Factor (ODF), which determines the number of chares per PE and GPU");
 *   every iteration each block packs its <=6 halo faces, exchanges them with
 *   its neighbours (same GPU, or a peer GPU over NVLink: GPU-aware
 *   communication), unpacks the received faces
 *   into its ghost layers and applies the 7-point Jacobi update out of place
 *   (two buffers; update formula SPEC.md L388).
 *
 * Conventions (all functions):
 *   - Return 0 (J3D_OK) on success, a negative J3D_E* code on failure; the
 *     thread-local message is jacobi3d_last_error().  No C++ exception ever
 *     crosses this boundary.
 *   - Pointers named host_* are host memory owned by the caller; the library
 *     never retains them after the call returns.  All device memory, streams,
 *     events, CUDA graphs and the NCCL communicator are owned by the context
 *     and released by jacobi3d_destroy.
 *   - A context is bound to one CUDA device and is not thread safe (one
 *     thread per context; different contexts may be driven concurrently).
 *   - Multi-GPU (n_gpus > 1): one rank per GPU -- a process per GPU (SPMD,
 *     e.g. torchrun) -- or ranks as threads of ONE process, several of which
 *     may share a GPU (dist.ThreadGroup: how the multi-rank paths run on a
 *     one-GPU machine).  Ranks that share a GPU must be threads of one
 *     process (J3D_EUNSUPPORTED otherwise: separate processes are separate
 *     CUDA contexts, which a GPU time-slices, and cross-rank waits need the
 *     ranks to run at the same time).
 *     create / ipc_connect / init / refresh_halos / iterate / residual /
 *     checksum / time / destroy are collective: every rank calls them in the
 *     same order with the same arguments.  get_block / set_block / block_info
 *     are rank-local.
 *   - Control plane (barrier, residual max, checksum sum): NCCL when the
 *     exchange backend is J3D_XCHG_NCCL, else one POSIX shared-memory
 *     segment per rank (same node; control.cu) -- no NCCL communicator is
 *     created for the P2P and host-staging backends.
 *   - Block data on the host is the block's owned cells, extent[2] planes of
 *     extent[1] rows of extent[0] doubles, x fastest (no ghost shell).
 */
#ifndef JACOBI3D_H
#define JACOBI3D_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define J3D_API __attribute__((visibility("default")))
#else
#define J3D_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define J3D_OK            0
#define J3D_EINVAL       -1  /* bad argument: extent < 1, unknown enum, NULL pointer         */
#define J3D_EDECOMP      -2  /* no divisible decomposition / blocks per GPU != ODF */
#define J3D_ENOMEM       -3  /* device or host allocation failed                             */
#define J3D_ECUDA        -4  /* CUDA runtime / driver error (message carries the CUDA string) */
#define J3D_ENCCL        -5  /* NCCL error                                                   */
#define J3D_ENOTLOCAL    -6  /* block id not owned by this rank                              */
#define J3D_ESTATE       -7  /* call not valid in the current state (e.g. residual before any
                                iteration, iterate with stale halos on a multi-GPU context)  */
#define J3D_ETIMEOUT     -8  /* a cross-GPU epoch wait did not complete in time              */
#define J3D_EUNSUPPORTED -9  /* feature not available on this device / build                 */

/* ---- variants: where pack/unpack run (Sec. 3.4.1) ---- */
#define J3D_UNFUSED      0  /* 6 pack + 6 unpack + 1 update kernels per block (13 launches)    */
#define J3D_FUSE_A       1  /* (A) packs fused: 1 pack + 6 unpack + 1 update       (8)        */
#define J3D_FUSE_B       2  /* (B) packs fused, unpacks fused: 1 + 1 + 1           (3)        */
#define J3D_FUSE_C       3  /* (C) unpack + update + pack in ONE kernel: the unpack is fused into
                               the update's prologue (ghosts read from the receive buffers), the
                               pack into its epilogue (new boundary values written to the send
                               buffers)                                             (1)        */
#define J3D_FUSE_DIRECT  4  /* B200 variant of (C): the epilogue stores the new boundary values
                               straight into the neighbour's ghost layer (same GPU: local store;
                               peer GPU: NVLink store into the peer's buffer), so there is no
                               unpack at all                                        (1)        */

/* ---- launch orchestration ----------------- */
#define J3D_PER_BLOCK    0  /* one launch per block; per-block prioritised streams: update on a
                               low-priority stream, (un)pack on a high-priority stream         */
#define J3D_BATCHED      1  /* one launch per kernel kind per GPU covering all its blocks       */
#define J3D_PERSISTENT   2  /* one launch per jacobi3d_iterate(n) call performing all n
                               iterations: the persistent grid walks n x (work items) in order
                               and an item of iteration k+1 starts as soon as the z-chunk slabs
                               it reads (own block and neighbour blocks) finished iteration k,
                               tracked by on-device completion counters -- no launch, no
                               host sync and no grid-wide tail between iterations (PAPER.md
                               L739-749: launch/sync overhead at fine granularity).  Across
                               GPUs the counters live in the IPC-mapped arena and a slab next
                               to a peer waits on the peer's counter over NVLink; the epilogue
                               stores every peer face straight into the peer's ghost layer
                               (no exchange kernels, no host-side epochs); the call ends with
                               a wait until the peers' writes into this GPU have landed.
                               Requires variant J3D_FUSE_DIRECT, use_graph == 0 and, for
                               n_gpus > 1, exchange AUTO / P2P; else J3D_EINVAL              */

/* ---- exchange backend between GPUs (same-GPU faces are always LOCAL) ---- */
#define J3D_XCHG_AUTO    0  /* P2P when every peer is reachable over NVLink, else NCCL          */
#define J3D_XCHG_NCCL    1  /* grouped ncclSend/ncclRecv, one group per iteration               */
#define J3D_XCHG_P2P     2  /* direct NVLink stores into the peer's buffers + epoch flags       */
#define J3D_XCHG_HOST    3  /* host staging (the paper's Charm-H / MPI-H):
                               device send buffer -> D2H into pinned POSIX shared memory ->
                               the neighbour's H2D into its receive buffer; same-node ranks   */

/* ---- initial conditions (readings R6, R7, R12) ---------------- */
#define J3D_INIT_DEFAULT 0  /* owned 0.0, global ghost shell = boundary             */
#define J3D_INIT_CONST   1  /* every cell = p[0] (owned and ghost)                              */
#define J3D_INIT_LINEAR  2  /* every cell = ((p0*i + p1*j) + p2*k) + p3 in global coordinates,
                               ghost cells at coordinate -1 and g                               */
#define J3D_INIT_HASH    3  /* owned = (splitmix64(splitmix64(seed) ^ gidx) >> 11) * 2^-53,
                               gidx = i + gx*(j + gy*k); global ghost shell = boundary          */

typedef struct jacobi3d jacobi3d_t; /* opaque context */

typedef struct {
    int64_t gx, gy, gz;   /* global OWNED cells per axis (the ghost shell is extra); >= 1        */
    int64_t bx, by, bz;   /* block extent; 0,0,0 = automatic (surface-minimising over ODF)      */
    int32_t odf;          /* blocks per GPU; >= 1                           */
    int32_t n_gpus;       /* ranks/GPUs in the job; >= 1                                         */
    int32_t rank;         /* this process's rank in [0, n_gpus)                                  */
    int32_t device;       /* CUDA device ordinal this rank uses                                  */
    int32_t variant;      /* J3D_UNFUSED .. J3D_FUSE_DIRECT                                      */
    int32_t launch;       /* J3D_PER_BLOCK | J3D_BATCHED | J3D_PERSISTENT                         */
    int32_t use_graph;    /* 1: capture one iteration per buffer parity into two CUDA graphs and
                             alternate them; 0: direct launches             */
    int32_t exchange;     /* J3D_XCHG_*                                                          */
    int32_t overlap;      /* 1 (BATCHED, n_gpus > 1): update the blocks' exterior (every tile x z
                             chunk touching a peer face) first, then run the exchange of those
                             faces on a separate stream while the interior updates (PAPER.md
                             Fig 1 manual overlap L79-107, overdecomposition overlap L146-156);
                             0: update everything, then exchange                               */
    int32_t reserved;     /* must be 0                                                           */
    double  boundary;     /* Dirichlet ghost value for DEFAULT and HASH inits (default 1.0)      */
} jacobi3d_config;

typedef struct {          /* filled by jacobi3d_plan: integers only, no GPU needed              */
    int32_t gpu_grid[3];  /* (px,py,pz): surface-minimising over n_gpus, lexicographic tie-break */
    int32_t blk_grid[3];  /* blocks per GPU along x,y,z; product == odf                          */
    int64_t blk_ext[3];   /* block extent (bx,by,bz)                                             */
    int64_t n_blocks;     /* odf * n_gpus; block id = x-fastest linear index on the global block
                             grid (gpu_grid * blk_grid)                                          */
    int64_t bytes_per_gpu;/* device bytes one rank allocates (2 ghosted buffers per block incl.
                             their x ghost arrays and row pitch padding, face buffers x 2
                             parities, flags, persistent-launch counters)                         */
    int32_t peer_faces_max; /* max over ranks of block faces whose neighbour is on another GPU  */
    int32_t local_faces;    /* block faces (this rank, rank 0 if plan-only) with a same-GPU nbr */
} jacobi3d_plan_info;

typedef struct {
    int64_t iterations;       /* Jacobi iterations completed since the last init               */
    int64_t kernel_launches;  /* kernels launched by the library since the last stats reset     */
    int64_t graph_launches;   /* cudaGraphLaunch calls since the last stats reset               */
    int64_t last_graph_parity;/* parity of the last graph launched (-1 if none)                 */
    int64_t launches_per_iter_block; /* kernel launches per interior block per iteration of the
                                        configured variant (13/8/3/1/1)              */
    int64_t tile_kind;        /* stencil tile configuration in use (kernels.cu J3D_TILES row)    */
    int64_t work_items;       /* stencil work items (tile x z chunk) per iteration on this rank  */
} jacobi3d_stats;

/* Plan the decomposition without touching a GPU (PAPER.md
 * L562-565 "decomposed in a way that minimizes the aggregate surface area";
 * tie-break and divisibility rule SPEC.md L358-361, L376-384).  cfg->rank is
 * used only for local_faces.  Returns J3D_EINVAL / J3D_EDECOMP on bad input. */
J3D_API int jacobi3d_plan(const jacobi3d_config *cfg, jacobi3d_plan_info *out);

/* Plan-only (no GPU) export of the persistent launch's dependency lists
 * (J3D_PERSISTENT): the slabs of rank cfg->rank are (block,
 * z chunk zc, tile row ty) with nzc z chunks per block (chunk zc = planes
 * [nz*zc/nzc, nz*(zc+1)/nzc)) and tile rows of tile_ty rows; an item of
 * iteration k of a slab starts once every slab in its list finished
 * iteration k-1.  Writes one row of 7 int64 per list entry: block id, zc,
 * ty, then the listed slab's owner rank, block id, zc, ty (peer slabs are
 * the ones whose counters are read over NVLink).  host_out may be NULL;
 * at most cap_rows rows are written; *n_rows = the total.  The same code
 * builds the context's device tables (setup.cu slab_dep_refs). */
J3D_API int jacobi3d_debug_slab_deps(const jacobi3d_config *cfg, int32_t tile_ty, int32_t nzc, int64_t *host_out,
                                     int64_t cap_rows, int64_t *n_rows);

/* Debug (no GPU): the shared-memory control plane of a multi-rank context on
 * its own (control.cu; the one the P2P and host-staging backends use for
 * barriers and reductions).  Rank `rank` of `n_ranks` (>= 2; every rank calls
 * this concurrently -- threads or processes of one node -- with the same key
 * and rounds) runs `rounds` collectives: out_sum[r] = sum over ranks of
 * values[r] (mod 2^64), out_max[r] = max over ranks of values[r], with an
 * extra barrier every third round.  J3D_ETIMEOUT if a rank does not show up
 * within J3D_TIMEOUT_S. */
J3D_API int jacobi3d_debug_control(const uint8_t *key, int32_t rank, int32_t n_ranks, int64_t rounds,
                                   const uint64_t *values, uint64_t *out_sum, uint64_t *out_max);

/* Fill out[128] with an NCCL unique id (call on rank 0 only, broadcast the
 * bytes to every rank before jacobi3d_create). */
J3D_API int jacobi3d_nccl_unique_id(uint8_t out[128]);

/* Create a context: plan, allocate every block's two ghosted buffers and face
 * buffers on cfg->device, create streams/events, load every kernel it will
 * launch (no lazy loading while ranks wait on each other), and for n_gpus > 1
 * take nccl_uid (128 bytes, identical on every rank; NULL allowed when
 * n_gpus == 1) as the job's key: the NCCL communicator's unique id with the
 * NCCL backend, else the name of the shared-memory control plane (any 128
 * bytes unique to the job).  A context with n_gpus > 1 must then be
 * connected with jacobi3d_ipc_export / jacobi3d_ipc_connect before init.
 * On failure everything allocated is freed and *out is NULL. */
J3D_API int jacobi3d_create(const jacobi3d_config *cfg, const uint8_t *nccl_uid, jacobi3d_t **out);

/* Multi-rank bootstrap.  export writes this rank's connection record into
 * host_out (capacity cap bytes, *len = bytes written; record size is
 * constant): the CUDA IPC handle of its arena, the arena's address (for
 * peers that are threads of the same process, which cannot open their own
 * IPC handle), a process token and the GPU's UUID.  The caller all-gathers
 * the records (torch.distributed, or dist.ThreadGroup for thread ranks) into
 * rank order and passes the concatenation to connect (collective), which
 * maps the neighbours' device memory (P2P), the neighbours' staging
 * segments (host backend) and every rank's control segment, and ends with a
 * barrier.  connect returns J3D_EUNSUPPORTED if ranks of different processes
 * share a GPU, if use_graph is set while some GPU hosts several ranks (graph
 * launches of one CUDA context share its internal streams, so a captured
 * epoch wait of one rank can block the peer work it waits for), or if a P2P
 * peer's GPU is not reachable.  n_gpus == 1: no-op. */
J3D_API int jacobi3d_ipc_export(jacobi3d_t *ctx, uint8_t *host_out, size_t cap, size_t *len);
J3D_API int jacobi3d_ipc_connect(jacobi3d_t *ctx, const uint8_t *host_all, size_t len_per_rank);

/* Initialise every local block, both buffers, including the ghost shell
 * (kinds above; p = 4 parameters, may be NULL for DEFAULT/HASH).  Resets the
 * iteration count to 0.  Collective. */
J3D_API int jacobi3d_init(jacobi3d_t *ctx, int kind, const double *p, uint64_t seed);

/* Overwrite the owned cells of a local block of the CURRENT buffer from host
 * memory (layout above).  Marks the halos stale: call
 * jacobi3d_refresh_halos (collective) before iterating; on a single-GPU
 * context jacobi3d_iterate refreshes automatically. */
J3D_API int jacobi3d_set_block(jacobi3d_t *ctx, int64_t block_id, const double *host_in);

/* Re-exchange every face of the current buffer (pack, exchange, unpack) so
 * that all ghost layers hold the neighbours' current values.  Collective. */
J3D_API int jacobi3d_refresh_halos(jacobi3d_t *ctx);

/* Enqueue n Jacobi iterations on the context's streams.  Asynchronous: it
 * returns once the work is queued; no host synchronisation per iteration.
 * J3D_PERSISTENT: one stencil launch for all n (plus, across GPUs, one small
 * end-of-call wait kernel).  J3D_ESTATE if halos are stale on a multi-GPU
 * context or P2P peers are not connected.  n = 0 enqueues nothing. */
J3D_API int jacobi3d_iterate(jacobi3d_t *ctx, int64_t n);

/* Wait for all queued work; surfaces deferred CUDA / NCCL errors. */
J3D_API int jacobi3d_synchronize(jacobi3d_t *ctx);

/* Copy the owned cells of a local block of the current buffer to host
 * memory (synchronous).  J3D_ENOTLOCAL if block_id is not on this rank. */
J3D_API int jacobi3d_get_block(jacobi3d_t *ctx, int64_t block_id, double *host_out);

/* Copy the owned sub-box [lo, lo+ext) (block-local owned coordinates, x
 * fastest) of a local block of the current buffer to host memory
 * (synchronous): sampled parity checks at sizes too large to copy back. */
J3D_API int jacobi3d_get_region(jacobi3d_t *ctx, int64_t block_id, const int64_t lo[3], const int64_t ext[3],
                                double *host_out);

/* Block geometry: global origin of the owned cells, extent, owner rank. */
J3D_API int jacobi3d_block_info(jacobi3d_t *ctx, int64_t block_id, int64_t origin[3], int64_t extent[3],
                        int32_t *owner_rank);

/* Global max |u^n - u^(n-1)| over owned cells (R11; the paper
 * runs fixed iteration counts and defines no residual).  Requires n >= 1
 * iterations since init / set_block (J3D_ESTATE otherwise).  Collective,
 * synchronous. */
J3D_API int jacobi3d_residual(jacobi3d_t *ctx, double *out);

/* Global order-independent checksum of the current owned cells:
 * sum over cells of splitmix64(bits(u) ^ splitmix64(gidx)) mod 2^64
 * (R15).  Collective, synchronous. */
J3D_API int jacobi3d_checksum(jacobi3d_t *ctx, uint64_t *out);

/* Timed run: warmup iterations, then iters iterations bracketed by CUDA
 * events on the context's main stream (after waiting for the context's
 * streams and, for n_gpus > 1, a barrier).  *ms_per_iter = this rank's
 * elapsed / iters.  Collective. */
J3D_API int jacobi3d_time(jacobi3d_t *ctx, int64_t warmup, int64_t iters, double *ms_per_iter);
/* (J3D_PERSISTENT: the timed iters iterations are one launch.) */

/* Stats / launch counters (SPEC.md L424 launch-count law). */
J3D_API int jacobi3d_get_stats(jacobi3d_t *ctx, jacobi3d_stats *out);
J3D_API int jacobi3d_reset_stats(jacobi3d_t *ctx);

/* Per-kernel timing of the dominant kernel (the stencil update): when
 * enabled, every stencil launch is bracketed by CUDA events on the stream it
 * is launched on.  read returns the summed event time (ms) and the launch
 * count since enabling, and the algorithmic bytes those launches moved
 * (16 B per lattice-site update). */
J3D_API int jacobi3d_profile_enable(jacobi3d_t *ctx, int enable);
J3D_API int jacobi3d_profile_read(jacobi3d_t *ctx, double *total_ms, int64_t *launches, double *alg_bytes);

/* Timing-only switch (exposed-halo measurement): when 1, the
 * cross-GPU exchange and its waits are skipped (results become invalid). */
J3D_API int jacobi3d_set_skip_exchange(jacobi3d_t *ctx, int skip);

/* Self-test of the stencil's division by 7: on the
 * current CUDA device, compare the kernel's correctly rounded s/7 -- the
 * fast path with the stencil's rare-path decision, and the exact routine --
 * with the IEEE division routine (__ddiv_rn) for n generated inputs (every
 * bit pattern incl. subnormals, +-inf and NaN, [0,7), dyadic integers,
 * near-subnormal and near-overflow sums, +-0, +-DBL_MAX); NaN results
 * compare by NaN-ness.
 * *mismatches = number of differing results; example[3] (may be NULL) =
 * first failing s, kernel result, IEEE result. */
J3D_API int jacobi3d_div7_selftest(uint64_t n, uint64_t seed, uint64_t *mismatches, double *example);

/* Free everything.  NULL-safe.  Collective when n_gpus > 1: it begins with a
 * barrier over the control plane, so no peer can still read (persistent
 * launch: slab counters) or write (epilogue / pack stores) this rank's memory
 * when it is freed. */
J3D_API int jacobi3d_destroy(jacobi3d_t *ctx);

/* Message of the last failing call on this thread ("" if none). */
J3D_API const char *jacobi3d_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* JACOBI3D_H */
