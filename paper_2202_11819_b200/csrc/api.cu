// api.cu -- the C ABI of include/jacobi3d.h.  Every entry point converts
// exceptions into J3D_E* codes and a thread-local message; nothing throws
// across the boundary.
#include "context.h"

using namespace j3d;

namespace {

static thread_local std::string g_err;


int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

template <class F>
int guarded(F&& f) {
    try {
        g_err.clear();
        return f();
    } catch (const Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return J3D_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return J3D_ECUDA;
    }
}

int validate_cfg(const jacobi3d_config* c) {
    if (!c) return fail(J3D_EINVAL, "config is NULL");
    if (c->variant < J3D_UNFUSED || c->variant > J3D_FUSE_DIRECT) return fail(J3D_EINVAL, "unknown variant");
    if (c->launch != J3D_PER_BLOCK && c->launch != J3D_BATCHED && c->launch != J3D_PERSISTENT)
        return fail(J3D_EINVAL, "unknown launch mode");
    if (c->launch == J3D_PERSISTENT &&
        (c->variant != J3D_FUSE_DIRECT || c->use_graph != 0 ||
         (c->n_gpus > 1 && c->exchange != J3D_XCHG_AUTO && c->exchange != J3D_XCHG_P2P)))
        return fail(J3D_EINVAL, "J3D_PERSISTENT needs variant J3D_FUSE_DIRECT, use_graph == 0 and P2P exchange");
    if (c->exchange < J3D_XCHG_AUTO || c->exchange > J3D_XCHG_HOST) return fail(J3D_EINVAL, "unknown exchange backend");
    if (c->n_gpus < 1 || c->rank < 0 || c->rank >= c->n_gpus) return fail(J3D_EINVAL, "rank / n_gpus out of range");
    if (c->odf < 1) return fail(J3D_EINVAL, "odf must be >= 1");
    if (c->reserved != 0 || (c->overlap != 0 && c->overlap != 1)) return fail(J3D_EINVAL, "bad overlap/reserved");
    return J3D_OK;
}


}  // namespace

// ======================================================================= C ABI
extern "C" {

const char* jacobi3d_last_error(void) { return g_err.c_str(); }

int jacobi3d_plan(const jacobi3d_config* cfg, jacobi3d_plan_info* out) {
    return guarded([&]() -> int {
        if (!out) return fail(J3D_EINVAL, "out is NULL");
        int rc = validate_cfg(cfg);
        if (rc) return rc;
        Plan P;
        std::string msg;
        rc = make_plan({cfg->gx, cfg->gy, cfg->gz}, {cfg->bx, cfg->by, cfg->bz}, cfg->odf, cfg->n_gpus, P, msg);
        if (rc) return fail(rc, msg);
        std::memset(out, 0, sizeof *out);
        for (int a = 0; a < 3; ++a) {
            out->gpu_grid[a] = P.gpu_grid[a];
            out->blk_grid[a] = P.blk_grid[a];
            out->blk_ext[a] = P.ext[a];
        }
        out->n_blocks = (int64_t)P.blocks.size();
        // bytes: same layout as build_layout
        const int64_t nx = P.ext[0], ny = P.ext[1], nz = P.ext[2];
        const int64_t pitch = align_up(XOFF + nx + 1, PITCH_ALIGN);
        const int64_t grid = align_up(pitch * (ny + 2) * (nz + 2) * 8, 256);
        const int64_t xg = align_up(align_up(ny, 2) * (nz + 2) * 8, 256);  // two x ghost arrays per buffer
        const int64_t buf = grid + 2 * xg;
        int64_t faces = 0;
        for (int f = 0; f < 6; ++f) faces += 4 * align_up(face_cells(P.ext, f) * 8, 256);
        const int64_t head = cfg->launch == J3D_PERSISTENT
                                 ? align_up(4096 + (int64_t)P.odf * nz * ((ny + 7) / 8) * 4, 4096)
                                 : 4096;
        out->bytes_per_gpu = head + (int64_t)P.odf * (2 * buf + faces);
        int32_t pmax = 0;
        for (int r = 0; r < P.n_gpus; ++r) {
            int32_t cnt = 0, loc = 0;
            for (int64_t id : P.by_rank[r])
                for (int f = 0; f < 6; ++f) {
                    const int64_t nb = P.blocks[id].nbr[f];
                    if (nb < 0) continue;
                    if (P.blocks[nb].owner != r) cnt++;
                    else loc++;
                }
            pmax = std::max(pmax, cnt);
            if (r == cfg->rank) out->local_faces = loc;
        }
        out->peer_faces_max = pmax;
        return J3D_OK;
    });
}

int jacobi3d_debug_slab_deps(const jacobi3d_config* cfg, int32_t tile_ty, int32_t nzc, int64_t* host_out,
                             int64_t cap_rows, int64_t* n_rows) {
    return guarded([&]() -> int {
        if (!n_rows) return fail(J3D_EINVAL, "n_rows is NULL");
        int rc = validate_cfg(cfg);
        if (rc) return rc;
        if (tile_ty < 1 || nzc < 1) return fail(J3D_EINVAL, "tile_ty and nzc must be >= 1");
        jacobi3d c;  // host-side state only: plan and face classification, no device
        c.cfg = *cfg;
        c.rank = cfg->rank;
        c.n_gpus = cfg->n_gpus;
        std::string msg;
        rc = make_plan({cfg->gx, cfg->gy, cfg->gz}, {cfg->bx, cfg->by, cfg->bz}, cfg->odf, cfg->n_gpus, c.plan, msg);
        if (rc) return fail(rc, msg);
        if (nzc > c.plan.ext[2]) return fail(J3D_EINVAL, "more z chunks than planes");
        classify(&c);
        const int nty = (int)((c.plan.ext[1] + tile_ty - 1) / tile_ty);
        const auto refs = slab_dep_refs(&c, nzc, nty);
        int64_t rows = 0;
        for (int l = 0; l < c.n_local; ++l)
            for (int zc = 0; zc < nzc; ++zc)
                for (int ty = 0; ty < nty; ++ty)
                    for (const SlabRef& e : refs[((size_t)l * nzc + zc) * nty + ty]) {
                        if (host_out && rows < cap_rows) {
                            int64_t* o = host_out + 7 * rows;
                            o[0] = c.gid[l];
                            o[1] = zc;
                            o[2] = ty;
                            o[3] = e.rank;
                            o[4] = c.plan.by_rank[e.rank][e.local];
                            o[5] = e.zc;
                            o[6] = e.ty;
                        }
                        ++rows;
                    }
        *n_rows = rows;
        return J3D_OK;
    });
}

int jacobi3d_debug_control(const uint8_t* key, int32_t rank, int32_t n_ranks, int64_t rounds, const uint64_t* values,
                           uint64_t* out_sum, uint64_t* out_max) {
    jacobi3d c;  // host-side state only: the control plane of a context, no device
    return guarded([&]() -> int {
        if (!key || !values || !out_sum || !out_max || rounds < 0) return fail(J3D_EINVAL, "NULL argument");
        if (n_ranks < 2 || rank < 0 || rank >= n_ranks) return fail(J3D_EINVAL, "rank / n_ranks out of range");
        c.rank = rank;
        c.n_gpus = n_ranks;
        uint64_t h = 1469598103934665603ULL;  // the job key exactly as jacobi3d_create derives it
        for (int i = 0; i < 128; ++i) h = (h ^ key[i]) * 1099511628211ULL;
        c.job_key = h;
        struct Teardown {
            jacobi3d* p;
            ~Teardown() { ctl_teardown(p); }
        } td{&c};
        ctl_setup_own(&c);
        ctl_connect(&c);
        ctl_barrier(&c);
        for (int64_t r = 0; r < rounds; ++r) {
            out_sum[r] = ctl_reduce(&c, values[r], false);
            out_max[r] = ctl_reduce(&c, values[r], true);
            if (r % 3 == 2) ctl_barrier(&c);
        }
        ctl_barrier(&c);  // every rank has read every slot before the segments go
        return J3D_OK;
    });
}

int jacobi3d_nccl_unique_id(uint8_t out[128]) {
    return guarded([&]() -> int {
        if (!out) return fail(J3D_EINVAL, "out is NULL");
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
        ncclUniqueId id;
        NK(ncclGetUniqueId(&id));
        std::memcpy(out, &id, 128);
        return J3D_OK;
    });
}

int jacobi3d_create(const jacobi3d_config* cfg, const uint8_t* nccl_uid, jacobi3d_t** out) {
    if (out) *out = nullptr;
    jacobi3d* c = nullptr;
    int rc = guarded([&]() -> int {
        if (!out) return fail(J3D_EINVAL, "out is NULL");
        int rc2 = validate_cfg(cfg);
        if (rc2) return rc2;
        if (cfg->n_gpus > 1 && !nccl_uid) return fail(J3D_EINVAL, "nccl_uid required when n_gpus > 1");
        c = new jacobi3d();
        c->cfg = *cfg;
        c->rank = cfg->rank;
        c->n_gpus = cfg->n_gpus;
        c->device = cfg->device;
        std::string msg;
        rc2 = make_plan({cfg->gx, cfg->gy, cfg->gz}, {cfg->bx, cfg->by, cfg->bz}, cfg->odf, cfg->n_gpus, c->plan, msg);
        if (rc2) return fail(rc2, msg);
        CK(cudaSetDevice(c->device));
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, c->device));
        if (prop.major < 10) throw Error(J3D_EUNSUPPORTED, "this build targets sm_100a (B200)");
        c->sms = prop.multiProcessorCount;
        classify(c);
        build_layout(c);
        c->overlap = cfg->overlap && cfg->launch == J3D_BATCHED && c->n_gpus > 1 &&
                     std::any_of(c->has_peer.begin(), c->has_peer.end(), [](uint8_t h) { return h != 0; });
        CK(cudaMalloc(&c->arena, (size_t)c->arena_bytes));
        CK(cudaMemset(c->arena, 0, (size_t)c->off_bufs));  // flags, scratch, persistent counters
        // face buffers start zeroed; done here, before any peer can map the
        // arena, so it can never race with a peer's NVLink stores
        CK(cudaMemset(c->arena + c->off_faces, 0, (size_t)(c->arena_bytes - c->off_faces)));
        CK(cudaMalloc(&c->d_descs, sizeof(StencilDesc) * 2 * c->n_local));
        CK(cudaMalloc(&c->d_tmaps, sizeof(CUtensorMap) * 2 * c->n_local));
        CK(cudaMalloc(&c->d_tmaps_pro, sizeof(CUtensorMap) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_tmaps_x, sizeof(CUtensorMap) * 2 * c->n_local));
        CK(cudaMalloc(&c->d_pack, sizeof(CopyDesc) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_unpack, sizeof(CopyDesc) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_unpack_nccl, sizeof(CopyDesc) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_push, sizeof(CopyDesc) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_pack_peer, sizeof(CopyDesc) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_unpack_peer, sizeof(CopyDesc) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_pack_local, sizeof(CopyDesc) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_unpack_local, sizeof(CopyDesc) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_geom, sizeof(BlockGeom) * c->n_local));
        CK(cudaMalloc(&c->d_sched, sizeof(unsigned int) * 2 * (c->n_local + 1)));
        CK(cudaMemset(c->d_sched, 0, sizeof(unsigned int) * 2 * (c->n_local + 1)));
        if (const char* e = std::getenv("J3D_PEERX_DIRECT")) c->peer_x_direct = std::atoi(e) != 0;
        if (const char* e = std::getenv("J3D_PEERX_PACK")) c->peer_x_pack = std::atoi(e) != 0;
        // a persistent launch has no separate kernels between iterations: every peer
        // face, x included, is stored by the epilogue straight into the peer's ghost layer
        if (cfg->launch == J3D_PERSISTENT) c->peer_x_direct = true;
        c->peer_base.assign(c->n_gpus, nullptr);
        build_static_tables(c);
        build_tables(c);
        CK(preload_kernels(c->tile_kind, c->tile_ys));
        CK(cudaStreamCreateWithFlags(&c->main, cudaStreamNonBlocking));
        int lo_pr = 0, hi_pr = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo_pr, &hi_pr));
        c->block_launches.assign(c->n_local, 0);
        if (cfg->launch == J3D_PER_BLOCK) {
            c->lo.assign(c->n_local, nullptr);
            c->hi.assign(c->n_local, nullptr);
            for (int l = 0; l < c->n_local; ++l) {
                CK(cudaStreamCreateWithPriority(&c->lo[l], cudaStreamNonBlocking, lo_pr));
                CK(cudaStreamCreateWithPriority(&c->hi[l], cudaStreamNonBlocking, hi_pr));
            }
        }
        auto mk = [](cudaEvent_t* e) { CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming)); };
        c->ev_st.assign(c->n_local, {nullptr, nullptr});
        c->ev_pk.assign(c->n_local, {nullptr, nullptr});
        c->ev_up.assign(c->n_local, {nullptr, nullptr});
        for (int l = 0; l < c->n_local; ++l)
            for (int p = 0; p < 2; ++p) {
                mk(&c->ev_st[l][p]);
                mk(&c->ev_pk[l][p]);
                mk(&c->ev_up[l][p]);
            }
        mk(&c->ev_xw[0]);
        mk(&c->ev_xw[1]);
        for (int p = 0; p < 2; ++p) {
            mk(&c->ev_ext[p]);
            mk(&c->ev_comm[p]);
        }
        if (c->overlap) CK(cudaStreamCreateWithPriority(&c->xstream, cudaStreamNonBlocking, hi_pr));
        mk(&c->ev_fork);
        CK(cudaEventCreate(&c->ev_t0));
        CK(cudaEventCreate(&c->ev_t1));
        CK(cudaHostAlloc((void**)&c->host_scratch, 64, cudaHostAllocDefault));
        if (c->n_gpus > 1) {
            uint64_t h = 1469598103934665603ULL;  // FNV-1a of the unique id: a job-wide key
            for (int i = 0; i < 128; ++i) h = (h ^ nccl_uid[i]) * 1099511628211ULL;
            c->job_key = h;
            // NCCL only where halos travel through it; the P2P and host-staging
            // backends use the shared-memory control plane (control.cu)
            if (cfg->exchange == J3D_XCHG_NCCL) {
                ncclUniqueId id;
                std::memcpy(&id, nccl_uid, 128);
                NK(ncclCommInitRank(&c->comm, c->n_gpus, id, c->rank));
            } else {
                c->ctl_needed = true;
                ctl_setup_own(c);
            }
        }
        if (c->host_needed) {
            g_drv.load();
            host_setup_own(c);
        }
        // the arena memsets and table copies ran on the legacy stream; never a
        // device-wide wait (ranks may share this GPU, see sync_streams)
        CK(cudaStreamSynchronize(0));
        CK(cudaStreamSynchronize(c->main));
        *out = c;
        return J3D_OK;
    });
    if (rc != J3D_OK && c) {
        std::string keep = g_err;
        destroy_ctx(c);
        g_err = keep;
    }
    return rc;
}

int jacobi3d_ipc_export(jacobi3d_t* c, uint8_t* host_out, size_t cap, size_t* len) {
    return guarded([&]() -> int {
        if (!c || !len) return fail(J3D_EINVAL, "NULL argument");
        *len = sizeof(IpcRecord);
        if (!host_out || cap < sizeof(IpcRecord)) return fail(J3D_EINVAL, "buffer too small");
        IpcRecord r;
        std::memset(&r, 0, sizeof r);
        r.magic = kIpcMagic;
        r.rank = c->rank;
        r.device = c->device;
        r.arena_bytes = (uint64_t)c->arena_bytes;
        r.process = process_token();
        r.arena_ptr = (uint64_t)(uintptr_t)c->arena;
        CK(cudaSetDevice(c->device));
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, c->device));
        static_assert(sizeof(prop.uuid) == 16, "uuid size");
        std::memcpy(r.uuid, &prop.uuid, 16);
        if (c->p2p_needed) CK(cudaIpcGetMemHandle(&r.handle, c->arena));
        std::memcpy(host_out, &r, sizeof r);
        return J3D_OK;
    });
}

int jacobi3d_ipc_connect(jacobi3d_t* c, const uint8_t* all, size_t len_per_rank) {
    return guarded([&]() -> int {
        if (!c || !all) return fail(J3D_EINVAL, "NULL argument");
        if (c->n_gpus == 1) return J3D_OK;
        if (len_per_rank != sizeof(IpcRecord)) return fail(J3D_EINVAL, "record size mismatch");
        CK(cudaSetDevice(c->device));
        std::vector<IpcRecord> rec(c->n_gpus);
        for (int r = 0; r < c->n_gpus; ++r) {
            std::memcpy(&rec[r], all + (size_t)r * len_per_rank, sizeof(IpcRecord));
            if (rec[r].magic != kIpcMagic || rec[r].rank != r || rec[r].arena_bytes != (uint64_t)c->arena_bytes)
                return fail(J3D_EINVAL, "bad IPC record for rank " + std::to_string(r));
        }
        // ranks on this GPU: threads of this process only.  Separate processes on
        // one GPU are separate CUDA contexts that the GPU time-slices, and our
        // cross-rank waits (epoch flags, persistent slab counters) need the ranks
        // to run at the same time.
        const IpcRecord& me = rec[c->rank];
        c->co_resident = 0;
        for (int r = 0; r < c->n_gpus; ++r) {
            if (std::memcmp(rec[r].uuid, me.uuid, 16) != 0) continue;
            c->co_resident += 1;
            if (rec[r].process != me.process && c->cfg.exchange != J3D_XCHG_NCCL)
                return fail(J3D_EUNSUPPORTED, "ranks " + std::to_string(c->rank) + " and " + std::to_string(r) +
                                                  " share a GPU from different processes; run ranks that share a "
                                                  "GPU as threads of one process (dist.ThreadGroup)");
        }
        bool shared = false;  // some GPU of the job hosts more than one rank (the same answer on every rank)
        for (int a = 0; a < c->n_gpus && !shared; ++a)
            for (int b = a + 1; b < c->n_gpus && !shared; ++b) shared = std::memcmp(rec[a].uuid, rec[b].uuid, 16) == 0;
        if (shared && c->cfg.use_graph)
            return fail(J3D_EUNSUPPORTED, "use_graph with ranks sharing a GPU: graph launches of one CUDA context share "
                                          "its internal streams, so one rank's captured epoch wait can block the "
                                          "peer work it waits for");
        c->persist_grid = std::max(1, c->grid_cap / std::max(1, c->co_resident));
        if (c->co_resident > 1) {
            // ranks sharing this GPU: every stream at the default priority.  High-priority
            // streams of one context share few hardware queues, so one rank's epoch wait on
            // its overlap exchange stream could sit in front of the peer's signal (seen as
            // intermittent hangs of the overlap mode with 2 and 4 thread ranks); no work has
            // been queued on these streams yet
            // ranks sharing this GPU: ONE stream per rank.  The per-block streams and the
            // overlap mode's exchange stream become the main stream (same launches in the
            // same order, no concurrency inside a rank): with several streams per rank,
            // one of which waits on peers' flags, runs deadlocked intermittently (overlap:
            // 1 in ~10-40 runs at 2 and 4 thread ranks; per-block: 1 in ~4 suites) -- a
            // hardware queue shared with a peer's stream; no work has been queued on
            // these streams yet
            for (auto* v : {&c->lo, &c->hi})
                for (auto& st : *v) {
                    CK(cudaStreamDestroy(st));
                    st = c->main;
                }
            c->streams_aliased = true;
            if (c->xstream) {
                CK(cudaStreamDestroy(c->xstream));
                c->xstream = nullptr;
            }
        }
        if (c->host_needed && !c->host_connected) host_connect(c);
        if (c->ctl_needed && !c->ctl_connected) ctl_connect(c);
        if (c->p2p_needed && !c->p2p_connected) {
            c->peer_ipc.assign(c->n_gpus, 0);
            for (int r : c->peer_ranks) {
                const IpcRecord& pr = rec[r];
                if (pr.device != c->device || pr.process != me.process) {
                    int can = 0;
                    CK(cudaDeviceCanAccessPeer(&can, c->device, pr.device));
                    if (!can && std::memcmp(pr.uuid, me.uuid, 16) != 0)
                        return fail(J3D_EUNSUPPORTED, "device " + std::to_string(c->device) +
                                                          " cannot access peer device " + std::to_string(pr.device));
                }
                if (pr.process == me.process) {  // a thread of this process: its arena address as is
                    if (pr.device != c->device) {
                        cudaError_t e = cudaDeviceEnablePeerAccess(pr.device, 0);
                        if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
                        else CK(e);
                    }
                    c->peer_base[r] = (char*)(uintptr_t)pr.arena_ptr;
                } else {
                    void* p = nullptr;
                    CK(cudaIpcOpenMemHandle(&p, pr.handle, cudaIpcMemLazyEnablePeerAccess));
                    c->peer_base[r] = (char*)p;
                    c->peer_ipc[r] = 1;
                }
            }
            c->p2p_connected = true;
            drop_graphs(c);
            build_tables(c);
        }
        CK(cudaStreamSynchronize(0));
        CK(cudaStreamSynchronize(c->main));
        // every rank connected before any rank enqueues work that waits on a peer
        ctl_barrier(c);
        return J3D_OK;
    });
}

int jacobi3d_init(jacobi3d_t* c, int kind, const double* p, uint64_t seed) {
    return guarded([&]() -> int {
        if (!c) return fail(J3D_EINVAL, "ctx is NULL");
        if (kind < J3D_INIT_DEFAULT || kind > J3D_INIT_HASH) return fail(J3D_EINVAL, "unknown init kind");
        if ((kind == J3D_INIT_CONST || kind == J3D_INIT_LINEAR) && !p) return fail(J3D_EINVAL, "params required");
        if ((c->p2p_needed && !c->p2p_connected) || (c->host_needed && !c->host_connected) ||
            (c->ctl_needed && !c->ctl_connected))
            return fail(J3D_ESTATE, "a multi-GPU context needs jacobi3d_ipc_export/jacobi3d_ipc_connect first");
        CK(cudaSetDevice(c->device));
        double pp[4] = {0, 0, 0, 0};
        if (p) std::memcpy(pp, p, sizeof pp);
        CK(launch_init(c->d_geom, c->n_local, (int)c->nx, (c->ny + 2) * (c->nz + 2), kind, pp, seed,
                       c->cfg.boundary, c->cfg.gx, c->cfg.gy, c->cfg.gz, c->main));
        count_launch(c, -1);
        c->iter = 0;
        c->iter_since_set = 0;
        c->halos_stale = false;
        // every collective state change ends with one exchange, which keeps the
        // epoch-slot sequence alternating and fills the
        // receive buffers the fused prologue reads
        refresh(c, 0);
        return J3D_OK;
    });
}

int jacobi3d_refresh_halos(jacobi3d_t* c) {
    return guarded([&]() -> int {
        if (!c) return fail(J3D_EINVAL, "ctx is NULL");
        CK(cudaSetDevice(c->device));
        refresh(c, (int)(c->iter & 1));
        c->halos_stale = false;
        return J3D_OK;
    });
}

static int block_local(jacobi3d* c, int64_t id, int* l) {
    if (id < 0 || id >= (int64_t)c->plan.blocks.size()) return fail(J3D_EINVAL, "block id out of range");
    const BlockPlan& b = c->plan.blocks[id];
    if (b.owner != c->rank) return fail(J3D_ENOTLOCAL, "block " + std::to_string(id) + " is on rank " + std::to_string(b.owner));
    *l = b.local;
    return J3D_OK;
}

static cudaMemcpy3DParms owned_copy(jacobi3d* c, int l, int par, double* host, bool to_host) {
    cudaMemcpy3DParms m;
    std::memset(&m, 0, sizeof m);
    double* dev = c->buf(l, par) + c->zs + c->pitch + XOFF;
    cudaPitchedPtr d = make_cudaPitchedPtr(dev, (size_t)c->pitch * 8, (size_t)c->nx, (size_t)(c->ny + 2));
    cudaPitchedPtr h = make_cudaPitchedPtr(host, (size_t)c->nx * 8, (size_t)c->nx, (size_t)c->ny);
    if (to_host) {
        m.srcPtr = d;
        m.dstPtr = h;
        m.kind = cudaMemcpyDeviceToHost;
    } else {
        m.srcPtr = h;
        m.dstPtr = d;
        m.kind = cudaMemcpyHostToDevice;
    }
    m.extent = make_cudaExtent((size_t)c->nx * 8, (size_t)c->ny, (size_t)c->nz);
    return m;
}

int jacobi3d_set_block(jacobi3d_t* c, int64_t id, const double* host_in) {
    return guarded([&]() -> int {
        if (!c || !host_in) return fail(J3D_EINVAL, "NULL argument");
        int l = 0;
        int rc = block_local(c, id, &l);
        if (rc) return rc;
        CK(cudaSetDevice(c->device));
        cudaMemcpy3DParms m = owned_copy(c, l, (int)(c->iter & 1), const_cast<double*>(host_in), false);
        CK(cudaMemcpy3DAsync(&m, c->main));
        wait_stream(c, c->main);
        c->halos_stale = true;
        c->iter_since_set = 0;
        return J3D_OK;
    });
}

int jacobi3d_get_block(jacobi3d_t* c, int64_t id, double* host_out) {
    return guarded([&]() -> int {
        if (!c || !host_out) return fail(J3D_EINVAL, "NULL argument");
        int l = 0;
        int rc = block_local(c, id, &l);
        if (rc) return rc;
        CK(cudaSetDevice(c->device));
        cudaMemcpy3DParms m = owned_copy(c, l, (int)(c->iter & 1), host_out, true);
        CK(cudaMemcpy3DAsync(&m, c->main));
        wait_stream(c, c->main);
        return J3D_OK;
    });
}

int jacobi3d_get_region(jacobi3d_t* c, int64_t id, const int64_t lo[3], const int64_t ext[3], double* host_out) {
    return guarded([&]() -> int {
        if (!c || !lo || !ext || !host_out) return fail(J3D_EINVAL, "NULL argument");
        int l = 0;
        int rc = block_local(c, id, &l);
        if (rc) return rc;
        const int64_t n[3] = {c->nx, c->ny, c->nz};
        for (int a = 0; a < 3; ++a)
            if (lo[a] < 0 || ext[a] < 1 || lo[a] + ext[a] > n[a]) return fail(J3D_EINVAL, "region outside the block");
        CK(cudaSetDevice(c->device));
        cudaMemcpy3DParms m;
        std::memset(&m, 0, sizeof m);
        double* dev = c->buf(l, (int)(c->iter & 1)) + (lo[2] + 1) * c->zs + (lo[1] + 1) * c->pitch + XOFF + lo[0];
        m.srcPtr = make_cudaPitchedPtr(dev, (size_t)c->pitch * 8, (size_t)ext[0], (size_t)(c->ny + 2));
        m.dstPtr = make_cudaPitchedPtr(host_out, (size_t)ext[0] * 8, (size_t)ext[0], (size_t)ext[1]);
        m.kind = cudaMemcpyDeviceToHost;
        m.extent = make_cudaExtent((size_t)ext[0] * 8, (size_t)ext[1], (size_t)ext[2]);
        CK(cudaMemcpy3DAsync(&m, c->main));
        wait_stream(c, c->main);
        return J3D_OK;
    });
}

int jacobi3d_block_info(jacobi3d_t* c, int64_t id, int64_t origin[3], int64_t extent[3], int32_t* owner) {
    return guarded([&]() -> int {
        if (!c) return fail(J3D_EINVAL, "ctx is NULL");
        if (id < 0 || id >= (int64_t)c->plan.blocks.size()) return fail(J3D_EINVAL, "block id out of range");
        const BlockPlan& b = c->plan.blocks[id];
        for (int a = 0; a < 3; ++a) {
            if (origin) origin[a] = b.origin[a];
            if (extent) extent[a] = c->plan.ext[a];
        }
        if (owner) *owner = b.owner;
        return J3D_OK;
    });
}

int jacobi3d_iterate(jacobi3d_t* c, int64_t n) {
    return guarded([&]() -> int {
        if (!c) return fail(J3D_EINVAL, "ctx is NULL");
        if (n < 0) return fail(J3D_EINVAL, "n must be >= 0");
        CK(cudaSetDevice(c->device));
        do_iterate(c, n);
        return J3D_OK;
    });
}

int jacobi3d_synchronize(jacobi3d_t* c) {
    return guarded([&]() -> int {
        if (!c) return fail(J3D_EINVAL, "ctx is NULL");
        CK(cudaSetDevice(c->device));
        sync_streams(c);
        if (c->comm) {
            ncclResult_t ar = ncclSuccess;
            NK(ncclCommGetAsyncError(c->comm, &ar));
            NK(ar);
        }
        return J3D_OK;
    });
}

int jacobi3d_residual(jacobi3d_t* c, double* out) {
    return guarded([&]() -> int {
        if (!c || !out) return fail(J3D_EINVAL, "NULL argument");
        if (c->iter_since_set < 1) return fail(J3D_ESTATE, "residual needs >= 1 iteration since init/set_block");
        CK(cudaSetDevice(c->device));
        unsigned long long* acc = (unsigned long long*)(c->arena + c->off_scratch);
        CK(cudaMemsetAsync(acc, 0, 8, c->main));
        CK(launch_residual(c->d_geom, c->n_local, (int)(c->iter & 1), acc, c->sms, c->main));
        count_launch(c, -1);
        if (c->comm) NK(ncclAllReduce(acc, acc, 1, ncclUint64, ncclMax, c->comm, c->main));
        // into pinned scratch, then the watchdog-polled wait (a pageable copy would
        // block in the driver, past the watchdog, if a peer had stopped)
        CK(cudaMemcpyAsync(c->host_scratch, acc, 8, cudaMemcpyDeviceToHost, c->main));
        wait_stream(c, c->main);
        uint64_t h = c->host_scratch[0];
        if (!c->comm) h = ctl_reduce(c, h, true);  // |differences| order like their bits; NaN wins
        double d;
        std::memcpy(&d, &h, 8);
        *out = d;
        return J3D_OK;
    });
}

int jacobi3d_checksum(jacobi3d_t* c, uint64_t* out) {
    return guarded([&]() -> int {
        if (!c || !out) return fail(J3D_EINVAL, "NULL argument");
        CK(cudaSetDevice(c->device));
        unsigned long long* acc = (unsigned long long*)(c->arena + c->off_scratch + 8);
        CK(cudaMemsetAsync(acc, 0, 8, c->main));
        CK(launch_checksum(c->d_geom, c->n_local, (int)(c->iter & 1), c->cfg.gx, c->cfg.gy, acc, c->sms, c->main));
        count_launch(c, -1);
        if (c->comm) NK(ncclAllReduce(acc, acc, 1, ncclUint64, ncclSum, c->comm, c->main));
        CK(cudaMemcpyAsync(c->host_scratch + 1, acc, 8, cudaMemcpyDeviceToHost, c->main));
        wait_stream(c, c->main);
        uint64_t h = c->host_scratch[1];
        if (!c->comm) h = ctl_reduce(c, h, false);
        *out = h;
        return J3D_OK;
    });
}

int jacobi3d_time(jacobi3d_t* c, int64_t warmup, int64_t iters, double* ms) {
    return guarded([&]() -> int {
        if (!c || !ms || iters < 1 || warmup < 0) return fail(J3D_EINVAL, "bad argument");
        CK(cudaSetDevice(c->device));
        do_iterate(c, warmup);
        sync_streams(c);
        ctl_barrier(c);
        CK(cudaEventRecord(c->ev_t0, c->main));
        do_iterate(c, iters);
        CK(cudaEventRecord(c->ev_t1, c->main));
        wait_stream(c, c->main);
        CK(cudaEventSynchronize(c->ev_t1));
        float f = 0;
        CK(cudaEventElapsedTime(&f, c->ev_t0, c->ev_t1));
        *ms = (double)f / (double)iters;
        return J3D_OK;
    });
}

int jacobi3d_get_stats(jacobi3d_t* c, jacobi3d_stats* out) {
    return guarded([&]() -> int {
        if (!c || !out) return fail(J3D_EINVAL, "NULL argument");
        std::memset(out, 0, sizeof *out);
        out->iterations = c->iter;
        out->kernel_launches = c->stat_launches;
        out->graph_launches = c->stat_graph_launches;
        out->last_graph_parity = c->stat_last_parity;
        int64_t mx = 0;
        for (int64_t v : c->block_launches) mx = std::max(mx, v);
        out->launches_per_iter_block = c->stat_iters > 0 ? mx / c->stat_iters : 0;
        out->tile_kind = c->tile_kind;
        out->work_items = c->n_items;
        return J3D_OK;
    });
}

int jacobi3d_reset_stats(jacobi3d_t* c) {
    if (!c) return fail(J3D_EINVAL, "ctx is NULL");
    c->stat_launches = c->stat_graph_launches = c->stat_iters = 0;
    c->stat_last_parity = -1;
    std::fill(c->block_launches.begin(), c->block_launches.end(), 0);
    return J3D_OK;
}

int jacobi3d_profile_enable(jacobi3d_t* c, int enable) {
    return guarded([&]() -> int {
        if (!c) return fail(J3D_EINVAL, "ctx is NULL");
        CK(cudaSetDevice(c->device));
        sync_streams(c);
        for (auto& pr : c->prof_events) {
            c->ev_pool.push_back(pr.first);
            c->ev_pool.push_back(pr.second);
        }
        c->prof_events.clear();
        c->prof = enable != 0;
        c->prof_ms = c->prof_bytes = c->prof_pending_bytes = 0;
        c->prof_launches = 0;
        return J3D_OK;
    });
}

int jacobi3d_profile_read(jacobi3d_t* c, double* total_ms, int64_t* launches, double* bytes) {
    return guarded([&]() -> int {
        if (!c) return fail(J3D_EINVAL, "ctx is NULL");
        CK(cudaSetDevice(c->device));
        sync_streams(c);
        for (auto& pr : c->prof_events) {
            float f = 0;
            CK(cudaEventElapsedTime(&f, pr.first, pr.second));
            c->prof_ms += f;
            c->prof_launches += 1;
            c->ev_pool.push_back(pr.first);
            c->ev_pool.push_back(pr.second);
        }
        c->prof_events.clear();
        c->prof_bytes += c->prof_pending_bytes;
        c->prof_pending_bytes = 0;
        if (total_ms) *total_ms = c->prof_ms;
        if (launches) *launches = c->prof_launches;
        if (bytes) *bytes = c->prof_bytes;
        return J3D_OK;
    });
}

int jacobi3d_set_skip_exchange(jacobi3d_t* c, int skip) {
    if (!c) return fail(J3D_EINVAL, "ctx is NULL");
    if ((skip != 0) != c->skip_exchange) drop_graphs(c);
    c->skip_exchange = skip != 0;
    return J3D_OK;
}

int jacobi3d_div7_selftest(uint64_t n, uint64_t seed, uint64_t* mismatches, double* example) {
    return guarded([&]() -> int {
        if (!mismatches) return fail(J3D_EINVAL, "NULL argument");
        int dev = 0, sms = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        unsigned long long* d = nullptr;
        CK(cudaMalloc(&d, 64));
        CK(cudaMemset(d, 0, 64));
        cudaError_t e = launch_div7_selftest(n, seed, d, (double*)(d + 1), sms, 0);
        unsigned long long h[4] = {0, 0, 0, 0};
        if (e == cudaSuccess) e = cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        cudaFree(d);
        CK(e);
        *mismatches = h[0];
        if (example) std::memcpy(example, h + 1, 24);
        return J3D_OK;
    });
}

int jacobi3d_destroy(jacobi3d_t* c) {
    return guarded([&]() -> int {
        destroy_ctx(c);
        return J3D_OK;
    });
}

}  // extern "C"
