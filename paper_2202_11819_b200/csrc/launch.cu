// launch.cu -- kernel launches and the per-iteration orchestration: per-block prioritised streams, batched launches, the overlap split, the two parity CUDA graphs, waits.
#include "context.h"

using namespace j3d;

namespace j3d {

cudaEvent_t pool_event(jacobi3d* c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
}

// ---------------------------------------------------------------- launches
void count_launch(jacobi3d* c, int l) {
    if (c->capturing) {
        c->graph_kernels[c->capture_parity] += 1;
        if (l >= 0) c->graph_block_launches[c->capture_parity][l] += 1;
    } else {
        c->stat_launches += 1;
        if (l >= 0) c->block_launches[l] += 1;
    }
}

// Limit for the persistent launch's on-device counter waits: the host-wait
// watchdog's J3D_TIMEOUT_S (default 600 s), so a legitimately late peer rank
// is waited for as long as the host would wait for it.
static uint64_t wait_limit_ns() { return (uint64_t)(timeout_s() * 1e9); }

void stencil(jacobi3d* c, int begin, int count, int parity, cudaStream_t st, int l) {
    if (count <= 0) return;
    Nvtx nv("j3d.stencil");
    StencilLaunch L;
    L.descs = c->d_descs;
    L.tmaps = c->d_tmaps;
    L.tmaps_pro = c->d_tmaps_pro;
    L.tmaps_x = c->d_tmaps_x;
    L.tma_mode = c->tma_mode;
    L.items = c->d_items + begin;
    L.n_items = count;
    L.parity = parity;
    L.grid = std::min(count, c->grid_cap);
    L.kind = c->tile_kind;
    L.faces = c->faces_fused;
    L.yside = c->tile_ys;
    L.prefetch = c->prefetch;
    L.depfence = c->depfence;
    L.sched = c->d_sched + 2 * (l + 1);  // one counter pair per concurrently running launch
    L.ctl = IterCtl{nullptr, nullptr, nullptr, 1, 0, 0, 0, 0};
    const int n_iter = c->persist_n;
    if (n_iter > 0) {  // J3D_PERSISTENT: n_iter iterations in this one launch
        const bool remote = c->n_remote_done > 0 && !c->skip_exchange;
        L.ctl = IterCtl{c->d_item_slab, remote ? c->d_slab_deps : c->d_slab_deps_local, c->d_done, n_iter,
                        c->slab_target, c->persist_base, remote ? 1 : 0, wait_limit_ns()};
        // ranks sharing this GPU (threads of one process) split it, so that every
        // rank's persistent grid is resident at once: their items wait on each other
        L.grid = c->persist_grid > 0 ? c->persist_grid : c->grid_cap;
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    const bool prof = c->prof && !c->capturing;
    if (prof) {
        e0 = pool_event(c);
        e1 = pool_event(c);
        CK(cudaEventRecord(e0, st));
    }
    CK(launch_stencil(L, st));
    count_launch(c, l);
    if (prof) {
        CK(cudaEventRecord(e1, st));
        c->prof_events.push_back({e0, e1});
        const int64_t cells = c->item_cells[begin + count] - c->item_cells[begin];  // exact owned cells updated
        c->prof_pending_bytes += 16.0 * (double)cells * (double)std::max(1, n_iter);
    }
}

void copies(jacobi3d* c, CopyDesc* table, int parity, int l, int face, bool fused, cudaStream_t st) {
    // table layout [(q*nl + l)*6 + f]
    const bool unpack = table == c->d_unpack || table == c->d_unpack_nccl || table == c->d_unpack_peer ||
                        table == c->d_unpack_local;
    Nvtx nv(unpack ? "j3d.unpack" : table == c->d_push ? "j3d.push" : "j3d.pack");
    const int nl = c->n_local;
    if (l < 0) {  // batched: every local block, fused over faces
        int64_t mx = 0;
        for (int f = 0; f < 6; ++f) mx = std::max<int64_t>(mx, face_cells(c->plan.ext, f));
        CK(launch_copy_faces(table + (int64_t)parity * nl * 6, 6, nl, mx, st));
        count_launch(c, -1);
        return;
    }
    CopyDesc* base = table + ((int64_t)parity * nl + l) * 6;
    if (fused) {
        int64_t mx = 0;
        for (int f = 0; f < 6; ++f)
            if (c->kind[l][f] != DIRICHLET) mx = std::max<int64_t>(mx, face_cells(c->plan.ext, f));
        if (mx == 0) return;
        CK(launch_copy_faces(base, 6, 1, mx, st));
        count_launch(c, l);
    } else {
        CK(launch_copy_faces(base + face, 1, 1, face_cells(c->plan.ext, face), st));
        count_launch(c, l);
    }
}

// Full halo refresh of buffer parity `par`: pack, exchange, unpack, batched on
// main.  With P2P peers it starts with an epoch barrier (slots 4/5): a peer's
// NVLink stores into our receive buffers may only begin once we have finished
// every earlier use of them (the caller's state change, e.g. init or
// set_block, or the last iteration of a previous run).
void refresh(jacobi3d* c, int par) {
    Nvtx nv("j3d.refresh");
    const int rc = (int)(c->refresh_count & 1);
    c->refresh_count++;
    if (c->n_gpus > 1) {
        p2p_sync(c, 4 + rc, c->main);
        host_sync(c, 4 + rc, c->main);
    }
    copies(c, c->d_pack, par, -1, 0, true, c->main);
    if (c->n_gpus > 1) {
        nccl_exchange(c, par, c->main);
        p2p_sync(c, 2 + rc, c->main);
        host_exchange(c, par, 2 + rc, c->main);
    }
    copies(c, c->d_unpack, par, -1, 0, true, c->main);
}

void fork_streams(jacobi3d* c) {
    CK(cudaEventRecord(c->ev_fork, c->main));
    for (int l = 0; l < c->n_local; ++l) {
        CK(cudaStreamWaitEvent(c->lo[l], c->ev_fork, 0));
        if (unfused_family(c)) CK(cudaStreamWaitEvent(c->hi[l], c->ev_fork, 0));
    }
}

void join_streams(jacobi3d* c, int q) {
    for (int l = 0; l < c->n_local; ++l) {
        CK(cudaStreamWaitEvent(c->main, c->ev_st[l][q], 0));
        if (unfused_family(c)) CK(cudaStreamWaitEvent(c->main, c->ev_up[l][q], 0));
    }
}

// One iteration with input parity p.  `first`: the streams must be forked
// from main (start of an iterate() call, or graph capture).
void enqueue_iteration(jacobi3d* c, int p, bool first, bool last) {
    const int q = p ^ 1;
    const int v = c->cfg.variant;
    const bool unf = unfused_family(c);
    if (c->cfg.launch == J3D_BATCHED) {
        if (c->overlap && !c->skip_exchange) {
            // exterior items (those touching a peer face) first; the exchange
            // of their faces runs on `comm` while the interior items update
            // (Fig 1 manual overlap, L79-107; ODF-driven overlap, L146-156)
            // (ranks sharing a GPU: no exchange stream, the exchange runs on main; api.cu)
            cudaStream_t xs = c->xstream ? c->xstream : c->main;
            stencil(c, 0, c->n_ext, p, c->main, -1);
            CK(cudaEventRecord(c->ev_ext[q], c->main));
            CK(cudaStreamWaitEvent(xs, c->ev_ext[q], 0));
            if (unf) copies(c, c->d_pack_peer, q, -1, 0, true, xs);
            else if (c->direct_push) copies(c, c->d_push, q, -1, 0, true, xs);
            cross_gpu_exchange(c, q, q, xs);
            if (unf) copies(c, c->d_unpack_peer, q, -1, 0, true, xs);
            else if (c->direct_nccl_unpack) copies(c, c->d_unpack_nccl, q, -1, 0, true, xs);
            CK(cudaEventRecord(c->ev_comm[q], xs));
            stencil(c, c->n_ext, c->n_items - c->n_ext, p, c->main, -1);
            if (unf) {
                copies(c, c->d_pack_local, q, -1, 0, true, c->main);
                copies(c, c->d_unpack_local, q, -1, 0, true, c->main);
            }
            CK(cudaStreamWaitEvent(c->main, c->ev_comm[q], 0));
            return;
        }
        stencil(c, 0, c->n_items, p, c->main, -1);
        if (unf) copies(c, c->d_pack, q, -1, 0, true, c->main);
        else if (c->direct_push && !c->skip_exchange) copies(c, c->d_push, q, -1, 0, true, c->main);
        cross_gpu_exchange(c, q, q, c->main);
        if (unf) copies(c, c->d_unpack, q, -1, 0, true, c->main);
        else if (c->direct_nccl_unpack && !c->skip_exchange) copies(c, c->d_unpack_nccl, q, -1, 0, true, c->main);
        return;
    }
    // ---- per-block streams
    const bool cap = c->capturing;
    if (first) fork_streams(c);
    const bool peers = c->n_gpus > 1 && !c->skip_exchange &&
                       std::any_of(c->has_peer.begin(), c->has_peer.end(), [](uint8_t h) { return h != 0; });
    for (int l : c->order) {
        cudaStream_t s = c->lo[l];
        if (!cap && !first) {
            if (unf) {
                CK(cudaStreamWaitEvent(s, c->ev_up[l][p], 0));
            } else {
                for (int f = 0; f < 6; ++f)
                    if (c->kind[l][f] == LOCAL) CK(cudaStreamWaitEvent(s, c->ev_st[c->nbr_local[l][f]][p], 0));
                if (c->has_peer[l] && peers) CK(cudaStreamWaitEvent(s, c->ev_xw[p], 0));
            }
        }
        stencil(c, c->item_begin[l], c->item_count[l], p, s, l);
        CK(cudaEventRecord(c->ev_st[l][q], s));
    }
    if (unf) {
        for (int l : c->order) {
            cudaStream_t s = c->hi[l];
            CK(cudaStreamWaitEvent(s, c->ev_st[l][q], 0));
            if (v == J3D_UNFUSED) {
                for (int f = 0; f < 6; ++f)
                    if (c->kind[l][f] != DIRICHLET) copies(c, c->d_pack, q, l, f, false, s);
            } else {
                copies(c, c->d_pack, q, l, 0, true, s);
            }
            CK(cudaEventRecord(c->ev_pk[l][q], s));
        }
    }
    if (peers) {
        for (int l = 0; l < c->n_local; ++l)
            if (c->has_peer[l]) CK(cudaStreamWaitEvent(c->main, unf ? c->ev_pk[l][q] : c->ev_st[l][q], 0));
        if (!unf && c->direct_push) copies(c, c->d_push, q, -1, 0, true, c->main);
        cross_gpu_exchange(c, q, q, c->main);
        if (!unf && c->direct_nccl_unpack) copies(c, c->d_unpack_nccl, q, -1, 0, true, c->main);
        CK(cudaEventRecord(c->ev_xw[q], c->main));
    }
    if (unf) {
        for (int l : c->order) {
            cudaStream_t s = c->hi[l];
            if (v == J3D_FUSE_B) {  // one fused unpack after ALL faces arrived
                for (int f = 0; f < 6; ++f)
                    if (c->kind[l][f] == LOCAL) CK(cudaStreamWaitEvent(s, c->ev_pk[c->nbr_local[l][f]][q], 0));
                if (c->has_peer[l] && peers) CK(cudaStreamWaitEvent(s, c->ev_xw[q], 0));
                copies(c, c->d_unpack, q, l, 0, true, s);
            } else {  // one unpack per face, each after its own face arrived
                for (int f = 0; f < 6; ++f) {
                    const int k = c->kind[l][f];
                    if (k == DIRICHLET) continue;
                    if (k == LOCAL) CK(cudaStreamWaitEvent(s, c->ev_pk[c->nbr_local[l][f]][q], 0));
                    else if (peers) CK(cudaStreamWaitEvent(s, c->ev_xw[q], 0));
                    copies(c, c->d_unpack, q, l, f, false, s);
                }
            }
            CK(cudaEventRecord(c->ev_up[l][q], s));
        }
    }
    if (last) join_streams(c, q);
}

void capture_graph(jacobi3d* c, int p) {
    c->graph_kernels[p] = 0;
    c->graph_block_launches[p].assign(c->n_local, 0);
    CK(cudaStreamBeginCapture(c->main, cudaStreamCaptureModeThreadLocal));
    c->capturing = true;
    c->capture_parity = p;
    try {
        enqueue_iteration(c, p, true, true);
    } catch (...) {
        c->capturing = false;
        cudaGraph_t g;
        cudaStreamEndCapture(c->main, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    c->capturing = false;
    cudaGraph_t g = nullptr;
    CK(cudaStreamEndCapture(c->main, &g));
    cudaError_t e = cudaGraphInstantiate(&c->graph[p], g, 0);
    cudaGraphDestroy(g);
    CK(e);
}

void drop_graphs(jacobi3d* c) {
    for (int p = 0; p < 2; ++p)
        if (c->graph[p]) {
            cudaGraphExecDestroy(c->graph[p]);
            c->graph[p] = nullptr;
        }
}

void do_iterate(jacobi3d* c, int64_t n) {
    if (n <= 0) return;
    Nvtx nv("j3d.iterate");
    if (c->halos_stale) {
        if (c->n_gpus > 1)
            throw Error(J3D_ESTATE, "halos are stale after set_block: call jacobi3d_refresh_halos on every rank");
        refresh(c, (int)(c->iter & 1));
        c->halos_stale = false;
    }
    if (c->p2p_needed && !c->p2p_connected)
        throw Error(J3D_ESTATE, "P2P exchange needs jacobi3d_ipc_export/jacobi3d_ipc_connect first");
    if (c->cfg.launch == J3D_PERSISTENT) {
        // one launch per call (split only to keep n x items inside the 32-bit work counter)
        const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(1 << 20, INT32_MAX / std::max(1, c->n_items)));
        for (int64_t left = n; left > 0;) {
            const int m = (int)std::min(left, cap);
            c->persist_n = m;
            stencil(c, 0, c->n_items, (int)(c->iter & 1), c->main, -1);
            c->persist_n = 0;
            c->persist_base += (uint32_t)m;
            if (c->n_remote_done > 0 && !c->skip_exchange) {  // peers' writes into this GPU have landed
                CK(launch_wait_counters(c->d_remote_done, c->n_remote_done, c->persist_base * c->slab_target,
                                        wait_limit_ns(), c->main));
                count_launch(c, -1);
            }
            c->iter += m;
            c->iter_since_set += m;
            c->stat_iters += m;
            left -= m;
        }
        return;
    }
    for (int64_t k = 0; k < n; ++k) {
        const int p = (int)(c->iter & 1);
        if (c->cfg.use_graph) {
            if (!c->graph[p]) capture_graph(c, p);
            CK(cudaGraphLaunch(c->graph[p], c->main));
            c->stat_graph_launches += 1;
            c->stat_last_parity = p;
            c->stat_launches += c->graph_kernels[p];
            for (int l = 0; l < c->n_local; ++l) c->block_launches[l] += c->graph_block_launches[p][l];
        } else {
            enqueue_iteration(c, p, k == 0, k == n - 1);
        }
        c->iter += 1;
        c->iter_since_set += 1;
        c->stat_iters += 1;
    }
}

void destroy_ctx(jacobi3d* c) {
    if (!c) return;
    // J3D_TRACE_DESTROY=1: print each step (diagnosing teardown of thread ranks)
    static const bool trace = std::getenv("J3D_TRACE_DESTROY") != nullptr;
    auto step = [&](const char* what) {
        if (trace) std::fprintf(stderr, "[j3d destroy rank %d] %s\n", c->rank, what), std::fflush(stderr);
    };
    cudaSetDevice(c->device);
    step("sync");
    try {
        sync_streams(c);
    } catch (...) {
        step("sync timed out");
    }
    step("barrier");
    // collective (jacobi3d.h): once every rank is here no peer still touches this
    // rank's arena -- persistent launches read the peers' slab counters over NVLink
    // until their own last iteration -- so freeing it cannot fault a slower peer
    bool abort_comm = false;
    if (c->n_gpus > 1 && (c->comm || c->ctl_connected)) {
        try {
            ctl_barrier(c);
        } catch (...) {
            abort_comm = true;
        }
    }
    step("graphs/events/streams");
    drop_graphs(c);
    for (auto& pr : c->prof_events) {
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
    }
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    for (auto& a : c->ev_st) for (auto e : a) if (e) cudaEventDestroy(e);
    for (auto& a : c->ev_pk) for (auto e : a) if (e) cudaEventDestroy(e);
    for (auto& a : c->ev_up) for (auto e : a) if (e) cudaEventDestroy(e);
    for (auto e : c->ev_xw) if (e) cudaEventDestroy(e);
    for (auto e : c->ev_ext) if (e) cudaEventDestroy(e);
    for (auto e : c->ev_comm) if (e) cudaEventDestroy(e);
    if (c->xstream) cudaStreamDestroy(c->xstream);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_t0) cudaEventDestroy(c->ev_t0);
    if (c->ev_t1) cudaEventDestroy(c->ev_t1);
    if (!c->streams_aliased) {
        for (auto s : c->lo) if (s) cudaStreamDestroy(s);
        for (auto s : c->hi) if (s) cudaStreamDestroy(s);
    }
    if (c->comm) {
        if (abort_comm) ncclCommAbort(c->comm);
        else ncclCommDestroy(c->comm);
    }
    step("ipc/host/ctl");
    for (size_t r = 0; r < c->peer_base.size(); ++r)
        if (c->peer_base[r] && r < c->peer_ipc.size() && c->peer_ipc[r]) cudaIpcCloseMemHandle(c->peer_base[r]);
    host_teardown(c);
    ctl_teardown(c);
    step("free host scratch");
    if (c->host_scratch) cudaFreeHost(c->host_scratch);
    step("free device");
    if (c->main) cudaStreamDestroy(c->main);
    cudaFree(c->d_descs);
    cudaFree(c->d_tmaps);
    cudaFree(c->d_tmaps_pro);
    cudaFree(c->d_tmaps_x);
    cudaFree(c->d_items);
    cudaFree(c->d_pack);
    cudaFree(c->d_unpack);
    cudaFree(c->d_unpack_nccl);
    cudaFree(c->d_stage_out);
    cudaFree(c->d_stage_in);
    cudaFree(c->d_push);
    cudaFree(c->d_item_slab);
    cudaFree(c->d_slab_deps);
    cudaFree(c->d_slab_deps_local);
    cudaFree(c->d_remote_done);
    cudaFree(c->d_pack_peer);
    cudaFree(c->d_unpack_peer);
    cudaFree(c->d_pack_local);
    cudaFree(c->d_unpack_local);
    cudaFree(c->d_geom);
    cudaFree(c->d_sched);
    cudaFree(c->arena);
    step("done");
    delete c;
}

// Host wait for all work queued on `st`.  Multi-GPU contexts poll with a
// watchdog (J3D_TIMEOUT_S, default 600 s): a peer that never signals its
// epoch (or an NCCL error) surfaces as J3D_ETIMEOUT / J3D_ENCCL instead of a
// hang.
double timeout_s() {
    double s = 600.0;
    if (const char* e = std::getenv("J3D_TIMEOUT_S")) s = std::atof(e);
    return s > 0 ? s : 600.0;
}

void wait_stream(jacobi3d* c, cudaStream_t st) {
    Nvtx nv("j3d.wait");
    if (c->n_gpus == 1) {
        CK(cudaStreamSynchronize(st));
        return;
    }
    const double limit = timeout_s();
    const auto t0 = std::chrono::steady_clock::now();
    int us = 20;
    for (;;) {
        const cudaError_t q = cudaStreamQuery(st);
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) CK(q);
        if (c->comm) {
            ncclResult_t ar = ncclSuccess;
            NK(ncclCommGetAsyncError(c->comm, &ar));
            NK(ar);
        }
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > limit)
            throw Error(J3D_ETIMEOUT, "cross-GPU wait did not complete within " + std::to_string((int)limit) +
                                          " s (a peer rank stopped, or the ranks called the collective API in "
                                          "different orders)");
        std::this_thread::sleep_for(std::chrono::microseconds(us));
        us = std::min(us * 2, 2000);
    }
}

// Wait for every stream of this context -- never cudaDeviceSynchronize: ranks
// that are threads of one process share the device, and a device-wide wait
// would also wait for a peer's queued work, which may itself wait for this
// rank's next call (a deadlock).
void sync_streams(jacobi3d* c) {
    if (c->main) wait_stream(c, c->main);
    for (auto s : c->lo) if (s && s != c->main) wait_stream(c, s);
    for (auto s : c->hi) if (s && s != c->main) wait_stream(c, s);
    if (c->xstream) wait_stream(c, c->xstream);
}


}  // namespace j3d
