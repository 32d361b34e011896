// setup.cu -- arena layout, face classification, device descriptor tables, TMA tensor maps and the work-item list of a context.
#include "context.h"

using namespace j3d;

namespace j3d {

Driver g_drv;

void build_layout(jacobi3d* c) {
    const Plan& P = c->plan;
    c->nx = P.ext[0];
    c->ny = P.ext[1];
    c->nz = P.ext[2];
    c->pitch = align_up(XOFF + c->nx + 1, PITCH_ALIGN);
    c->zs = c->pitch * (c->ny + 2);
    c->buf_elems = c->zs * (c->nz + 2);
    c->grid_bytes = align_up(c->buf_elems * 8, 256);
    c->xg_pitch = align_up(c->ny, 2);  // TMA: row strides are multiples of 16 bytes
    c->xg_bytes = align_up(c->xg_pitch * (c->nz + 2) * 8, 256);
    c->buf_bytes = c->grid_bytes + 2 * c->xg_bytes;
    for (int f = 0; f < 6; ++f) c->face_bytes[f] = align_up(face_cells(P.ext, f) * 8, 256);
    c->faces_per_block_bytes = 0;
    for (int f = 0; f < 6; ++f) c->faces_per_block_bytes += 4 * c->face_bytes[f];  // send/recv x 2 parities
    c->off_flags = 0;
    c->off_scratch = 2048;
    // J3D_PERSISTENT slab completion counters (at most one slab per plane of each
    // local block); inside the arena so peers read them over NVLink
    c->off_done = 4096;
    // one counter per (block, z chunk, tile row): chunks >= 1 plane, tile rows >= 8 rows
    const int64_t done_bytes =
        c->cfg.launch == J3D_PERSISTENT ? (int64_t)c->n_local * c->nz * ((c->ny + 7) / 8) * 4 : 0;
    c->off_bufs = align_up(c->off_done + done_bytes, 4096);
    c->off_faces = c->off_bufs + (int64_t)c->n_local * 2 * c->buf_bytes;
    c->arena_bytes = c->off_faces + (int64_t)c->n_local * c->faces_per_block_bytes;
}

void classify(jacobi3d* c) {
    const Plan& P = c->plan;
    c->gid = P.by_rank[c->rank];
    c->n_local = (int)c->gid.size();
    c->kind.assign(c->n_local, {});
    c->nbr_local.assign(c->n_local, {});
    c->has_peer.assign(c->n_local, 0);
    int xchg = c->cfg.exchange == J3D_XCHG_AUTO ? J3D_XCHG_P2P : c->cfg.exchange;
    std::vector<int> peers;
    for (int l = 0; l < c->n_local; ++l) {
        const BlockPlan& b = P.blocks[c->gid[l]];
        for (int f = 0; f < 6; ++f) {
            if (b.nbr[f] < 0) {
                c->kind[l][f] = DIRICHLET;
                c->nbr_local[l][f] = -1;
            } else {
                const BlockPlan& n = P.blocks[b.nbr[f]];
                c->nbr_local[l][f] = n.local;
                if (n.owner == c->rank) {
                    c->kind[l][f] = LOCAL;
                } else {
                    c->kind[l][f] = xchg == J3D_XCHG_NCCL ? PEER_NCCL : xchg == J3D_XCHG_HOST ? PEER_HOST : PEER_P2P;
                    if (xchg == J3D_XCHG_HOST) c->host_needed = true;
                    c->has_peer[l] = 1;
                    if (std::find(peers.begin(), peers.end(), n.owner) == peers.end()) peers.push_back(n.owner);
                    if (xchg == J3D_XCHG_P2P) c->p2p_needed = true;
                }
            }
        }
    }
    std::sort(peers.begin(), peers.end());
    c->peer_ranks = peers;
    c->order.clear();
    for (int l = 0; l < c->n_local; ++l)
        if (c->has_peer[l]) c->order.push_back(l);
    for (int l = 0; l < c->n_local; ++l)
        if (!c->has_peer[l]) c->order.push_back(l);
    if (const char* e = std::getenv("J3D_ORDER_SEED")) {  // test hook: perturbed launch order
        uint64_t st = std::strtoull(e, nullptr, 10) * 0x9E3779B97F4A7C15ULL + 1;
        for (int i = (int)c->order.size() - 1; i > 0; --i) {
            st ^= st << 13; st ^= st >> 7; st ^= st << 17;
            std::swap(c->order[i], c->order[(int)(st % (uint64_t)(i + 1))]);
        }
    }
}

// Source of the ghost values of face f of local block l for buffer parity par
// (what an unpack or a fused prologue reads).
FaceRef recv_src(const jacobi3d* c, int l, int f, int par) {
    if (c->kind[l][f] == LOCAL)  // same GPU: read the neighbour's send buffer in place
        return c->contiguous(c->face_buf(c->nbr_local[l][f], f ^ 1, par, false), f);
    return c->contiguous(c->face_buf(l, f, par, true), f);
}

// Destination of the pack of face f of local block l for parity par.
FaceRef pack_dst(const jacobi3d* c, int l, int f, int par) {
    if (c->kind[l][f] == PEER_P2P) {  // GPU-aware: straight into the peer's receive buffer (NVLink)
        const int r = c->plan.blocks[c->plan.blocks[c->gid[l]].nbr[f]].owner;
        return c->contiguous(c->face_buf(c->nbr_local[l][f], f ^ 1, par, true, r), f);
    }
    return c->contiguous(c->face_buf(l, f, par, false), f);
}

// TMA map over a contiguous receive buffer of face f (layout: x faces (y, z),
// y faces (x, z), z faces (x, y); owned coordinates).  Boxes: an x ghost
// vector (TY x 1), a y ghost row (W x 1), a ghost plane (W x (TY+2)) -- the
// shapes the stencil's stage expects (kernels.cu stencil_tma_kernel).
static void encode_recv_map(const jacobi3d* c, CUtensorMap* m, const double* p, int f) {
    const int tk = c->tile_kind;
    const cuuint64_t na = (cuuint64_t)c->face_na(f), nb = (cuuint64_t)c->face_nb(f);
    cuuint64_t dims[2] = {na, nb};
    cuuint64_t strides[1] = {na * 8};
    cuuint32_t box[2];
    if (f < 2) { box[0] = (cuuint32_t)tile_shape(tk).ty; box[1] = 1; }
    else if (f < 4) { box[0] = (cuuint32_t)stencil_box_w(tk); box[1] = 1; }
    else { box[0] = (cuuint32_t)stencil_box_w(tk); box[1] = (cuuint32_t)stencil_box_h(tk); }
    cuuint32_t es[2] = {1, 1};
    DK(g_drv.encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(p), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
}

void build_tables(jacobi3d* c) {
    const int nl = c->n_local;
    const int v = c->cfg.variant;
    // ---- stencil descriptors [2*l + p]; strategy C's receive-buffer maps [(2*l + p)*6 + f]
    std::vector<StencilDesc> descs(2 * nl);
    std::vector<CUtensorMap> pro_maps((size_t)2 * nl * 6);
    std::memset(pro_maps.data(), 0, pro_maps.size() * sizeof(CUtensorMap));
    c->faces_fused = false;
    for (int l = 0; l < nl; ++l)
        for (int p = 0; p < 2; ++p) {
            const int q = p ^ 1;
            StencilDesc& d = descs[2 * l + p];
            std::memset(&d, 0, sizeof d);
            d.in = c->buf(l, p);
            d.out = c->buf(l, q);
            d.nx = (int32_t)c->nx;
            d.ny = (int32_t)c->ny;
            d.nz = (int32_t)c->nz;
            d.pitch = c->pitch;
            d.zs = c->zs;
            if (v == J3D_FUSE_C || v == J3D_FUSE_DIRECT) {
                for (int f = 0; f < 6; ++f) {
                    const int k = c->kind[l][f];
                    if (k == DIRICHLET) continue;
                    // direct ghost stores: same GPU, or a peer's y/z ghost layer over NVLink.
                    // Peer x faces (one 8-byte cell per row, scattered NVLink stores cost
                    // ~10% of the update, profiles/r01_multi_gpu.md) are instead packed
                    // from the output after the update and pushed to the peer's receive
                    // buffer (capturing them in the epilogue cost the update 1.7%).
                    bool direct = v == J3D_FUSE_DIRECT && (k == LOCAL || (k == PEER_P2P && (f >= 2 || c->peer_x_direct)));
                    if (direct) {
                        const int r = k == LOCAL ? -1 : c->plan.blocks[c->plan.blocks[c->gid[l]].nbr[f]].owner;
                        if (k == PEER_P2P && !c->p2p_connected) continue;  // filled after ipc_connect
                        d.epi[f] = c->layer(c->buf(c->nbr_local[l][f], q, r), f ^ 1, true);
                        d.epi_mask |= 1u << f;
                    } else if (v == J3D_FUSE_DIRECT && f < 2 && c->peer_x_pack) {
                        continue;  // peer x face: packed from the output by the push kernel
                    } else if (v == J3D_FUSE_DIRECT) {
                        // NCCL / host-staged face, or peer x face, of the direct
                        // variant: the epilogue packs into the local send buffer;
                        // after the exchange a batched unpack kernel writes the
                        // received face into the ghost layer (keeps the stencil's
                        // prologue empty)
                        if (k == PEER_P2P && !c->p2p_connected) continue;
                        d.epi[f] = c->contiguous(c->face_buf(l, f, q, false), f);
                        d.epi_mask |= 1u << f;
                    } else {
                        if (k == PEER_P2P && !c->p2p_connected) continue;
                        d.epi[f] = pack_dst(c, l, f, q);
                        d.epi_mask |= 1u << f;
                        d.pro[f] = recv_src(c, l, f, p);
                        // the producer loads these ghosts with TMA from the receive buffer when
                        // its row stride is a multiple of 16 bytes (TMA); else the consumer
                        // warps patch them with generic loads (patch_stage)
                        const int64_t pitch_elems = c->face_na(f);
                        const bool room = !(f == 2 || f == 3) || c->tile_ys;
                        if (room && pitch_elems % 2 == 0 && ((uintptr_t)d.pro[f].p & 15) == 0) {
                            d.pro_tma |= 1u << f;
                            encode_recv_map(c, &pro_maps[(size_t)(2 * l + p) * 6 + f], d.pro[f].p, f);
                        } else {
                            d.pro_mask |= 1u << f;
                        }
                    }
                }
                for (int f = 0; f < 2; ++f)  // x-face destinations are contiguous in y (kernels.cu HOISTX1)
                    if ((d.epi_mask & (1u << f)) && d.epi[f].sa != 1)
                        throw Error(J3D_EUNSUPPORTED, "x-face destination with a row stride != 1");
                if (d.epi_mask | d.pro_mask | d.pro_tma) c->faces_fused = true;
            }
        }
    CK(cudaMemcpy(c->d_descs, descs.data(), descs.size() * sizeof(StencilDesc), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_tmaps_pro, pro_maps.data(), pro_maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));

    // ---- pack / unpack copy descriptors [(q*nl + l)*6 + f]
    std::vector<CopyDesc> pack(2 * nl * 6), unpack(2 * nl * 6);
    for (int q = 0; q < 2; ++q)
        for (int l = 0; l < nl; ++l)
            for (int f = 0; f < 6; ++f) {
                CopyDesc& pk = pack[(q * nl + l) * 6 + f];
                CopyDesc& up = unpack[(q * nl + l) * 6 + f];
                std::memset(&pk, 0, sizeof pk);
                std::memset(&up, 0, sizeof up);
                const int k = c->kind[l][f];
                if (k == DIRICHLET) continue;
                if (k == PEER_P2P && !c->p2p_connected) continue;
                pk.src = c->layer(c->buf(l, q), f, false);
                pk.dst = pack_dst(c, l, f, q);
                pk.na = (int32_t)c->face_na(f);
                pk.nb = (int32_t)c->face_nb(f);
                up.src = recv_src(c, l, f, q);
                up.dst = c->layer(c->buf(l, q), f, true);
                up.na = pk.na;
                up.nb = pk.nb;
            }
    CK(cudaMemcpy(c->d_pack, pack.data(), pack.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_unpack, unpack.data(), unpack.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
    // direct variant: faces that travel through the buffers (NCCL, host staging,
    // peer x faces) -- the push of peer x faces (local send buffer -> the
    // peer's receive buffer over NVLink, coalesced) and the post-exchange unpack
    c->direct_nccl_unpack = false;
    c->direct_push = false;
    std::vector<CopyDesc> push(2 * nl * 6);
    for (int q = 0; q < 2; ++q)
        for (int l = 0; l < nl; ++l)
            for (int f = 0; f < 6; ++f) {
                const int i = (q * nl + l) * 6 + f;
                const int k = c->kind[l][f];
                CopyDesc& up = unpack[i];
                std::memset(&push[i], 0, sizeof(CopyDesc));
                const bool px = k == PEER_P2P && f < 2 && c->p2p_connected && !c->peer_x_direct;
                if (!via_buffers(k) && !px) std::memset(&up, 0, sizeof up);
                else if (v == J3D_FUSE_DIRECT) c->direct_nccl_unpack = true;
                // x faces that leave through buffers: pushed from the output (peer_x_pack)
                // or from the send buffer the epilogue filled (P2P only)
                if (v == J3D_FUSE_DIRECT && f < 2 && (px || (via_buffers(k) && c->peer_x_pack))) {
                    push[i].src = c->peer_x_pack ? c->layer(c->buf(l, q), f, false)
                                                 : c->contiguous(c->face_buf(l, f, q, false), f);
                    push[i].dst = pack_dst(c, l, f, q);
                    push[i].na = (int32_t)c->face_na(f);
                    push[i].nb = (int32_t)c->face_nb(f);
                    c->direct_push = true;
                }
            }
    CK(cudaMemcpy(c->d_unpack_nccl, unpack.data(), unpack.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_push, push.data(), push.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
    // peer-only / local-only tables for the overlap mode
    {
        std::vector<CopyDesc> pk_peer(pack), up_peer(2 * nl * 6), pk_loc(pack), up_loc(2 * nl * 6);
        std::vector<CopyDesc> up_all(2 * nl * 6);
        for (int q = 0; q < 2; ++q)
            for (int l = 0; l < nl; ++l)
                for (int f = 0; f < 6; ++f) {
                    const int i = (q * nl + l) * 6 + f;
                    const int k = c->kind[l][f];
                    CopyDesc up;
                    std::memset(&up, 0, sizeof up);
                    if (k != DIRICHLET && !(k == PEER_P2P && !c->p2p_connected)) {
                        up.src = recv_src(c, l, f, q);
                        up.dst = c->layer(c->buf(l, q), f, true);
                        up.na = (int32_t)c->face_na(f);
                        up.nb = (int32_t)c->face_nb(f);
                    }
                    const bool peer = is_peer_kind(k);
                    if (!peer) std::memset(&pk_peer[i], 0, sizeof(CopyDesc));
                    if (peer || k == DIRICHLET) std::memset(&pk_loc[i], 0, sizeof(CopyDesc));
                    if (peer) up_peer[i] = up;
                    else if (k == LOCAL) up_loc[i] = up;
                    if (!peer && k != LOCAL) std::memset(&up_peer[i], 0, sizeof(CopyDesc));
                }
        for (auto& d : up_peer) if (d.na == 0) std::memset(&d, 0, sizeof d);
        CK(cudaMemcpy(c->d_pack_peer, pk_peer.data(), pk_peer.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->d_unpack_peer, up_peer.data(), up_peer.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->d_pack_local, pk_loc.data(), pk_loc.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->d_unpack_local, up_loc.data(), up_loc.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
    }
    build_persist_deps(c);
}

// J3D_PERSISTENT dependency tables (IterCtl, device.cuh).  A slab is one row
// of tiles (all tx) of one block over one z chunk: (l, zc, ty).  An item of
// slab (l, zc, ty) reads, of the previous iteration's output, its own cells,
// the boundary planes of chunks zc-1 / zc+1 and the boundary rows of tile
// rows ty-1 / ty+1 (same block), the x ghost columns the x neighbours' slab
// (zc, ty) wrote, for an edge tile row the y ghost row the y neighbour's edge
// slab wrote, for an edge chunk the z ghost plane the z neighbour's edge slab
// wrote -- and by symmetry of the 7-point neighbourhood exactly those slabs
// read, in the previous iteration, the cells its own stores overwrite.
// (Diagonal neighbours' corner cells are fetched by the TMA box but never
// used.)  slab_dep_refs lists them symbolically (rank, local block, zc,
// ty) -- jacobi3d_debug_slab_deps exports that list without a GPU, and
// tests/test_persistent_rule.py checks it against the brute-force hazard set.
std::vector<std::vector<SlabRef>> slab_dep_refs(const jacobi3d* c, int nzc, int nty) {
    const int nl = c->n_local;
    std::vector<std::vector<SlabRef>> out((size_t)nl * nzc * nty);
    // slab (zc, ty) of the neighbour across face f of block l; none for a
    // Dirichlet face or a peer face whose halo does not travel by P2P stores
    auto across = [&](int l, int f, int zc, int ty, std::vector<SlabRef>& d) {
        const int k = c->kind[l][f];
        if (k != LOCAL && k != PEER_P2P) return;
        const int r = k == LOCAL ? c->rank : c->plan.blocks[c->plan.blocks[c->gid[l]].nbr[f]].owner;
        d.push_back(SlabRef{r, c->nbr_local[l][f], zc, ty});
    };
    for (int l = 0; l < nl; ++l)
        for (int zc = 0; zc < nzc; ++zc)
            for (int ty = 0; ty < nty; ++ty) {
                std::vector<SlabRef>& d = out[((size_t)l * nzc + zc) * nty + ty];
                d.push_back(SlabRef{c->rank, l, zc, ty});
                if (zc > 0) d.push_back(SlabRef{c->rank, l, zc - 1, ty});
                if (zc + 1 < nzc) d.push_back(SlabRef{c->rank, l, zc + 1, ty});
                if (ty > 0) d.push_back(SlabRef{c->rank, l, zc, ty - 1});
                if (ty + 1 < nty) d.push_back(SlabRef{c->rank, l, zc, ty + 1});
                for (int f = 0; f < 2; ++f) across(l, f, zc, ty, d);
                if (ty == 0) across(l, 2, zc, nty - 1, d);
                if (ty == nty - 1) across(l, 3, zc, 0, d);
                if (zc == 0) across(l, 4, nzc - 1, ty, d);
                if (zc == nzc - 1) across(l, 5, 0, ty, d);
                if (d.size() > (size_t)MAX_DEPS) throw Error(J3D_EUNSUPPORTED, "slab dependency table overflow");
            }
    return out;
}

// The tables the kernel reads: slab_dep_refs resolved to counter addresses
// (a peer's through its IPC-mapped arena, tagged for a system-scope acquire;
// known only after jacobi3d_ipc_connect).  `remote` collects the peer
// counters for the end-of-call wait.  The second table drops every remote
// entry (timing with the exchange elided, jacobi3d_set_skip_exchange).
void build_persist_deps(jacobi3d* c) {
    if (c->cfg.launch != J3D_PERSISTENT) return;
    const int nzc = c->persist_nzc, nty = c->persist_nty;
    auto sid = [&](int l, int zc, int ty) { return ((int64_t)l * nzc + zc) * nty + ty; };
    const std::vector<std::vector<SlabRef>> refs = slab_dep_refs(c, nzc, nty);
    std::vector<const unsigned int*> deps((size_t)c->n_slabs * MAX_DEPS, nullptr), local(deps);
    std::vector<const unsigned int*> remote;
    for (int64_t s = 0; s < (int64_t)refs.size(); ++s) {
        int n = 0, nloc = 0;
        for (const SlabRef& e : refs[s]) {
            if (e.rank == c->rank) {
                const unsigned int* p = c->d_done + sid(e.local, e.zc, e.ty);
                deps[(size_t)s * MAX_DEPS + n++] = p;
                local[(size_t)s * MAX_DEPS + nloc++] = p;
            } else if (c->p2p_connected) {
                const uintptr_t p = (uintptr_t)((const unsigned int*)(c->peer_base[e.rank] + c->off_done) +
                                                sid(e.local, e.zc, e.ty));
                deps[(size_t)s * MAX_DEPS + n++] = (const unsigned int*)(p | 1);  // tag: system scope (device.cuh)
                if (std::find(remote.begin(), remote.end(), (const unsigned int*)p) == remote.end())
                    remote.push_back((const unsigned int*)p);
            }
        }
    }
    CK(cudaMemcpy(c->d_slab_deps, deps.data(), deps.size() * sizeof(void*), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_slab_deps_local, local.data(), local.size() * sizeof(void*), cudaMemcpyHostToDevice));
    if (c->d_remote_done) cudaFree(c->d_remote_done);
    c->d_remote_done = nullptr;
    c->n_remote_done = (int)remote.size();
    if (!remote.empty()) {
        CK(cudaMalloc(&c->d_remote_done, remote.size() * sizeof(void*)));
        CK(cudaMemcpy(c->d_remote_done, remote.data(), remote.size() * sizeof(void*), cudaMemcpyHostToDevice));
    }
}

void build_static_tables(jacobi3d* c) {
    const int nl = c->n_local;
    // ---- tensor maps [2*l + p] over each input buffer
    g_drv.load();
    // 192x22 tiles (11 consumer warps, 5-stage ring, 1 CTA/SM) when they divide
    // the block width, else 128x30 (15 consumer warps) for wide blocks, 96x16
    // one-cell-per-lane tiles for 96-wide blocks (BASELINE configs[4]) and
    // 64x16 (2 CTAs/SM, 6 stages) for other narrow ones.  Sweeps: profiles/.
    // 96-wide blocks (BASELINE configs[4]): 96x16 one-cell-per-lane tiles, 4 warps x 4 rows,
    // 7 stages (round 2: 333 -> 348 GLUPS persistent on 96^3 blocks, profiles/r02_tuning_log.md)
    // (strategy C keeps 96x16 x 8 warps: kind 23's 7 stages leave no room for the y
    // side rows its TMA-fed prologue needs, 283 vs 181 GLUPS batched)
    c->tile_kind = (c->nx % 192 == 0) ? 0 : c->nx >= 128 ? 1 : (c->nx == 96) ? (c->cfg.variant == J3D_FUSE_C ? 12 : 23) : 4;
    if (c->tile_kind == 0) {
        // 192x24 (12 consumer warps) when 22-row tiles would leave a mostly empty last
        // tile row: measured on 192x96x96 blocks 1144 -> 1248 GLUPS (4 GPUs), equal at 1536
        auto waste = [&](int ty) { return (double)(((c->ny + ty - 1) / ty) * ty - c->ny) / (double)c->ny; };
        if (waste(24) + 0.005 < waste(22)) c->tile_kind = 21;
        // the largest blocks (1536^3, BASELINE configs[1]): 192x24 with 6 warps x 4 rows --
        // fewer per-plane instructions per update, which matters under the 1 kW cap
        // (374 -> 384 GLUPS, profiles/r02_tuning_log.md)
        if (c->ny >= 1536 && c->ny % 24 == 0) c->tile_kind = 26;
    }
    if (c->tile_kind <= 1 || c->tile_kind == 21 || c->tile_kind == 26) {  // small grids: the wide tiles cannot keep every SM busy -> 64x16, 2 CTAs/SM
        const TileShape t = tile_shape(c->tile_kind);
        const int64_t tiles = ((c->nx + t.tx - 1) / t.tx) * ((c->ny + t.ty - 1) / t.ty) * nl;
        const int64_t max_items = tiles * std::max<int64_t>(1, c->nz / 24);
        if (max_items < 4LL * c->sms) c->tile_kind = 4;
    }
    if (const char* e = std::getenv("J3D_TILE")) {  // tuning override (bench sweeps)
        const int k = std::atoi(e);
        if (k >= 0 && k < num_tile_kinds()) c->tile_kind = k;
    }
    const TileShape ts = tile_shape(c->tile_kind);
    c->tile_ys = c->cfg.variant == J3D_FUSE_C && tile_yside(c->tile_kind);
    std::vector<CUtensorMap> maps(2 * nl);
    CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    if (const char* e = std::getenv("J3D_L2PROMO")) {  // tuning override
        const int v = std::atoi(e);
        promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
              : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }
    // over the owned columns only (x in [0, nx): the halo columns beyond a block
    // edge are zero-filled out of bounds, never fetched) and every row / plane
    // including the y / z ghost layers
    for (int l = 0; l < nl; ++l)
        for (int p = 0; p < 2; ++p) {
            cuuint64_t dims[3] = {(cuuint64_t)c->nx, (cuuint64_t)(c->ny + 2), (cuuint64_t)(c->nz + 2)};
            cuuint64_t strides[2] = {(cuuint64_t)(c->pitch * 8), (cuuint64_t)(c->zs * 8)};
            cuuint32_t box[3] = {(cuuint32_t)stencil_box_w(c->tile_kind), (cuuint32_t)stencil_box_h(c->tile_kind), 1};
            cuuint32_t es[3] = {1, 1, 1};
            DK(g_drv.encode(&maps[2 * l + p], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->buf(l, p) + XOFF, dims, strides,
                            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
        }
    CK(cudaMemcpy(c->d_tmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
    // x ghost vectors: (y, z, side) over the two x ghost arrays of a buffer, box TY x 1 x 1
    std::vector<CUtensorMap> xmaps(2 * nl);
    for (int l = 0; l < nl; ++l)
        for (int p = 0; p < 2; ++p) {
            cuuint64_t dims[3] = {(cuuint64_t)c->ny, (cuuint64_t)(c->nz + 2), 2};
            cuuint64_t strides[2] = {(cuuint64_t)(c->xg_pitch * 8), (cuuint64_t)c->xg_bytes};
            cuuint32_t box[3] = {(cuuint32_t)ts.ty, 1, 1};
            cuuint32_t es[3] = {1, 1, 1};
            DK(g_drv.encode(&xmaps[2 * l + p], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->xghost(c->buf(l, p), 0), dims,
                            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
        }
    CK(cudaMemcpy(c->d_tmaps_x, xmaps.data(), xmaps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
    if (const char* e = std::getenv("J3D_TMA_HINT")) c->tma_mode = std::atoi(e) % 3;
    if (const char* e = std::getenv("J3D_PREFETCH")) c->prefetch = std::atoi(e) != 0;
    if (const char* e = std::getenv("J3D_DEPFENCE")) c->depfence = std::atoi(e) != 0;

    // ---- work items: per block, z-chunk outer, then ty, tx (x fastest), peer-face blocks first
    int occ = 1;
    CK(stencil_occupancy(c->tile_kind, c->tile_ys, &occ));
    occ = std::max(1, occ);
    c->grid_cap = c->sms * occ;
    const int64_t ntx = (c->nx + ts.tx - 1) / ts.tx, nty = (c->ny + ts.ty - 1) / ts.ty;
    const int64_t tiles = ntx * nty * nl;
    // z chunks of ~96 planes: items are handed out dynamically in list order
    // (z chunk outer, then tiles), so x/y-neighbouring tiles -- whose halos
    // overlap -- run concurrently and share halo rows through L2, while each
    // chunk re-reads only 2 extra planes (2% at 96).  Measured sweep: 96
    // beats 32/64/128/full depth (profiles/).
    int64_t best_zc = std::max<int64_t>(1, (c->nz + 95) / 96);
    // small problems: shorter chunks until there are >= 8 items per CTA slot
    // (at least 16 planes per chunk): the last round of items is then short
    // (measured: 96^3 blocks, ODF 64: 198 -> 225 GLUPS in round 1 with >= 6 / 24)
    if (c->cfg.launch == J3D_PERSISTENT) {
        // persistent launch: iterations overlap, so there is no per-iteration tail to
        // shorten -- two items per CTA slot keep the SMs busy, and longer chunks re-read
        // fewer boundary planes (96^3 blocks: 24 -> 48 planes, 311 -> 330 GLUPS; 192^3
        // single block: 16 planes, 284 -> 342 GLUPS)
        // Across GPUs, chunks down to 12 planes: slabs next to a peer run last in each
        // iteration, and shorter chunks let the rest of the GPU run ahead while they
        // wait (4 GPUs: one 192^3 block 832 -> 929 GLUPS).  Four items per slot
        // helped too before the wavefront slab order below; with it, two (4 GPUs:
        // 192x96x96 blocks, 48- instead of 32-plane chunks, 1337 -> 1375-1401 GLUPS;
        // profiles/r02_tuning_log.md)
        const int64_t per_slot = 2, min_planes = c->n_gpus > 1 ? 12 : 16;
        while (tiles * best_zc < per_slot * (int64_t)c->grid_cap && c->nz / (best_zc + 1) >= min_planes) ++best_zc;
    } else {
        // (round 2: >= 8 items per CTA slot, >= 16 planes: 96^3 blocks batched 297 -> 306 GLUPS)
        while (tiles * best_zc < 8 * (int64_t)c->grid_cap && c->nz / (best_zc + 1) >= 16) ++best_zc;
    }
    if (const char* e = std::getenv("J3D_ZCHUNK")) {  // tuning override: planes per z chunk
        const int64_t L = std::atoll(e);
        if (L > 0) best_zc = std::max<int64_t>(1, (c->nz + L - 1) / L);
    }
    int tile_order = 0;  // tuning override: tile order inside a z chunk
    if (const char* e = std::getenv("J3D_TILE_ORDER")) tile_order = std::atoi(e);
    std::vector<WorkItem> items;
    c->item_begin.assign(nl, 0);
    c->item_count.assign(nl, 0);
    auto is_peer = [&](int l, int f) { return is_peer_kind(c->kind[l][f]); };
    auto exterior = [&](const WorkItem& w) {  // does the item compute a cell adjacent to a peer face?
        const int l = w.blk;
        return (is_peer(l, 0) && w.tx == 0) || (is_peer(l, 1) && w.tx == ntx - 1) ||
               (is_peer(l, 2) && w.ty == 0) || (is_peer(l, 3) && w.ty == nty - 1) ||
               (is_peer(l, 4) && w.z0 == 0) || (is_peer(l, 5) && w.z1 == c->nz);
    };
    for (int l : c->order) {
        c->item_begin[l] = (int)items.size();
        for (int64_t zc = 0; zc < best_zc; ++zc) {
            const int z0 = (int)(c->nz * zc / best_zc), z1 = (int)(c->nz * (zc + 1) / best_zc);
            if (z1 <= z0) continue;
            if (tile_order == 1) {  // y fastest
                for (int64_t tx = 0; tx < ntx; ++tx)
                    for (int64_t ty = 0; ty < nty; ++ty)
                        items.push_back(WorkItem{l, (int16_t)tx, (int16_t)ty, z0, z1});
            } else if (tile_order >= 2) {  // bands of `tile_order` tile rows, column-major inside a band
                for (int64_t b0 = 0; b0 < nty; b0 += tile_order)
                    for (int64_t tx = 0; tx < ntx; ++tx)
                        for (int64_t ty = b0; ty < std::min<int64_t>(nty, b0 + tile_order); ++ty)
                            items.push_back(WorkItem{l, (int16_t)tx, (int16_t)ty, z0, z1});
            } else {  // x fastest
                for (int64_t ty = 0; ty < nty; ++ty)
                    for (int64_t tx = 0; tx < ntx; ++tx)
                        items.push_back(WorkItem{l, (int16_t)tx, (int16_t)ty, z0, z1});
            }
        }
        c->item_count[l] = (int)items.size() - c->item_begin[l];
    }
    // Batched launch: the last round of the dynamic scheduler (the final grid_cap
    // items) in half-height items, so the launch's tail -- SMs idle while the last
    // items finish -- is half as long (J3D_TAILSPLIT=0: off)
    int tail_split = 1;
    if (const char* e = std::getenv("J3D_TAILSPLIT")) tail_split = std::atoi(e);
    if (tail_split && c->cfg.launch == J3D_BATCHED && !c->overlap) {
        // mode 1: the last grid_cap items in halves; mode 2: also the last grid_cap in
        // quarters and the grid_cap before them in halves
        const size_t n0 = items.size(), k = std::min(n0, (size_t)c->grid_cap);
        std::vector<WorkItem> out;
        out.reserve(n0 + 4 * k);
        for (size_t i = 0; i < n0; ++i) {
            const WorkItem& w = items[i];
            int parts = 1;
            if (i >= n0 - k) parts = tail_split >= 2 ? 4 : 2;
            else if (tail_split >= 2 && i + 2 * k >= n0) parts = 2;
            while (parts > 1 && (w.z1 - w.z0) / parts < 4) parts /= 2;
            for (int q = 0; q < parts; ++q)
                out.push_back(WorkItem{w.blk, w.tx, w.ty, w.z0 + (w.z1 - w.z0) * q / parts,
                                       w.z0 + (w.z1 - w.z0) * (q + 1) / parts});
        }
        items.swap(out);
        for (int l = 0; l < nl; ++l) c->item_count[l] = 0;
        for (size_t i = 0; i < items.size(); ++i) {  // blocks stay contiguous in the list
            const int l = items[i].blk;
            if (c->item_count[l]++ == 0) c->item_begin[l] = (int)i;
        }
    }
    c->n_ext = 0;
    if (c->overlap) {  // BATCHED only: exterior items of every block first (stable order otherwise)
        std::stable_partition(items.begin(), items.end(), exterior);
        c->n_ext = (int)std::count_if(items.begin(), items.end(), exterior);
    } else if (c->cfg.launch == J3D_PERSISTENT && c->n_gpus > 1) {
        // persistent: slabs that wait on a peer LAST -- the peer's matching slabs
        // were the last of its previous iteration too, so a GPU may run up to an
        // iteration ahead of a slower neighbour instead of meeting it at every
        // iteration start.  Whole slabs (tile rows) move: a slab completes only
        // with all its tiles, so splitting one would delay every dependant of it.
        auto zc_of = [&](const WorkItem& w) {
            int zc = 0;
            while ((int)(c->nz * (zc + 1) / best_zc) <= w.z0) ++zc;
            return zc;
        };
        //
        // Within the interior, slabs run in decreasing dependency distance from the
        // exterior (hops over this GPU's slab dependencies, slab_dep_refs): the first
        // slabs of iteration k+1 then depend only on slabs that ran early in
        // iteration k.  Plain list order put, e.g., chunk 1 first when chunk 0 is
        // exterior, and it waited for the end of the previous iteration at every
        // iteration start (one 192^3 block per GPU: 28.5 instead of 21 us per
        // iteration with the exchange elided).  Measured (profiles/r02_tuning_log.md):
        // 96^3 and 192x96x96 blocks on 4 GPUs +3-4 %, one 192^3 block on 2 GPUs
        // +9.5 %, on 4 GPUs -5 % (peer waits appear there).
        const size_t ns = (size_t)nl * best_zc * nty;
        std::vector<int> depth(ns, INT32_MAX);
        auto row_slab = [&](const WorkItem& w) { return ((size_t)w.blk * best_zc + zc_of(w)) * nty + w.ty; };
        std::vector<size_t> frontier;
        for (const WorkItem& w : items)
            if (exterior(w) && depth[row_slab(w)] != 0) {
                depth[row_slab(w)] = 0;
                frontier.push_back(row_slab(w));
            }
        const std::vector<std::vector<SlabRef>> refs = slab_dep_refs(c, (int)best_zc, (int)nty);
        for (int dd = 1; !frontier.empty(); ++dd) {  // breadth-first over local dependencies
            std::vector<size_t> next;
            for (size_t s : frontier)
                for (const SlabRef& e : refs[s]) {
                    if (e.rank != c->rank) continue;
                    const size_t t = ((size_t)e.local * best_zc + e.zc) * nty + e.ty;
                    if (depth[t] == INT32_MAX) {
                        depth[t] = dd;
                        next.push_back(t);
                    }
                }
            frontier.swap(next);
        }
        int wave = 1;  // tuning hook J3D_WAVE: 0 exterior last only, 1 deepest first, 2 exterior first
        if (const char* e = std::getenv("J3D_WAVE")) wave = std::atoi(e);
        if (wave == 0) {
            std::stable_partition(items.begin(), items.end(), [&](const WorkItem& w) { return depth[row_slab(w)] != 0; });
        } else {
            std::stable_sort(items.begin(), items.end(), [&](const WorkItem& a, const WorkItem& b) {
                const int da = depth[row_slab(a)], db = depth[row_slab(b)];
                return wave == 2 ? da < db : da > db;
            });
        }
    }
    c->n_items = (int)items.size();
    c->item_cells.assign(items.size() + 1, 0);
    for (size_t i = 0; i < items.size(); ++i) {
        const WorkItem& w = items[i];
        const int64_t ex = std::min<int64_t>(ts.tx, c->nx - (int64_t)w.tx * ts.tx);
        const int64_t ey = std::min<int64_t>(ts.ty, c->ny - (int64_t)w.ty * ts.ty);
        c->item_cells[i + 1] = c->item_cells[i] + ex * ey * (w.z1 - w.z0);
    }
    if (c->cfg.launch == J3D_PERSISTENT) {
        // slab = (local block, z chunk, tile row); the dependency tables are built by
        // build_persist_deps
        const int nzc = (int)best_zc;
        c->persist_nzc = nzc;
        c->persist_nty = (int)nty;
        c->n_slabs = nl * nzc * (int)nty;
        if ((int64_t)c->n_slabs * 4 > c->off_bufs - c->off_done)
            throw Error(J3D_EUNSUPPORTED, "persistent slab counters exceed their arena region");
        c->slab_target = (uint32_t)(ts.ncw * ntx);
        std::vector<int32_t> slab(items.size());
        for (size_t i = 0; i < items.size(); ++i) {
            const WorkItem& w = items[i];
            int zc = 0;
            while ((int)(c->nz * (zc + 1) / best_zc) <= w.z0) ++zc;
            // slab flag SLAB_PEER: some item of the slab touches a peer face (its
            // stores reach the peer; the peer reads its counter over NVLink)
            const bool peer = is_peer(w.blk, 0) || is_peer(w.blk, 1) || (is_peer(w.blk, 2) && w.ty == 0) ||
                              (is_peer(w.blk, 3) && w.ty == nty - 1) || (is_peer(w.blk, 4) && zc == 0) ||
                              (is_peer(w.blk, 5) && zc == nzc - 1);
            slab[i] = (int32_t)(((int64_t)w.blk * nzc + zc) * nty + w.ty) | (peer ? SLAB_PEER : 0);
        }
        CK(cudaMalloc(&c->d_item_slab, std::max<size_t>(1, slab.size()) * sizeof(int32_t)));
        CK(cudaMemcpy(c->d_item_slab, slab.data(), slab.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        CK(cudaMalloc(&c->d_slab_deps, (size_t)c->n_slabs * MAX_DEPS * sizeof(void*)));
        CK(cudaMalloc(&c->d_slab_deps_local, (size_t)c->n_slabs * MAX_DEPS * sizeof(void*)));
        c->d_done = (unsigned int*)(c->arena + c->off_done);  // zeroed with the arena at create
        c->persist_base = 0;
    }
    CK(cudaMalloc(&c->d_items, std::max<size_t>(1, items.size()) * sizeof(WorkItem)));
    CK(cudaMemcpy(c->d_items, items.data(), items.size() * sizeof(WorkItem), cudaMemcpyHostToDevice));

    // ---- block geometry
    std::vector<BlockGeom> geo(nl);
    for (int l = 0; l < nl; ++l) {
        const BlockPlan& b = c->plan.blocks[c->gid[l]];
        geo[l].buf[0] = c->buf(l, 0);
        geo[l].buf[1] = c->buf(l, 1);
        geo[l].ox = b.origin[0];
        geo[l].oy = b.origin[1];
        geo[l].oz = b.origin[2];
        geo[l].nx = (int32_t)c->nx;
        geo[l].ny = (int32_t)c->ny;
        geo[l].nz = (int32_t)c->nz;
        geo[l].pitch = c->pitch;
        geo[l].zs = c->zs;
        geo[l].xg_off = c->grid_bytes / 8;
        geo[l].xg_side = c->xg_bytes / 8;
        geo[l].xg_pitch = c->xg_pitch;
    }
    CK(cudaMemcpy(c->d_geom, geo.data(), geo.size() * sizeof(BlockGeom), cudaMemcpyHostToDevice));
}


}  // namespace j3d
