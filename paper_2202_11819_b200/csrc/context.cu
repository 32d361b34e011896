// context.cu -- the C-ABI (include/jacobi3d.h) and the per-iteration
// orchestration of the Jacobi3D hot path.
//
// One context = one rank = one GPU.  It owns one device arena holding, for
// each of its ODF blocks, the two ghosted fp64 buffers
// and, per face and buffer parity, a send and a receive buffer; plus epoch
// flags for the NVLink P2P backend.  Every rank lays its arena out
// identically, so a peer's buffer address is (peer arena base + the same
// offset) once the arenas are mapped with CUDA IPC.
//
// Per iteration i (input parity p = i&1, output parity q = p^1), SURVEY §3.5:
//   UNFUSED/A/B : update(p)  -> pack(q) -> [exchange q] -> unpack(q)
//   FUSE_C      : update(p) with prologue reading recv[p], epilogue writing
//                 send[q] (or the peer's recv[q] over NVLink) -> [exchange q]
//   FUSE_DIRECT : update(p) with the epilogue storing into the neighbours'
//                 ghost layers of buffer q (local or NVLink) -> [exchange q]
// with no host synchronisation: dependencies are stream order, CUDA events
// (per-block mode) and, across GPUs, NCCL or epoch flags written/waited with
// stream memory operations (capturable into the two CUDA graphs, one per
// buffer parity, that PAPER.md L529-530 alternates).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/jacobi3d.h"
#include "device.cuh"
#include "kernels.h"
#include "plan.h"

namespace j3d {

static thread_local std::string g_err;

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(call)                                                                                          \
    do {                                                                                                  \
        cudaError_t e_ = (call);                                                                          \
        if (e_ != cudaSuccess)                                                                            \
            throw Error(e_ == cudaErrorMemoryAllocation ? J3D_ENOMEM : J3D_ECUDA,                         \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                              \
    } while (0)
#define NK(call)                                                                                          \
    do {                                                                                                  \
        ncclResult_t r_ = (call);                                                                         \
        if (r_ != ncclSuccess) throw Error(J3D_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)
#define DK(call)                                                                                          \
    do {                                                                                                  \
        CUresult r_ = (call);                                                                             \
        if (r_ != CUDA_SUCCESS) throw Error(J3D_ECUDA, std::string(#call) + ": CUresult " + std::to_string((int)r_)); \
    } while (0)

// ---------------------------------------------------------------- driver entry points
typedef CUresult (*fn_encode_tiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*fn_write64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*fn_wait64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

struct Driver {
    fn_encode_tiled encode = nullptr;
    fn_write64 write64 = nullptr;
    fn_wait64 wait64 = nullptr;
    void load() {
        if (encode) return;
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw Error(J3D_EUNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
        encode = (fn_encode_tiled)p;
        CK(cudaGetDriverEntryPointByVersion("cuStreamWriteValue64", &p, 12000, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw Error(J3D_EUNSUPPORTED, "cuStreamWriteValue64 unavailable");
        write64 = (fn_write64)p;
        CK(cudaGetDriverEntryPointByVersion("cuStreamWaitValue64", &p, 12000, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw Error(J3D_EUNSUPPORTED, "cuStreamWaitValue64 unavailable");
        wait64 = (fn_wait64)p;
    }
};
static Driver g_drv;

enum FaceKind { DIRICHLET = 0, LOCAL = 1, PEER_NCCL = 2, PEER_P2P = 3, PEER_HOST = 4 };
// faces whose data travels through the send/receive buffers in a separate exchange step
static inline bool via_buffers(int k) { return k == PEER_NCCL || k == PEER_HOST; }
static inline bool is_peer_kind(int k) { return k == PEER_NCCL || k == PEER_P2P || k == PEER_HOST; }

static inline int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

struct IpcRecord {
    uint64_t magic;
    int32_t rank, device;
    uint64_t arena_bytes;
    cudaIpcMemHandle_t handle;
};
static const uint64_t kIpcMagic = 0x4a33445f49504331ULL;  // "J3D_IPC1"

}  // namespace j3d

using namespace j3d;

struct jacobi3d {
    jacobi3d_config cfg{};
    Plan plan;
    int rank = 0, n_gpus = 1, device = 0, sms = 148;
    int64_t nx = 0, ny = 0, nz = 0, pitch = 0, zs = 0, buf_elems = 0;
    int n_local = 0;
    std::vector<int64_t> gid;                 // local index -> global block id
    std::vector<std::array<int, 6>> kind;     // FaceKind per local block face
    std::vector<std::array<int, 6>> nbr_local;// neighbour's local index (LOCAL) or its owner-local index (PEER)
    std::vector<uint8_t> has_peer;

    // arena layout (identical on every rank)
    char* arena = nullptr;
    int64_t arena_bytes = 0, off_flags = 0, off_scratch = 0, off_bufs = 0, buf_bytes = 0, off_faces = 0;
    std::array<int64_t, 6> face_bytes{};
    int64_t faces_per_block_bytes = 0;
    std::vector<char*> peer_base;  // mapped arenas (index = rank), nullptr for self
    bool p2p_needed = false, p2p_connected = false;
    // host staging (J3D_XCHG_HOST): one POSIX shared-memory segment per rank,
    // [flags: 8 slots x n_gpus uint64 | staging: per local block, face, parity],
    // registered with CUDA so stream memory ops and DMA copies reach it
    bool host_needed = false, host_connected = false;
    uint64_t job_key = 0;
    size_t shm_bytes = 0;
    std::vector<char*> shm_base;      // mapped segments (index = rank; own included)
    std::vector<char*> shm_dev;       // device-visible address of each mapped segment

    // device tables
    StencilDesc* d_descs = nullptr;
    CUtensorMap* d_tmaps = nullptr;
    CUtensorMap* d_tmaps_split = nullptr;
    int tma_mode = 0;
    WorkItem* d_items = nullptr;
    CopyDesc* d_pack = nullptr;
    CopyDesc* d_unpack = nullptr;
    CopyDesc* d_unpack_nccl = nullptr;         // unpack of NCCL faces only (direct variant)
    CopyDesc* d_pack_peer = nullptr;           // peer faces only (overlap mode)
    CopyDesc* d_unpack_peer = nullptr;
    CopyDesc* d_pack_local = nullptr;          // same-GPU faces only (overlap mode)
    CopyDesc* d_unpack_local = nullptr;
    bool overlap = false;                      // exterior-first split with the exchange on `comm`
    int n_ext = 0;                             // items [0, n_ext) touch a peer face
    cudaStream_t xstream = nullptr;            // exchange stream (overlap mode)
    std::array<cudaEvent_t, 2> ev_ext{}, ev_comm{};
    bool direct_nccl_unpack = false;
    BlockGeom* d_geom = nullptr;
    unsigned int* d_sched = nullptr;            // [2*(n_local+1)] stencil work counters
    bool xsector_ok = true;  // J3D_XSECTOR=0 disables whole-sector x-ghost stores (tuning)
    std::vector<int> item_begin, item_count;  // per local block, in d_items
    std::vector<int64_t> item_cells;          // prefix sums of owned cells per item (profiling bytes)
    int n_items = 0, tile_kind = 0, grid_cap = 0;
    bool faces_fused = false;                   // stencil launches carry prologue/epilogue faces
    std::vector<int> order;                     // local blocks, peer-face blocks first

    // streams, events
    cudaStream_t main = nullptr;
    std::vector<cudaStream_t> lo, hi;
    std::vector<std::array<cudaEvent_t, 2>> ev_st, ev_pk, ev_up;
    std::array<cudaEvent_t, 2> ev_xw{};
    cudaEvent_t ev_fork = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;

    ncclComm_t comm = nullptr;
    std::vector<int> peer_ranks;  // distinct neighbour ranks

    // state
    int64_t iter = 0;             // iterations since init
    int64_t iter_since_set = 0;   // for residual validity
    bool halos_stale = false;
    bool skip_exchange = false;
    int64_t refresh_count = 0;
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    int64_t graph_kernels[2] = {0, 0};
    std::vector<int64_t> graph_block_launches[2];
    bool capturing = false;
    int capture_parity = 0;

    // stats
    int64_t stat_launches = 0, stat_graph_launches = 0, stat_last_parity = -1, stat_iters = 0;
    std::vector<int64_t> block_launches;

    // profiling
    bool prof = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
    std::vector<cudaEvent_t> ev_pool;
    double prof_ms = 0, prof_bytes = 0, prof_pending_bytes = 0;
    int64_t prof_launches = 0;

    // ------------------------------------------------------------ addresses
    double* buf(int l, int par, int rank_base = -1) const {
        const char* base = rank_base < 0 ? arena : peer_base[rank_base];
        return (double*)(base + off_bufs + ((int64_t)l * 2 + par) * buf_bytes);
    }
    double* face_buf(int l, int f, int par, bool recv, int rank_base = -1) const {
        const char* base = rank_base < 0 ? arena : peer_base[rank_base];
        int64_t o = off_faces + (int64_t)l * faces_per_block_bytes;
        for (int g = 0; g < f; ++g) o += 4 * face_bytes[g];
        o += ((recv ? 2 : 0) + par) * face_bytes[f];
        return (double*)(base + o);
    }
    uint64_t* flags(int rank_base = -1) const {
        const char* base = rank_base < 0 ? arena : peer_base[rank_base];
        return (uint64_t*)(base + off_flags);
    }
    int64_t face_na(int f) const { return f < 2 ? ny : nx; }
    int64_t face_nb(int f) const { return f < 4 ? nz : ny; }
    // owned (ghost=false) or ghost layer of a block buffer on face f as a FaceRef over (a,b)
    FaceRef layer(double* b, int f, bool ghost) const {
        const int a = f >> 1;
        const int64_t n = a == 0 ? nx : a == 1 ? ny : nz;
        const int64_t c = (f & 1) ? (ghost ? n : n - 1) : (ghost ? -1 : 0);
        double* o = b + zs + pitch + XOFF;  // owned (0,0,0)
        if (a == 0) return FaceRef{o + c, pitch, zs};
        if (a == 1) return FaceRef{o + c * pitch, 1, zs};
        return FaceRef{o + c * zs, 1, pitch};
    }
    FaceRef contiguous(double* p, int f) const { return FaceRef{p, 1, face_na(f)}; }
};

namespace {

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
    if (c->launch != J3D_PER_BLOCK && c->launch != J3D_BATCHED) return fail(J3D_EINVAL, "unknown launch mode");
    if (c->exchange < J3D_XCHG_AUTO || c->exchange > J3D_XCHG_HOST) return fail(J3D_EINVAL, "unknown exchange backend");
    if (c->n_gpus < 1 || c->rank < 0 || c->rank >= c->n_gpus) return fail(J3D_EINVAL, "rank / n_gpus out of range");
    if (c->odf < 1) return fail(J3D_EINVAL, "odf must be >= 1");
    if (c->reserved != 0 || (c->overlap != 0 && c->overlap != 1)) return fail(J3D_EINVAL, "bad overlap/reserved");
    return J3D_OK;
}

bool unfused_family(const jacobi3d* c) { return c->cfg.variant <= J3D_FUSE_B; }

// ---------------------------------------------------------------- setup
void build_layout(jacobi3d* c) {
    const Plan& P = c->plan;
    c->nx = P.ext[0];
    c->ny = P.ext[1];
    c->nz = P.ext[2];
    c->pitch = align_up(XOFF + c->nx + 1, PITCH_ALIGN);
    c->zs = c->pitch * (c->ny + 2);
    c->buf_elems = c->zs * (c->nz + 2);
    c->buf_bytes = align_up(c->buf_elems * 8, 256);
    for (int f = 0; f < 6; ++f) c->face_bytes[f] = align_up(face_cells(P.ext, f) * 8, 256);
    c->faces_per_block_bytes = 0;
    for (int f = 0; f < 6; ++f) c->faces_per_block_bytes += 4 * c->face_bytes[f];  // send/recv x 2 parities
    c->off_flags = 0;
    c->off_scratch = 2048;
    c->off_bufs = 4096;
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

void build_tables(jacobi3d* c) {
    const int nl = c->n_local;
    const int v = c->cfg.variant;
    // ---- stencil descriptors [2*l + p]
    std::vector<StencilDesc> descs(2 * nl);
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
                    bool direct = v == J3D_FUSE_DIRECT && (k == LOCAL || k == PEER_P2P);
                    if (direct) {
                        const int r = k == LOCAL ? -1 : c->plan.blocks[c->plan.blocks[c->gid[l]].nbr[f]].owner;
                        if (k == PEER_P2P && !c->p2p_connected) continue;  // filled after ipc_connect
                        d.epi[f] = c->layer(c->buf(c->nbr_local[l][f], q, r), f ^ 1, true);
                        d.epi_mask |= 1u << f;
                        if (f < 2 && (c->nx % 4) == 0 && c->xsector_ok) d.xsector |= 1u << f;  // whole-sector x-ghost stores
                    } else if (v == J3D_FUSE_DIRECT) {
                        // NCCL face of the direct variant: epilogue packs into the
                        // send buffer; after the exchange a batched unpack kernel
                        // writes the received face into the ghost layer (keeps the
                        // stencil's prologue empty)
                        d.epi[f] = pack_dst(c, l, f, q);
                        d.epi_mask |= 1u << f;
                    } else {
                        if (k == PEER_P2P && !c->p2p_connected) continue;
                        d.epi[f] = pack_dst(c, l, f, q);
                        d.epi_mask |= 1u << f;
                        d.pro[f] = recv_src(c, l, f, p);
                        d.pro_mask |= 1u << f;
                    }
                }
                if (d.epi_mask | d.pro_mask) c->faces_fused = true;
            }
        }
    CK(cudaMemcpy(c->d_descs, descs.data(), descs.size() * sizeof(StencilDesc), cudaMemcpyHostToDevice));

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
    // NCCL faces only (direct variant's post-exchange unpack)
    c->direct_nccl_unpack = false;
    for (int q = 0; q < 2; ++q)
        for (int l = 0; l < nl; ++l)
            for (int f = 0; f < 6; ++f) {
                CopyDesc& up = unpack[(q * nl + l) * 6 + f];
                if (!via_buffers(c->kind[l][f])) std::memset(&up, 0, sizeof up);
                else if (v == J3D_FUSE_DIRECT) c->direct_nccl_unpack = true;
            }
    CK(cudaMemcpy(c->d_unpack_nccl, unpack.data(), unpack.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
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
}

void build_static_tables(jacobi3d* c) {
    const int nl = c->n_local;
    // ---- tensor maps [2*l + p] over each input buffer
    g_drv.load();
    // 192x22 tiles (11 consumer warps, 5-stage ring, 1 CTA/SM) when they divide
    // the block width, else 128x30 (15 consumer warps) for wide blocks and
    // 64x16 (2 CTAs/SM, 6 stages) for narrow ones.  Bench sweeps: profiles/.
    c->tile_kind = (c->nx % 192 == 0) ? 0 : c->nx >= 128 ? 1 : 4;
    {  // small grids: the wide tiles cannot keep every SM busy -> 64x16, 2 CTAs/SM
        const TileShape t = tile_shape(c->tile_kind);
        const int64_t tiles = ((c->nx + t.tx - 1) / t.tx) * ((c->ny + t.ty - 1) / t.ty) * nl;
        const int64_t max_items = tiles * std::max<int64_t>(1, c->nz / 24);
        if (c->tile_kind != 4 && max_items < 4LL * c->sms) c->tile_kind = 4;
    }
    if (const char* e = std::getenv("J3D_TILE")) {  // tuning override (bench sweeps)
        const int k = std::atoi(e);
        if (k >= 0 && k < num_tile_kinds()) c->tile_kind = k;
    }
    const TileShape ts = tile_shape(c->tile_kind);
    std::vector<CUtensorMap> maps(2 * nl);
    CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    if (const char* e = std::getenv("J3D_L2PROMO")) {  // tuning override
        const int v = std::atoi(e);
        promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
              : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }
    for (int l = 0; l < nl; ++l)
        for (int p = 0; p < 2; ++p) {
            cuuint64_t dims[3] = {(cuuint64_t)(XOFF + c->nx + 1), (cuuint64_t)(c->ny + 2), (cuuint64_t)(c->nz + 2)};  // up to the +x ghost: the row padding is never fetched (TMA zero-fills beyond)
            cuuint64_t strides[2] = {(cuuint64_t)(c->pitch * 8), (cuuint64_t)(c->zs * 8)};
            cuuint32_t box[3] = {(cuuint32_t)stencil_box_w(c->tile_kind), (cuuint32_t)stencil_box_h(c->tile_kind), 1};
            cuuint32_t es[3] = {1, 1, 1};
            DK(g_drv.encode(&maps[2 * l + p], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->buf(l, p), dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
        }
    CK(cudaMemcpy(c->d_tmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
    // split maps: box heights 2 and H-4 (for the L2-policy split loads)
    std::vector<CUtensorMap> maps2(4 * nl);
    for (int l = 0; l < nl; ++l)
        for (int p = 0; p < 2; ++p)
            for (int h = 0; h < 2; ++h) {
                cuuint64_t dims[3] = {(cuuint64_t)(XOFF + c->nx + 1), (cuuint64_t)(c->ny + 2), (cuuint64_t)(c->nz + 2)};  // up to the +x ghost: the row padding is never fetched (TMA zero-fills beyond)
                cuuint64_t strides[2] = {(cuuint64_t)(c->pitch * 8), (cuuint64_t)(c->zs * 8)};
                const int H = stencil_box_h(c->tile_kind);
                cuuint32_t box[3] = {(cuuint32_t)stencil_box_w(c->tile_kind), (cuuint32_t)(h == 0 ? 2 : std::max(1, H - 4)), 1};
                cuuint32_t es[3] = {1, 1, 1};
                DK(g_drv.encode(&maps2[(2 * l + p) * 2 + h], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->buf(l, p), dims,
                                strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
            }
    CK(cudaMemcpy(c->d_tmaps_split, maps2.data(), maps2.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
    if (const char* e = std::getenv("J3D_TMA_HINT")) c->tma_mode = std::atoi(e) & 3;
    if (c->tma_mode == 3 && stencil_box_h(c->tile_kind) < 6) c->tma_mode = 0;

    // ---- work items: per block, z-chunk outer, then ty, tx (x fastest), peer-face blocks first
    int occ = 1;
    CK(stencil_occupancy(c->tile_kind, false, &occ));
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
    // small problems: shorter chunks until there are >= 6 items per CTA slot
    // (at least 24 planes per chunk): the last round of items is then short
    // (measured: 96^3 blocks, ODF 64: 198 -> 225 GLUPS)
    while (tiles * best_zc < 6 * (int64_t)c->grid_cap && c->nz / (best_zc + 1) >= 24) ++best_zc;
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
    c->n_ext = 0;
    if (c->overlap) {  // BATCHED only: exterior items of every block first (stable order otherwise)
        std::stable_partition(items.begin(), items.end(), exterior);
        c->n_ext = (int)std::count_if(items.begin(), items.end(), exterior);
    }
    c->n_items = (int)items.size();
    c->item_cells.assign(items.size() + 1, 0);
    for (size_t i = 0; i < items.size(); ++i) {
        const WorkItem& w = items[i];
        const int64_t ex = std::min<int64_t>(ts.tx, c->nx - (int64_t)w.tx * ts.tx);
        const int64_t ey = std::min<int64_t>(ts.ty, c->ny - (int64_t)w.ty * ts.ty);
        c->item_cells[i + 1] = c->item_cells[i] + ex * ey * (w.z1 - w.z0);
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
    }
    CK(cudaMemcpy(c->d_geom, geo.data(), geo.size() * sizeof(BlockGeom), cudaMemcpyHostToDevice));
}

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

void stencil(jacobi3d* c, int begin, int count, int parity, cudaStream_t st, int l) {
    if (count <= 0) return;
    StencilLaunch L;
    L.descs = c->d_descs;
    L.tmaps = c->d_tmaps;
    L.tmaps_split = c->d_tmaps_split;
    L.tma_mode = c->tma_mode;
    L.items = c->d_items + begin;
    L.n_items = count;
    L.parity = parity;
    L.grid = std::min(count, c->grid_cap);
    L.kind = c->tile_kind;
    L.faces = c->faces_fused;
    L.sched = c->d_sched + 2 * (l + 1);  // one counter pair per concurrently running launch
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
        c->prof_pending_bytes += 16.0 * (double)cells;
    }
}

void copies(jacobi3d* c, CopyDesc* table, int parity, int l, int face, bool fused, cudaStream_t st) {
    // table layout [(q*nl + l)*6 + f]
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

// NCCL faces: one group per exchange on the main stream (C4).  Messages to a
// peer are posted in the canonical order (sender block id, sender face) on
// both sides so the k-th send matches the k-th receive.
void nccl_exchange(jacobi3d* c, int par, cudaStream_t st) {
    struct Msg { int64_t key; int l, f; bool send; };
    std::vector<Msg> msgs;
    for (int l = 0; l < c->n_local; ++l)
        for (int f = 0; f < 6; ++f) {
            if (c->kind[l][f] != PEER_NCCL) continue;
            const int64_t me = c->gid[l], nb = c->plan.blocks[me].nbr[f];
            msgs.push_back({me * 6 + f, l, f, true});
            msgs.push_back({nb * 6 + (f ^ 1), l, f, false});
        }
    if (msgs.empty()) return;
    std::stable_sort(msgs.begin(), msgs.end(), [](const Msg& a, const Msg& b) { return a.key < b.key; });
    NK(ncclGroupStart());
    for (const Msg& m : msgs) {
        const int peer = c->plan.blocks[c->plan.blocks[c->gid[m.l]].nbr[m.f]].owner;
        const size_t n = (size_t)face_cells(c->plan.ext, m.f);
        if (m.send) NK(ncclSend(c->face_buf(m.l, m.f, par, false), n, ncclFloat64, peer, c->comm, st));
        else NK(ncclRecv(c->face_buf(m.l, m.f, par, true), n, ncclFloat64, peer, c->comm, st));
    }
    NK(ncclGroupEnd());
}

// P2P epoch flags: toggle protocol on slot s (consecutive syncs always use
// different slots).  Signal: write 1 into every
// neighbour rank's flag[s][me] (stream write = release fence after all prior
// work on the stream, i.e. after our NVLink stores).  Wait: until own
// flag[s][r] == 1 for every neighbour r, then reset it to 0.
void p2p_sync(jacobi3d* c, int slot, cudaStream_t st) {
    if (!c->p2p_needed) return;
    const int n = c->n_gpus;
    for (int r : c->peer_ranks) {
        uint64_t* f = c->flags(r) + slot * n + c->rank;
        DK(g_drv.write64((CUstream)st, (CUdeviceptr)f, 1, 0));
    }
    for (int r : c->peer_ranks) {
        uint64_t* f = c->flags() + slot * n + r;
        DK(g_drv.wait64((CUstream)st, (CUdeviceptr)f, 1, CU_STREAM_WAIT_VALUE_EQ));
        DK(g_drv.write64((CUstream)st, (CUdeviceptr)f, 0, 0));
    }
}

// ---------------------------------------------------------------- host staging
int64_t shm_flags_bytes(const jacobi3d* c) { return align_up(8 * 8 * (int64_t)c->n_gpus, 4096); }
int64_t shm_area_offset(const jacobi3d* c, int l, int f, int par) {
    int64_t o = shm_flags_bytes(c) + (int64_t)l * 2 * [&] {
        int64_t t = 0;
        for (int g = 0; g < 6; ++g) t += c->face_bytes[g];
        return t;
    }();
    for (int g = 0; g < f; ++g) o += 2 * c->face_bytes[g];
    return o + par * c->face_bytes[f];
}
std::string shm_name(uint64_t key, int rank) {
    char b[64];
    std::snprintf(b, sizeof b, "/j3d_%016llx_%d", (unsigned long long)key, rank);
    return b;
}

void host_setup_own(jacobi3d* c) {  // at create: own segment (peers map it in ipc_connect)
    int64_t per_block = 0;
    for (int g = 0; g < 6; ++g) per_block += 2 * c->face_bytes[g];
    c->shm_bytes = (size_t)(shm_flags_bytes(c) + per_block * c->n_local);
    c->shm_base.assign(c->n_gpus, nullptr);
    c->shm_dev.assign(c->n_gpus, nullptr);
    const std::string nm = shm_name(c->job_key, c->rank);
    shm_unlink(nm.c_str());
    const int fd = shm_open(nm.c_str(), O_CREAT | O_RDWR, 0600);
    if (fd < 0) throw Error(J3D_ENOMEM, "shm_open " + nm + " failed");
    if (ftruncate(fd, (off_t)c->shm_bytes) != 0) {
        close(fd);
        throw Error(J3D_ENOMEM, "ftruncate of the staging segment failed");
    }
    void* p = mmap(nullptr, c->shm_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw Error(J3D_ENOMEM, "mmap of the staging segment failed");
    std::memset(p, 0, (size_t)shm_flags_bytes(c));
    c->shm_base[c->rank] = (char*)p;
    CK(cudaHostRegister(p, c->shm_bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
    void* d = nullptr;
    CK(cudaHostGetDevicePointer(&d, p, 0));
    c->shm_dev[c->rank] = (char*)d;
}

void host_connect(jacobi3d* c) {  // map every neighbour rank's segment
    for (int r : c->peer_ranks) {
        const std::string nm = shm_name(c->job_key, r);
        const int fd = shm_open(nm.c_str(), O_RDWR, 0600);
        if (fd < 0) throw Error(J3D_EINVAL, "shm_open " + nm + " failed (ranks must share one node)");
        void* p = mmap(nullptr, c->shm_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (p == MAP_FAILED) throw Error(J3D_ENOMEM, "mmap of a neighbour's staging segment failed");
        c->shm_base[r] = (char*)p;
        CK(cudaHostRegister(p, c->shm_bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
        void* d = nullptr;
        CK(cudaHostGetDevicePointer(&d, p, 0));
        c->shm_dev[r] = (char*)d;
    }
    c->host_connected = true;
}

void host_teardown(jacobi3d* c) {
    for (size_t r = 0; r < c->shm_base.size(); ++r) {
        if (!c->shm_base[r]) continue;
        cudaHostUnregister(c->shm_base[r]);
        munmap(c->shm_base[r], c->shm_bytes);
        if ((int)r == c->rank) shm_unlink(shm_name(c->job_key, c->rank).c_str());
        c->shm_base[r] = nullptr;
    }
}

// Host-staged exchange of the PEER_HOST faces of parity par on stream st:
// D2H of my send buffers into my segment, epoch signal into each neighbour's
// segment flags, wait for theirs, H2D of their staging areas into my receive
// buffers.  Flags: toggle protocol on slot (same rules as P2P, see p2p_sync).
void host_exchange(jacobi3d* c, int par, int slot, cudaStream_t st) {
    if (!c->host_needed) return;
    const int n = c->n_gpus;
    for (int l = 0; l < c->n_local; ++l)
        for (int f = 0; f < 6; ++f)
            if (c->kind[l][f] == PEER_HOST)
                CK(cudaMemcpyAsync(c->shm_base[c->rank] + shm_area_offset(c, l, f, par),
                                   c->face_buf(l, f, par, false), (size_t)face_cells(c->plan.ext, f) * 8,
                                   cudaMemcpyDeviceToHost, st));
    for (int r : c->peer_ranks)
        DK(g_drv.write64((CUstream)st, (CUdeviceptr)((uint64_t*)c->shm_dev[r] + slot * n + c->rank), 1, 0));
    for (int r : c->peer_ranks) {
        CUdeviceptr f = (CUdeviceptr)((uint64_t*)c->shm_dev[c->rank] + slot * n + r);
        DK(g_drv.wait64((CUstream)st, f, 1, CU_STREAM_WAIT_VALUE_EQ));
        DK(g_drv.write64((CUstream)st, f, 0, 0));
    }
    for (int l = 0; l < c->n_local; ++l)
        for (int f = 0; f < 6; ++f)
            if (c->kind[l][f] == PEER_HOST) {
                const int r = c->plan.blocks[c->plan.blocks[c->gid[l]].nbr[f]].owner;
                CK(cudaMemcpyAsync(c->face_buf(l, f, par, true),
                                   c->shm_base[r] + shm_area_offset(c, c->nbr_local[l][f], f ^ 1, par),
                                   (size_t)face_cells(c->plan.ext, f) * 8, cudaMemcpyHostToDevice, st));
            }
}

// epoch barrier through the host segments (refresh pre-barrier of the host backend)
void host_sync(jacobi3d* c, int slot, cudaStream_t st) {
    if (!c->host_needed) return;
    const int n = c->n_gpus;
    for (int r : c->peer_ranks)
        DK(g_drv.write64((CUstream)st, (CUdeviceptr)((uint64_t*)c->shm_dev[r] + slot * n + c->rank), 1, 0));
    for (int r : c->peer_ranks) {
        CUdeviceptr f = (CUdeviceptr)((uint64_t*)c->shm_dev[c->rank] + slot * n + r);
        DK(g_drv.wait64((CUstream)st, f, 1, CU_STREAM_WAIT_VALUE_EQ));
        DK(g_drv.write64((CUstream)st, f, 0, 0));
    }
}

void cross_gpu_exchange(jacobi3d* c, int par, int slot, cudaStream_t st) {
    if (c->n_gpus == 1 || c->skip_exchange) return;
    nccl_exchange(c, par, st);
    p2p_sync(c, slot, st);
    host_exchange(c, par, slot, st);
}

// Full halo refresh of buffer parity `par`: pack, exchange, unpack, batched on
// main.  With P2P peers it starts with an epoch barrier (slots 4/5): a peer's
// NVLink stores into our receive buffers may only begin once we have finished
// every earlier use of them (the caller's state change, e.g. init or
// set_block, or the last iteration of a previous run).
void refresh(jacobi3d* c, int par) {
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
            stencil(c, 0, c->n_ext, p, c->main, -1);
            CK(cudaEventRecord(c->ev_ext[q], c->main));
            CK(cudaStreamWaitEvent(c->xstream, c->ev_ext[q], 0));
            if (unf) copies(c, c->d_pack_peer, q, -1, 0, true, c->xstream);
            cross_gpu_exchange(c, q, q, c->xstream);
            if (unf) copies(c, c->d_unpack_peer, q, -1, 0, true, c->xstream);
            else if (c->direct_nccl_unpack) copies(c, c->d_unpack_nccl, q, -1, 0, true, c->xstream);
            CK(cudaEventRecord(c->ev_comm[q], c->xstream));
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
    if (c->halos_stale) {
        if (c->n_gpus > 1)
            throw Error(J3D_ESTATE, "halos are stale after set_block: call jacobi3d_refresh_halos on every rank");
        refresh(c, (int)(c->iter & 1));
        c->halos_stale = false;
    }
    if (c->p2p_needed && !c->p2p_connected)
        throw Error(J3D_ESTATE, "P2P exchange needs jacobi3d_ipc_export/jacobi3d_ipc_connect first");
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
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
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
    for (auto s : c->lo) if (s) cudaStreamDestroy(s);
    for (auto s : c->hi) if (s) cudaStreamDestroy(s);
    if (c->comm) ncclCommDestroy(c->comm);
    for (size_t r = 0; r < c->peer_base.size(); ++r)
        if (c->peer_base[r]) cudaIpcCloseMemHandle(c->peer_base[r]);
    host_teardown(c);
    if (c->main) cudaStreamDestroy(c->main);
    cudaFree(c->d_descs);
    cudaFree(c->d_tmaps);
    cudaFree(c->d_tmaps_split);
    cudaFree(c->d_items);
    cudaFree(c->d_pack);
    cudaFree(c->d_unpack);
    cudaFree(c->d_unpack_nccl);
    cudaFree(c->d_pack_peer);
    cudaFree(c->d_unpack_peer);
    cudaFree(c->d_pack_local);
    cudaFree(c->d_unpack_local);
    cudaFree(c->d_geom);
    cudaFree(c->d_sched);
    cudaFree(c->arena);
    delete c;
}

// Host wait for all work queued on `st`.  Multi-GPU contexts poll with a
// watchdog (J3D_TIMEOUT_S, default 600 s): a peer that never signals its
// epoch (or an NCCL error) surfaces as J3D_ETIMEOUT / J3D_ENCCL instead of a
// hang.
void wait_stream(jacobi3d* c, cudaStream_t st) {
    if (c->n_gpus == 1) {
        CK(cudaStreamSynchronize(st));
        return;
    }
    double limit = 600.0;
    if (const char* e = std::getenv("J3D_TIMEOUT_S")) limit = std::atof(e);
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

void nccl_barrier(jacobi3d* c) {
    if (c->n_gpus == 1 || !c->comm) return;
    double* s = (double*)(c->arena + c->off_scratch + 64);
    NK(ncclAllReduce(s, s, 1, ncclFloat64, ncclSum, c->comm, c->main));
    wait_stream(c, c->main);
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
        const int64_t buf = align_up(pitch * (ny + 2) * (nz + 2) * 8, 256);
        int64_t faces = 0;
        for (int f = 0; f < 6; ++f) faces += 4 * align_up(face_cells(P.ext, f) * 8, 256);
        out->bytes_per_gpu = 4096 + (int64_t)P.odf * (2 * buf + faces);
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
        CK(cudaMemset(c->arena, 0, 4096));
        // face buffers start zeroed; done here, before any peer can map the
        // arena, so it can never race with a peer's NVLink stores
        CK(cudaMemset(c->arena + c->off_faces, 0, (size_t)(c->arena_bytes - c->off_faces)));
        CK(cudaMalloc(&c->d_descs, sizeof(StencilDesc) * 2 * c->n_local));
        CK(cudaMalloc(&c->d_tmaps, sizeof(CUtensorMap) * 2 * c->n_local));
        CK(cudaMalloc(&c->d_tmaps_split, sizeof(CUtensorMap) * 4 * c->n_local));
        CK(cudaMalloc(&c->d_pack, sizeof(CopyDesc) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_unpack, sizeof(CopyDesc) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_unpack_nccl, sizeof(CopyDesc) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_pack_peer, sizeof(CopyDesc) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_unpack_peer, sizeof(CopyDesc) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_pack_local, sizeof(CopyDesc) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_unpack_local, sizeof(CopyDesc) * 12 * c->n_local));
        CK(cudaMalloc(&c->d_geom, sizeof(BlockGeom) * c->n_local));
        CK(cudaMalloc(&c->d_sched, sizeof(unsigned int) * 2 * (c->n_local + 1)));
        CK(cudaMemset(c->d_sched, 0, sizeof(unsigned int) * 2 * (c->n_local + 1)));
        if (const char* e = std::getenv("J3D_XSECTOR")) c->xsector_ok = std::atoi(e) != 0;
        c->peer_base.assign(c->n_gpus, nullptr);
        build_static_tables(c);
        build_tables(c);
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
        if (c->n_gpus > 1) {
            ncclUniqueId id;
            std::memcpy(&id, nccl_uid, 128);
            NK(ncclCommInitRank(&c->comm, c->n_gpus, id, c->rank));
            uint64_t h = 1469598103934665603ULL;  // FNV-1a of the unique id: a job-wide key
            for (int i = 0; i < 128; ++i) h = (h ^ nccl_uid[i]) * 1099511628211ULL;
            c->job_key = h;
        }
        if (c->host_needed) {
            g_drv.load();
            host_setup_own(c);
        }
        CK(cudaDeviceSynchronize());
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
        CK(cudaSetDevice(c->device));
        if (c->p2p_needed) CK(cudaIpcGetMemHandle(&r.handle, c->arena));
        std::memcpy(host_out, &r, sizeof r);
        return J3D_OK;
    });
}

int jacobi3d_ipc_connect(jacobi3d_t* c, const uint8_t* all, size_t len_per_rank) {
    return guarded([&]() -> int {
        if (!c || !all) return fail(J3D_EINVAL, "NULL argument");
        if (c->host_needed && !c->host_connected) {
            CK(cudaSetDevice(c->device));
            host_connect(c);
        }
        if (!c->p2p_needed) return J3D_OK;
        if (len_per_rank != sizeof(IpcRecord)) return fail(J3D_EINVAL, "record size mismatch");
        CK(cudaSetDevice(c->device));
        for (int r : c->peer_ranks) {
            IpcRecord rec;
            std::memcpy(&rec, all + (size_t)r * len_per_rank, sizeof rec);
            if (rec.magic != kIpcMagic || rec.rank != r || rec.arena_bytes != (uint64_t)c->arena_bytes)
                return fail(J3D_EINVAL, "bad IPC record for rank " + std::to_string(r));
            int can = 0;
            cudaDeviceCanAccessPeer(&can, c->device, rec.device);
            if (!can && rec.device != c->device)
                return fail(J3D_EUNSUPPORTED, "device " + std::to_string(c->device) + " cannot access peer device " +
                                                  std::to_string(rec.device));
            void* p = nullptr;
            CK(cudaIpcOpenMemHandle(&p, rec.handle, cudaIpcMemLazyEnablePeerAccess));
            c->peer_base[r] = (char*)p;
        }
        c->p2p_connected = true;
        drop_graphs(c);
        build_tables(c);
        CK(cudaDeviceSynchronize());
        return J3D_OK;
    });
}

int jacobi3d_init(jacobi3d_t* c, int kind, const double* p, uint64_t seed) {
    return guarded([&]() -> int {
        if (!c) return fail(J3D_EINVAL, "ctx is NULL");
        if (kind < J3D_INIT_DEFAULT || kind > J3D_INIT_HASH) return fail(J3D_EINVAL, "unknown init kind");
        if ((kind == J3D_INIT_CONST || kind == J3D_INIT_LINEAR) && !p) return fail(J3D_EINVAL, "params required");
        if ((c->p2p_needed && !c->p2p_connected) || (c->host_needed && !c->host_connected))
            return fail(J3D_ESTATE, "P2P / host exchange needs jacobi3d_ipc_export/jacobi3d_ipc_connect first");
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
        wait_stream(c, c->main);
        CK(cudaDeviceSynchronize());
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
        if (c->n_gpus > 1) NK(ncclAllReduce(acc, acc, 1, ncclUint64, ncclMax, c->comm, c->main));
        unsigned long long h = 0;
        CK(cudaMemcpyAsync(&h, acc, 8, cudaMemcpyDeviceToHost, c->main));
        wait_stream(c, c->main);
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
        if (c->n_gpus > 1) NK(ncclAllReduce(acc, acc, 1, ncclUint64, ncclSum, c->comm, c->main));
        unsigned long long h = 0;
        CK(cudaMemcpyAsync(&h, acc, 8, cudaMemcpyDeviceToHost, c->main));
        wait_stream(c, c->main);
        *out = (uint64_t)h;
        return J3D_OK;
    });
}

int jacobi3d_time(jacobi3d_t* c, int64_t warmup, int64_t iters, double* ms) {
    return guarded([&]() -> int {
        if (!c || !ms || iters < 1 || warmup < 0) return fail(J3D_EINVAL, "bad argument");
        CK(cudaSetDevice(c->device));
        do_iterate(c, warmup);
        wait_stream(c, c->main);
        CK(cudaDeviceSynchronize());
        nccl_barrier(c);
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
        CK(cudaDeviceSynchronize());
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
        CK(cudaDeviceSynchronize());
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
