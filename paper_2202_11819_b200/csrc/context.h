// context.h -- internal state of a Jacobi3D context (one rank, one GPU) and
// the functions the csrc translation units share:
//   setup.cu        arena layout, face classification, device tables, tensor maps, work items
//   launch.cu       kernel launches (stencil, face copies) and the per-iteration orchestration
//   exchange.cu     cross-GPU exchange: NCCL, NVLink P2P epochs, host staging
//   api.cu          the C ABI (include/jacobi3d.h)
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
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <mutex>
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

// NVTX range on the host timeline around each phase the library enqueues
// (stencil, pack, exchange, unpack, waits): header-only NVTX v3, a no-op unless
// a profiler is attached (phase ranges for the exposed-halo cross-check)
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

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
    void load() {  // once per process; ranks may be threads of one process
        static std::mutex m;
        std::lock_guard<std::mutex> g(m);
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
extern Driver g_drv;

enum FaceKind { DIRICHLET = 0, LOCAL = 1, PEER_NCCL = 2, PEER_P2P = 3, PEER_HOST = 4 };
// faces whose data travels through the send/receive buffers in a separate exchange step
static inline bool via_buffers(int k) { return k == PEER_NCCL || k == PEER_HOST; }
static inline bool is_peer_kind(int k) { return k == PEER_NCCL || k == PEER_P2P || k == PEER_HOST; }

static inline int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// One rank's connection record (jacobi3d_ipc_export): the CUDA IPC handle of
// its arena for peers in other processes, the raw arena address for peers in
// the same process (ranks run as threads; an IPC handle cannot be opened in
// the process that exported it), and the GPU's UUID, which tells ranks that
// share a GPU apart from ranks on different GPUs.
struct IpcRecord {
    uint64_t magic;
    int32_t rank, device;
    uint64_t arena_bytes;          // offset 16 (tests read it)
    cudaIpcMemHandle_t handle;
    uint64_t process;              // process_token() of the exporting process
    uint64_t arena_ptr;            // the arena's device address in that process
    uint8_t uuid[16];              // cudaDeviceProp::uuid of the rank's GPU
};
static const uint64_t kIpcMagic = 0x4a33445f49504332ULL;  // "J3D_IPC2"
uint64_t process_token();          // random, fixed for the life of the process

}  // namespace j3d

using namespace j3d;

struct jacobi3d {
    jacobi3d_config cfg{};
    Plan plan;
    int rank = 0, n_gpus = 1, device = 0, sms = 148;
    int64_t nx = 0, ny = 0, nz = 0, pitch = 0, zs = 0, buf_elems = 0;
    int64_t grid_bytes = 0;  // the ghosted 3D array of one buffer (256-B aligned)
    int64_t xg_pitch = 0;    // x ghost arrays: doubles per z plane (ny rounded up to even)
    int64_t xg_bytes = 0;    // one x ghost array (nz+2 planes), 256-B aligned
    int n_local = 0;
    std::vector<int64_t> gid;                 // local index -> global block id
    std::vector<std::array<int, 6>> kind;     // FaceKind per local block face
    std::vector<std::array<int, 6>> nbr_local;// neighbour's local index (LOCAL) or its owner-local index (PEER)
    std::vector<uint8_t> has_peer;

    // arena layout (identical on every rank)
    char* arena = nullptr;
    int64_t arena_bytes = 0, off_flags = 0, off_scratch = 0, off_done = 0, off_bufs = 0, buf_bytes = 0, off_faces = 0;
    std::array<int64_t, 6> face_bytes{};
    int64_t faces_per_block_bytes = 0;
    std::vector<char*> peer_base;  // mapped arenas (index = rank), nullptr for self
    std::vector<uint8_t> peer_ipc; // peer_base[r] was opened with cudaIpcOpenMemHandle (else same process)
    bool p2p_needed = false, p2p_connected = false;
    // host control plane (n_gpus > 1 without an NCCL communicator, control.cu):
    // one POSIX shared-memory segment per rank with a collective sequence
    // number and two value slots -- barrier, sum and max over all ranks
    bool ctl_needed = false, ctl_connected = false;
    uint64_t ctl_seq = 0;
    std::vector<char*> ctl_base;   // mapped segments (index = rank; own included)
    int co_resident = 1;           // ranks of this job on this GPU (threads of one process)
    bool streams_aliased = false;  // co_resident > 1: lo / hi are the main stream (api.cu connect)
    int persist_grid = 0;          // persistent grid: grid_cap / co_resident (all co-resident ranks fit)
    uint64_t* host_scratch = nullptr;  // pinned: residual / checksum results
    // host staging (J3D_XCHG_HOST): one POSIX shared-memory segment per rank,
    // [flags: 8 slots x n_gpus uint64 | staging: per local block, face, parity],
    // registered with CUDA so stream memory ops and DMA copies reach it
    bool host_needed = false, host_connected = false;
    uint64_t job_key = 0;
    size_t shm_bytes = 0;
    std::vector<char*> shm_base;      // mapped segments (index = rank; own included)
    std::vector<char*> shm_dev;       // device-visible address of each mapped segment
    CopyDesc* d_stage_out = nullptr;  // [(q*nl + l)*6 + f] send buffer -> own segment (staged D2H)
    CopyDesc* d_stage_in = nullptr;   // [(q*nl + l)*6 + f] neighbour's segment -> receive buffer (staged H2D)

    // device tables
    StencilDesc* d_descs = nullptr;
    CUtensorMap* d_tmaps = nullptr;
    CUtensorMap* d_tmaps_pro = nullptr;  // [2*l + p][6] strategy C: maps over the receive buffers the prologue reads
    CUtensorMap* d_tmaps_x = nullptr;  // [2*l + p] x ghost vectors of each buffer
    // L2 policy of the stencil's plane loads: evict_last (2) ranks the input planes ahead
    // of the output lines in L2.  Measured: 1536^3 383.0 -> 388.5 GLUPS over 100 steps with
    // the same DRAM bytes (ncu 1.033x) in a shorter launch (profiles/r02_tuning_log.md);
    // J3D_TMA_HINT=0 / 1: plain / evict_first
    int tma_mode = 2;
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
    bool direct_nccl_unpack = false;             // direct variant: post-exchange unpack of buffered faces
    bool direct_push = false;                    // direct variant: peer x faces pushed send -> peer recv
    CopyDesc* d_push = nullptr;
    BlockGeom* d_geom = nullptr;
    unsigned int* d_sched = nullptr;            // [2*(n_local+1)] stencil work counters
    bool peer_x_pack = true;     // peer x faces packed from the output by the push kernel (J3D_PEERX_PACK=0:
                                 // captured by the stencil epilogue into the send buffer; tuning)
    bool peer_x_direct = false;  // J3D_PEERX_DIRECT=1: peer x ghosts stored over NVLink from the epilogue (tuning)
    std::vector<int> item_begin, item_count;  // per local block, in d_items
    std::vector<int64_t> item_cells;          // prefix sums of owned cells per item (profiling bytes)
    int n_items = 0, tile_kind = 0, grid_cap = 0;
    bool tile_ys = false;                     // strategy C: the tile instance with y side rows (kernels.cu)
    bool depfence = false;                    // J3D_DEPFENCE=1: extra fence after the dependency polling (experiment)
    bool prefetch = false;                    // J3D_PREFETCH=1: claim the next work item when the current one starts
                                              // (measured slower: fine384 348 vs 353, 1536^3 376 vs 384 GLUPS)
    // J3D_PERSISTENT: slab dependency tables and completion counters (device.cuh IterCtl)
    int32_t* d_item_slab = nullptr;             // [n_items]
    const unsigned int** d_slab_deps = nullptr;        // [n_slabs][MAX_DEPS] counter pointers (local / peer)
    const unsigned int** d_slab_deps_local = nullptr;  // the same without the peer entries (skip_exchange)
    const unsigned int** d_remote_done = nullptr;      // every peer counter some slab waits for
    int n_remote_done = 0;
    unsigned int* d_done = nullptr;             // [n_slabs], in the arena at off_done
    int n_slabs = 0, persist_nzc = 0, persist_nty = 0;
    uint32_t slab_target = 0;                   // consumer warps x tiles per slab
    uint32_t persist_base = 0;                  // iterations counted in d_done (mod 2^32)
    int persist_n = 0;                          // set while launching a persistent stencil
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
    // x ghost array `side` (0: -x, 1: +x) of a block buffer; element (y, z) at
    // [(z+1)*xg_pitch + y], z in [-1, nz] (device.cuh layout)
    double* xghost(double* b, int side) const { return (double*)((char*)b + grid_bytes + side * xg_bytes); }
    // owned (ghost=false) or ghost layer of a block buffer on face f as a FaceRef over (a,b)
    FaceRef layer(double* b, int f, bool ghost) const {
        const int a = f >> 1;
        const int64_t n = a == 0 ? nx : a == 1 ? ny : nz;
        const int64_t c = (f & 1) ? (ghost ? n : n - 1) : (ghost ? -1 : 0);
        double* o = b + zs + pitch + XOFF;  // owned (0,0,0)
        if (a == 0 && ghost) return FaceRef{xghost(b, f & 1) + xg_pitch, 1, xg_pitch};
        if (a == 0) return FaceRef{o + c, pitch, zs};
        if (a == 1) return FaceRef{o + c * pitch, 1, zs};
        return FaceRef{o + c * zs, 1, pitch};
    }
    FaceRef contiguous(double* p, int f) const { return FaceRef{p, 1, face_na(f)}; }
};

namespace j3d {

inline bool unfused_family(const jacobi3d* c) { return c->cfg.variant <= J3D_FUSE_B; }

// setup.cu
void build_layout(jacobi3d* c);
void classify(jacobi3d* c);
FaceRef recv_src(const jacobi3d* c, int l, int f, int par);
FaceRef pack_dst(const jacobi3d* c, int l, int f, int par);
void build_tables(jacobi3d* c);
void build_static_tables(jacobi3d* c);
void build_persist_deps(jacobi3d* c);
struct SlabRef { int32_t rank, local, zc, ty; };  // slab (local block, z chunk, tile row) of a rank
std::vector<std::vector<SlabRef>> slab_dep_refs(const jacobi3d* c, int nzc, int nty);

// launch.cu
cudaEvent_t pool_event(jacobi3d* c);
void count_launch(jacobi3d* c, int l);
void stencil(jacobi3d* c, int begin, int count, int parity, cudaStream_t st, int l);
void copies(jacobi3d* c, CopyDesc* table, int parity, int l, int face, bool fused, cudaStream_t st);
void refresh(jacobi3d* c, int par);
void fork_streams(jacobi3d* c);
void join_streams(jacobi3d* c, int q);
void enqueue_iteration(jacobi3d* c, int p, bool first, bool last);
void capture_graph(jacobi3d* c, int p);
void drop_graphs(jacobi3d* c);
void do_iterate(jacobi3d* c, int64_t n);
void destroy_ctx(jacobi3d* c);
void wait_stream(jacobi3d* c, cudaStream_t st);
void sync_streams(jacobi3d* c);
double timeout_s();

// control.cu
void ctl_setup_own(jacobi3d* c);
void ctl_connect(jacobi3d* c);
void ctl_teardown(jacobi3d* c);
void ctl_barrier(jacobi3d* c);                         // every rank (NCCL all-reduce if a communicator exists)
uint64_t ctl_reduce(jacobi3d* c, uint64_t v, bool max);  // sum / max over ranks of a host value (no communicator)

// exchange.cu
void nccl_exchange(jacobi3d* c, int par, cudaStream_t st);
void p2p_sync(jacobi3d* c, int slot, cudaStream_t st);
void host_setup_own(jacobi3d* c);
void host_connect(jacobi3d* c);
void host_teardown(jacobi3d* c);
void host_exchange(jacobi3d* c, int par, int slot, cudaStream_t st);
void host_sync(jacobi3d* c, int slot, cudaStream_t st);
void cross_gpu_exchange(jacobi3d* c, int par, int slot, cudaStream_t st);

}  // namespace j3d
