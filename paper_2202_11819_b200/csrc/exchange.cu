// exchange.cu -- cross-GPU halo exchange: grouped NCCL send/recv, NVLink P2P epoch flags, host staging through POSIX shared memory.
#include "context.h"

using namespace j3d;

namespace j3d {

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
    // copy tables of the staged exchange [(q*nl + l)*6 + f]: device send buffer ->
    // this rank's segment (D2H), the neighbour's segment -> device receive buffer
    // (H2D), both through the segments' device-mapped addresses
    const int nl = c->n_local;
    std::vector<CopyDesc> out((size_t)2 * nl * 6), in((size_t)2 * nl * 6);
    std::memset(out.data(), 0, out.size() * sizeof(CopyDesc));
    std::memset(in.data(), 0, in.size() * sizeof(CopyDesc));
    for (int q = 0; q < 2; ++q)
        for (int l = 0; l < nl; ++l)
            for (int f = 0; f < 6; ++f) {
                if (c->kind[l][f] != PEER_HOST) continue;
                const size_t i = ((size_t)q * nl + l) * 6 + f;
                const int r = c->plan.blocks[c->plan.blocks[c->gid[l]].nbr[f]].owner;
                out[i].src = c->contiguous(c->face_buf(l, f, q, false), f);
                out[i].dst = c->contiguous((double*)(c->shm_dev[c->rank] + shm_area_offset(c, l, f, q)), f);
                in[i].src = c->contiguous((double*)(c->shm_dev[r] + shm_area_offset(c, c->nbr_local[l][f], f ^ 1, q)), f);
                in[i].dst = c->contiguous(c->face_buf(l, f, q, true), f);
                out[i].na = in[i].na = (int32_t)c->face_na(f);
                out[i].nb = in[i].nb = (int32_t)c->face_nb(f);
            }
    if (!c->d_stage_out) CK(cudaMalloc(&c->d_stage_out, out.size() * sizeof(CopyDesc)));
    if (!c->d_stage_in) CK(cudaMalloc(&c->d_stage_in, in.size() * sizeof(CopyDesc)));
    CK(cudaMemcpy(c->d_stage_out, out.data(), out.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_stage_in, in.data(), in.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
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
// The D2H / H2D moves are copy kernels over the segments' device-mapped
// addresses (zero-copy through pinned host memory; write-through stores,
// cache-volatile loads), not DMA engine copies: the copy engines are shared
// by every stream of a CUDA context, so with ranks that are threads of one
// process a copy waiting for a peer's flag could sit in front of the peer's
// own D2H copy in an engine queue (a deadlock seen on the GPU).
void host_exchange(jacobi3d* c, int par, int slot, cudaStream_t st) {
    if (!c->host_needed) return;
    const int n = c->n_gpus;
    const int64_t mx = std::max(face_cells(c->plan.ext, 0), std::max(face_cells(c->plan.ext, 2), face_cells(c->plan.ext, 4)));
    CK(launch_stage_copy(c->d_stage_out + (int64_t)par * c->n_local * 6, 6, c->n_local, mx, false, st));
    count_launch(c, -1);
    for (int r : c->peer_ranks)
        DK(g_drv.write64((CUstream)st, (CUdeviceptr)((uint64_t*)c->shm_dev[r] + slot * n + c->rank), 1, 0));
    for (int r : c->peer_ranks) {
        CUdeviceptr f = (CUdeviceptr)((uint64_t*)c->shm_dev[c->rank] + slot * n + r);
        DK(g_drv.wait64((CUstream)st, f, 1, CU_STREAM_WAIT_VALUE_EQ));
        DK(g_drv.write64((CUstream)st, f, 0, 0));
    }
    CK(launch_stage_copy(c->d_stage_in + (int64_t)par * c->n_local * 6, 6, c->n_local, mx, true, st));
    count_launch(c, -1);
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
    Nvtx nv("j3d.exchange");
    nccl_exchange(c, par, st);
    p2p_sync(c, slot, st);
    host_exchange(c, par, slot, st);
}


}  // namespace j3d
