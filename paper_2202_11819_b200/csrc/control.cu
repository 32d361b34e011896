// control.cu -- the host control plane of a multi-GPU context: barrier, sum
// and max over all ranks ("Only a max-allreduce for the
// residual, a sum-allreduce for the checksum, and a timing barrier").
//
// With the NCCL exchange backend the context owns a communicator and these
// go through NCCL.  The P2P and host-staging backends move no halo byte
// through NCCL, so they do not create one: the control plane is one POSIX
// shared-memory segment per rank (same node: NVLink peers and host staging
// need that anyway) holding a collective sequence number and two value
// slots.  Collective k: every rank writes its value into slot k&1, publishes
// seq = k (release), and waits until every rank's seq >= k (acquire); then
// it reads every rank's slot k&1.  Two slots suffice: a rank rewrites slot
// k&1 only in collective k+2, which it enters after passing collective k+1,
// which every other rank enters only after it has read slot k&1.  The same
// code serves ranks that are processes and ranks that are threads of one
// process (paper_2202_11819_b200.dist.ThreadGroup), so the multi-rank paths
// can run on one GPU.  Waits are polled with the J3D_TIMEOUT_S watchdog.
#include "context.h"

#include <random>

#include <sys/stat.h>

using namespace j3d;

namespace j3d {

namespace {

struct CtlSeg {
    alignas(64) uint64_t seq;
    alignas(64) uint64_t val[2];
};
constexpr size_t kCtlBytes = 4096;
static_assert(sizeof(CtlSeg) <= kCtlBytes, "control segment");

std::string ctl_name(uint64_t key, int rank) {
    char b[64];
    std::snprintf(b, sizeof b, "/j3d_%016llx_c%d", (unsigned long long)key, rank);
    return b;
}

CtlSeg* seg(jacobi3d* c, int r) { return reinterpret_cast<CtlSeg*>(c->ctl_base[r]); }

char* map_segment(const std::string& nm, bool create) {
    if (create) shm_unlink(nm.c_str());
    int fd = shm_open(nm.c_str(), create ? (O_CREAT | O_RDWR) : O_RDWR, 0600);
    if (fd < 0 && !create) {  // a peer that has not created its segment yet: wait for it
        const double limit = timeout_s();
        const auto t0 = std::chrono::steady_clock::now();
        while (fd < 0 && std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < limit) {
            std::this_thread::sleep_for(std::chrono::milliseconds(1));
            fd = shm_open(nm.c_str(), O_RDWR, 0600);
        }
    }
    if (fd < 0)
        throw Error(create ? J3D_ENOMEM : J3D_ETIMEOUT,
                    "shm_open " + nm + " failed" + (create ? "" : " (ranks must share one node)"));
    if (create && ftruncate(fd, (off_t)kCtlBytes) != 0) {
        close(fd);
        throw Error(J3D_ENOMEM, "ftruncate of the control segment failed");
    }
    if (!create) {  // the creator may not have sized it yet
        const double limit = timeout_s();
        const auto t0 = std::chrono::steady_clock::now();
        struct stat sb;
        while (fstat(fd, &sb) == 0 && sb.st_size < (off_t)kCtlBytes) {
            if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
                close(fd);
                throw Error(J3D_ETIMEOUT, "control segment " + nm + " was never sized");
            }
            std::this_thread::sleep_for(std::chrono::milliseconds(1));
        }
    }
    void* p = mmap(nullptr, kCtlBytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw Error(J3D_ENOMEM, "mmap of a control segment failed");
    return (char*)p;
}

// publish seq = k, then wait until every rank reached k
void arrive_and_wait(jacobi3d* c, uint64_t k) {
    Nvtx nv("j3d.collective");
    __atomic_store_n(&seg(c, c->rank)->seq, k, __ATOMIC_RELEASE);
    const double limit = timeout_s();
    const auto t0 = std::chrono::steady_clock::now();
    int us = 1;
    for (int r = 0; r < c->n_gpus; ++r) {
        while (__atomic_load_n(&seg(c, r)->seq, __ATOMIC_ACQUIRE) < k) {
            const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (el > limit)
                throw Error(J3D_ETIMEOUT, "rank " + std::to_string(r) + " did not reach collective " +
                                              std::to_string(k) + " within " + std::to_string((int)limit) +
                                              " s (a rank stopped, or the ranks called the collective API in "
                                              "different orders)");
            if (us < 64) {
                std::this_thread::yield();
                ++us;
            } else {
                std::this_thread::sleep_for(std::chrono::microseconds(us < 1000 ? (us += 16) : us));
            }
        }
    }
}

}  // namespace

uint64_t process_token() {
    static const uint64_t tok = [] {
        std::random_device rd;
        return ((uint64_t)rd() << 32) ^ (uint64_t)rd() ^ ((uint64_t)getpid() << 17);
    }();
    return tok;
}

void ctl_setup_own(jacobi3d* c) {
    c->ctl_base.assign(c->n_gpus, nullptr);
    char* p = map_segment(ctl_name(c->job_key, c->rank), true);
    std::memset(p, 0, kCtlBytes);
    c->ctl_base[c->rank] = p;
}

void ctl_connect(jacobi3d* c) {
    for (int r = 0; r < c->n_gpus; ++r)
        if (!c->ctl_base[r]) c->ctl_base[r] = map_segment(ctl_name(c->job_key, r), false);
    c->ctl_connected = true;
}

void ctl_teardown(jacobi3d* c) {
    for (size_t r = 0; r < c->ctl_base.size(); ++r) {
        if (!c->ctl_base[r]) continue;
        munmap(c->ctl_base[r], kCtlBytes);
        if ((int)r == c->rank) shm_unlink(ctl_name(c->job_key, c->rank).c_str());
        c->ctl_base[r] = nullptr;
    }
}

void ctl_barrier(jacobi3d* c) {
    if (c->n_gpus == 1) return;
    if (c->comm) {  // NCCL backend: the communicator's all-reduce
        double* s = (double*)(c->arena + c->off_scratch + 64);
        NK(ncclAllReduce(s, s, 1, ncclFloat64, ncclSum, c->comm, c->main));
        wait_stream(c, c->main);
        return;
    }
    if (!c->ctl_connected) throw Error(J3D_ESTATE, "multi-GPU context not connected (jacobi3d_ipc_connect)");
    arrive_and_wait(c, ++c->ctl_seq);
}

uint64_t ctl_reduce(jacobi3d* c, uint64_t v, bool max) {
    if (c->n_gpus == 1) return v;
    if (!c->ctl_connected) throw Error(J3D_ESTATE, "multi-GPU context not connected (jacobi3d_ipc_connect)");
    const uint64_t k = ++c->ctl_seq;
    __atomic_store_n(&seg(c, c->rank)->val[k & 1], v, __ATOMIC_RELAXED);
    arrive_and_wait(c, k);  // release / acquire order the slot writes
    uint64_t out = 0;
    for (int r = 0; r < c->n_gpus; ++r) {
        const uint64_t x = __atomic_load_n(&seg(c, r)->val[k & 1], __ATOMIC_RELAXED);
        out = max ? std::max(out, x) : out + x;  // sum mod 2^64 (the checksum's definition, R15)
    }
    return out;
}

}  // namespace j3d
