// kernels.cu -- sm_100a kernels of the Jacobi3D hot path.
//
//   stencil_tma_kernel  the 7-point Jacobi update (formula
//                       SPEC.md L388, order self,-x,+x,-y,+y,-z,+z, IEEE /7),
//                       optionally with the unpack fused into its prologue and
//                       the pack fused into its epilogue (PAPER.md L515-524,
//                       strategy C) or with the epilogue storing straight into
//                       the neighbour's ghost layer (J3D_FUSE_DIRECT).
//   copy_faces_kernel   pack / unpack of the <=6 halo faces (PAPER.md L81, L98,
//                       L205, L210), unfused (one face per launch) or fused
//                       (one thread per element of the largest face looping
//                       over the six faces, the paper's choice, L519-524).
//   init_kernel, checksum_kernel, residual_kernel: setup and reporting.
//
// Stencil design: HBM-bound (16 B per lattice-site
// update, 0.44 flop/B), so no tensor cores.  A persistent grid of CTAs walks
// a list of work items (block, xy tile, z range) -- for J3D_PERSISTENT, n
// iterations of that list, with per-slab completion counters ordering the
// iterations.  Per CTA one producer warp streams (TX+8) x (TY+2) xy-planes of
// the input buffer -- the tile plus its 1-cell halo, y/z ghost rows included,
// x ghost values from the separate x ghost arrays for tiles at a block x
// edge -- into an NSTAGE-deep shared-memory ring with TMA
// (cp.async.bulk.tensor.3d, mbarrier complete_tx).  NCW consumer warps march
// up z holding the stages of planes z-1, z, z+1, read all seven inputs of a
// cell from shared memory and write the new plane to HBM (16-byte vector
// stores for the cell-pair lane map).  Every input plane is fetched once per
// tile (plus the halo, which neighbouring tiles fetch concurrently and
// therefore mostly hit in L2), every output cell written once: the
// compulsory 16 B/LUP.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <type_traits>

#include "device.cuh"
#include "kernels.h"

namespace j3d {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait suspends the waiting warp (up to the hint) instead of spinning, so
// waiting warps do not take issue slots from the ones computing (a spinning
// wait loop was 18 % of all warp instructions on 96^3 blocks, ncu)
#ifndef J3D_SUSPEND_NS
#define J3D_SUSPEND_NS 1000000
#endif
constexpr uint32_t kSuspendNs = J3D_SUSPEND_NS;
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(kSuspendNs)
        : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const unsigned int* p, bool sys) {
    uint32_t v;
    if (sys) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Persistent launches: wait until the slabs item `it` depends on have
// finished `iters` iterations (IterCtl, device.cuh), then order the async
// proxy (TMA) after the acquired generic-proxy writes.  A wait beyond the
// context's limit (J3D_TIMEOUT_S) means a peer stopped or a bug: trap rather
// than hang the GPU.
__device__ __forceinline__ void wait_counter(const unsigned int* p, uint32_t need, bool sys, uint64_t limit_ns) {
    if ((int32_t)(ld_acquire_u32(p, sys) - need) >= 0) return;
    const uint64_t t0 = global_ns();
    while ((int32_t)(ld_acquire_u32(p, sys) - need) < 0) {
        __nanosleep(128);
        if (global_ns() - t0 > limit_ns) __trap();
    }
}

// Called by the whole producer warp: lane j polls the item's j-th dependency
// (one round trip for all of them instead of up to MAX_DEPS in sequence).
// The warp barrier orders every lane's acquire before lane 0's later
// operations (barriers are part of the causality order); lane 0 -- which
// issues the TMA loads -- then orders the async proxy after the generic-proxy
// writes those acquires observed.  (An extra fence at the acquires' scope,
// `fence` = 1: J3D_DEPFENCE, measured for the record in
// profiles/r02_tuning_log.md.)
__device__ __noinline__ void wait_slabs(const IterCtl ctl, int it, uint32_t iters, int lane, bool fence) {
    const uint32_t need = iters * ctl.target;
    const unsigned int* const* dp = ctl.slab_deps + (int64_t)(ctl.item_slab[it] & SLAB_MASK) * MAX_DEPS;
    const uintptr_t p = lane < MAX_DEPS ? reinterpret_cast<uintptr_t>(dp[lane]) : 0;
    // bit 0 tags a peer GPU's counter: acquire at system scope
    if (p) wait_counter(reinterpret_cast<const unsigned int*>(p & ~uintptr_t(1)), need, (p & 1) != 0, ctl.timeout_ns);
    __syncwarp();
    if (lane == 0) {
        if (fence) {
            if (ctl.sys) __threadfence_system();
            else __threadfence();
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
}

__device__ __forceinline__ void tmap_acquire(const CUtensorMap* m) {
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(m))
                 : "memory");
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                                                 uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// Descriptor loads on rare paths: volatile so the compiler cannot hoist
// them out of the plane loop (which would pin ~36 registers for the six
// FaceRefs in the hot loop).
__device__ __forceinline__ FaceRef load_face(const FaceRef* f) {
    FaceRef r;
    uint64_t p;
    asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(p) : "l"(f));
    asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(r.sa) : "l"(reinterpret_cast<const char*>(f) + 8));
    asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(r.sb) : "l"(reinterpret_cast<const char*>(f) + 16));
    r.p = reinterpret_cast<double*>(p);
    return r;
}

__device__ __forceinline__ void st_global_v2(double* p, double a, double b) {
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// Correctly rounded s / 7 (IEEE round-to-nearest-even) without the generic
// division routine (whose slow path is a CALL that costs the stencil ~20
// registers).  Normal results: q = RN(s*y) with y = RN(1/7) is a faithful
// quotient (7y = 1 - 2^-54 exactly, so s*y lies within half an ulp of s/7);
// the remainder e = s - 7q is then exact in one FMA and RN(q + e*y) =
// RN(s/7) (Markstein's correction theorem); for exact quotients e == 0 and
// the result is q.  Subnormal results and zeros (|s| < 7*2^-1022): s is an
// integer N times 2^-1074 with |N| < 2^55, and RN(s/7) = 2^-1074 * (N/7
// rounded to nearest -- 7 is odd, so there are no ties), done in integer
// arithmetic, with the sign of s (so -0/7 = -0).  Non-finite s: the fast
// path gives NaN for s = +-inf (e = inf - inf), so the exact routine returns
// s * y there (+-inf / 7 = +-inf; NaN stays NaN).  DESIGN.md "Division";
// checked against __ddiv_rn on the GPU by jacobi3d_div7_selftest.
constexpr double kDiv7Tiny = 0x1.cp-1020;  // 7 * 2^-1022: below it s/7 is subnormal (or s is 0)
constexpr double kDiv7Min = 0x1p-1022;     // smallest normal double

// Fast path, valid for finite |s| >= kDiv7Tiny: three fp64 ops, no branch.
__device__ __forceinline__ double div7_fast(double s) {
    const double y = 0x1.2492492492492p-3;  // RN(1/7)
    const double q = __dmul_rn(s, y);
    const double e = __fma_rn(-q, 7.0, s);
    return __fma_rn(e, y, q);  // exact quotients: e == 0 and the result is q
}

// The stencil's decision: a fast-path result r = div7_fast(s) is kept unless
// it is zero, subnormal or NaN (one DSETP: !(|r| >= 2^-1022), unordered
// compare).  Every s outside that set is finite with |s| >= kDiv7Tiny, where
// the fast path is exact; the set contains every s the fast path can get
// wrong (+-0 -- it returns +0 for -0 --, the subnormal quotients, +-inf and
// NaN).  Flagged planes go through div7() below.
__device__ __forceinline__ bool div7_rare(double r) { return !(fabs(r) >= kDiv7Min); }

// All s (the stencil calls it only on the rare path, see stencil_tma_kernel).
__device__ __forceinline__ double div7(double s) {
    double r = div7_fast(s);
    if (fabs(s) < kDiv7Tiny) {  // |s/7| < 2^-1022: subnormal quotient (or zero)
        const long long n = __double2ll_rn(__dmul_rn(__dmul_rn(s, 0x1p537), 0x1p537));  // exact
        const long long a = n < 0 ? -n : n;
        long long k = a / 7;
        if (a - 7 * k >= 4) k += 1;
        r = copysign(__dmul_rn((double)k, 0x1p-1074), s);  // sign kept for zero results too
    } else if (!(fabs(s) <= 0x1.fffffffffffffp+1023)) {  // +-inf (an overflowed sum) or NaN
        r = __dmul_rn(s, 0x1.2492492492492p-3);          // +-inf * y = +-inf; NaN -> NaN
    }
    return r;
}

// The update's sum: SPEC.md L388, left to right (no reassociation, no FMA).
__device__ __forceinline__ double sum7(double c, double xm, double xp, double ym, double yp, double zm, double zp) {
    double s = __dadd_rn(c, xm);
    s = __dadd_rn(s, xp);
    s = __dadd_rn(s, ym);
    s = __dadd_rn(s, yp);
    s = __dadd_rn(s, zm);
    return __dadd_rn(s, zp);
}

// ------------------------------------------------------------------ stencil
// Tile shape: TX cells along x (a warp covers 64 with double2 per lane, CPL
// column groups), NCW consumer warps each owning RPW rows (TY = NCW*RPW),
// NSTAGE plane buffers in the TMA ring, MINB CTAs per SM targeted.
template <int TX_, int NCW_, int RPW_, int NSTAGE_, int MINB_, int MAP_ = 0, bool YSREQ_ = false>
struct Tile {
    static constexpr int TX = TX_, NCW = NCW_, RPW = RPW_, NSTAGE = NSTAGE_, MINB = MINB_;
    // MAP 0: a lane owns cell pairs (x, x+1), x = x0 + 64c + 2*lane (16-byte accesses);
    // MAP 1: a lane owns single cells x = x0 + 32k + lane (any TX multiple of 32,
    //        e.g. a 96-wide block in one tile)
    static constexpr int MAP = MAP_;
    static constexpr int TY = NCW * RPW;
    static constexpr int CPL = TX / 64;
    static constexpr int KPL = TX / 32;
    static constexpr int HX = 4;      // halo columns kept left of the tile in smem
    static constexpr int W = TX + 2 * HX;  // smem row: x0-4 .. x0+TX+3: the same 32-B sectors as x0-1 .. x0+TX,
                                           // 16-B aligned interior, rows a multiple of 64 B
    static constexpr int H = TY + 2;  // y0-1 .. y0+TY
    static constexpr uint32_t TX_BYTES = W * H * 8;
    // x ghost vectors of the tile's rows after the box: -x at SIDE_OFF, +x at
    // SIDE_OFF + SIDE_STRIDE (TMA destinations are 128-byte aligned)
    static constexpr int SIDE_OFF = (W * H * 8 + 127) / 128 * 128;
    static constexpr int SIDE_STRIDE = (TY * 8 + 127) / 128 * 128;
    // strategy C's y ghost rows, loaded from the receive buffers (-y at YSIDE_OFF,
    // +y at YSIDE_OFF + YSIDE_STRIDE) and copied into the tile's ghost row by the
    // warp that reads it
    static constexpr int YSIDE_OFF = SIDE_OFF + 2 * SIDE_STRIDE;
    static constexpr int YSIDE_STRIDE = (W * 8 + 127) / 128 * 128;
    static constexpr int BAR_BYTES = 2 * NSTAGE * 8 + 2 * 4 * 8 + 4 * 4 + 128;
    // the y side rows only where they keep MINB CTAs per SM (228 KB per SM, 1 KB
    // reserved per CTA); otherwise strategy C patches y ghost rows generically.
    // only in the instances strategy C launches (J3D_TILES_YS): the extra shared memory
    // per stage costs the other variants up to 6 % (small192: 330 vs 350 GLUPS)
    static constexpr bool YS =
        YSREQ_ && MINB * (NSTAGE * (YSIDE_OFF + 2 * YSIDE_STRIDE) + BAR_BYTES + 1024) <= 233472;
    static constexpr int STAGE_BYTES = YS ? YSIDE_OFF + 2 * YSIDE_STRIDE : YSIDE_OFF;
    static constexpr int SMEM_BYTES = NSTAGE * STAGE_BYTES + BAR_BYTES;
    static constexpr int THREADS = 32 * (NCW + 1);
    // the consumers hold the stages of planes z-1, z, z+1; at least one more is in flight
    static_assert((MAP == 1 ? TX % 32 : TX % 64) == 0 && W <= 256 && H <= 256 && NSTAGE >= 4, "tile shape");
};

// Rare path (strategy C prologue, "unpack fused into the update"): overwrite
// the ghost cells of one freshly landed plane stage with the receive-buffer
// values, restricted to the cells THIS warp will read (its rows' centres for
// a ghost plane; the -y / +y ghost row next to its rows; its rows' -x / +x
// ghost columns), so only a __syncwarp is needed afterwards.
template <class T>
__device__ __forceinline__ void patch_stage(const StencilDesc* __restrict__ d, double* st, int zz, int x0, int y0,
                                         int warp, int lane) {
    constexpr int W = T::W;
    const int nx = d->nx, ny = d->ny, nz = d->nz;
    const uint32_t pro = d->pro_mask;
    const int r0 = warp * T::RPW;
    if (zz < 0 || zz >= nz) {
        const int f = zz < 0 ? 4 : 5;
        if (!(pro & (1u << f))) return;
        const FaceRef F = d->pro[f];
        for (int r = 0; r < T::RPW; ++r) {
            const int y = y0 + r0 + r;
            if (y >= ny) break;
            for (int lx = lane; lx < T::TX; lx += 32) {
                const int x = x0 + lx;
                if (x < nx) st[(r0 + r + 1) * W + lx + T::HX] = F.p[x * F.sa + y * F.sb];
            }
        }
        return;
    }
    if ((pro & 4u) && y0 == 0 && warp == 0) {
        const FaceRef F = load_face(&d->pro[2]);
        for (int lx = lane; lx < T::TX; lx += 32) {
            const int x = x0 + lx;
            if (x < nx) st[lx + T::HX] = F.p[x * F.sa + zz * F.sb];
        }
    }
    if (pro & 8u) {
        const int gl = ny - y0;  // tile-local row of the +y ghost
        if (gl <= T::TY && gl - 1 >= r0 && gl - 1 < r0 + T::RPW) {
            const FaceRef F = load_face(&d->pro[3]);
            for (int lx = lane; lx < T::TX; lx += 32) {
                const int x = x0 + lx;
                if (x < nx) st[(gl + 1) * W + lx + T::HX] = F.p[x * F.sa + zz * F.sb];
            }
        }
    }
    if (lane < T::RPW) {
        const int y = y0 + r0 + lane;
        if (y < ny) {
            // the -x / +x ghost of the row: its halo column (cell-pair map) or its
            // entry of the stage's x ghost vector (one-cell map reads it there)
            if ((pro & 1u) && x0 == 0) {
                const FaceRef F = load_face(&d->pro[0]);
                const int i = T::MAP == 1 ? T::SIDE_OFF / 8 + r0 + lane : (r0 + lane + 1) * W + T::HX - 1;
                st[i] = F.p[y * F.sa + zz * F.sb];
            }
            if (pro & 2u) {
                const int gx = nx - x0;  // tile-local x of the +x ghost
                if (gx <= T::TX) {
                    const FaceRef F = load_face(&d->pro[1]);
                    const int i = T::MAP == 1 ? (T::SIDE_OFF + T::SIDE_STRIDE) / 8 + r0 + lane
                                              : (r0 + lane + 1) * W + gx + T::HX;
                    st[i] = F.p[y * F.sa + zz * F.sb];
                }
            }
        }
    }
}

// Rare path (strategy C / direct epilogue, "pack fused into the update"):
// store the new values of a boundary cell pair to the face destinations.
__device__ __forceinline__ void epi_store(const StencilDesc* __restrict__ d, uint32_t epi, int x, int y, int z,
                                          double vx, double vy, bool has2) {
    const int nx = d->nx, ny = d->ny, nz = d->nz;
    if ((epi & 1u) && x == 0) { const FaceRef f = load_face(&d->epi[0]); f.p[y * f.sa + z * f.sb] = vx; }
    if (epi & 2u) {
        const FaceRef f = load_face(&d->epi[1]);
        if (x == nx - 1) f.p[y * f.sa + z * f.sb] = vx;
        else if (has2 && x + 1 == nx - 1) f.p[y * f.sa + z * f.sb] = vy;
    }
    if ((epi & 4u) && y == 0) {
        const FaceRef f = load_face(&d->epi[2]);
        f.p[x * f.sa + z * f.sb] = vx;
        if (has2) f.p[(x + 1) * f.sa + z * f.sb] = vy;
    }
    if ((epi & 8u) && y == ny - 1) {
        const FaceRef f = load_face(&d->epi[3]);
        f.p[x * f.sa + z * f.sb] = vx;
        if (has2) f.p[(x + 1) * f.sa + z * f.sb] = vy;
    }
    if ((epi & 16u) && z == 0) {
        const FaceRef f = load_face(&d->epi[4]);
        f.p[x * f.sa + y * f.sb] = vx;
        if (has2) f.p[(x + 1) * f.sa + y * f.sb] = vy;
    }
    if ((epi & 32u) && z == nz - 1) {
        const FaceRef f = load_face(&d->epi[5]);
        f.p[x * f.sa + y * f.sb] = vx;
        if (has2) f.p[(x + 1) * f.sa + y * f.sb] = vy;
    }
}

// Work distribution: the producer of each CTA takes items in list order from
// a global counter (sched[0]), so the items of one z chunk -- in particular
// y- and x-neighbouring tiles, whose halos overlap -- run at the same time
// and the overlapping halo rows/columns are served from L2.  A 4-deep item
// queue in shared memory hands the indices to the consumer warps.  The last
// CTA to finish resets the counter (sched[1] counts finished CTAs), so the
// kernel is reusable and graph-capturable without a memset.
template <class T>
__global__ void __launch_bounds__(T::THREADS, T::MINB)
    stencil_tma_kernel(const StencilDesc* __restrict__ descs, const CUtensorMap* __restrict__ tmaps,
                       const CUtensorMap* __restrict__ tmapsp, const CUtensorMap* __restrict__ tmapsx,
                       const WorkItem* __restrict__ items, int n_items, int parity, int flags,
                       unsigned int* __restrict__ sched, const IterCtl ctl) {
    constexpr int NCW = T::NCW, RPW = T::RPW, CPL = T::CPL, W = T::W, NSTAGE = T::NSTAGE, IQ = 4;
    // The kernel has no static shared memory, so the dynamic window starts at
    // shared offset 0 (1024-B aligned); indexing the __shared__ array directly
    // keeps the state space known to the compiler (LDS, not generic LD).
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * T::STAGE_BYTES);
    uint64_t* empty = full + NSTAGE;
    uint64_t* qfull = empty + NSTAGE;
    uint64_t* qempty = qfull + IQ;
    volatile int* queue = reinterpret_cast<volatile int*>(qempty + IQ);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool faces = flags & 1;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NCW);
        }
        for (int i = 0; i < IQ; ++i) {
            mbar_init(&qfull[i], 1);
            mbar_init(&qempty[i], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NCW) {  // ---------------- producer warp: item scheduling + TMA plane loads
        int s = 0, qs = 0;
        uint32_t ph = 0, qph = 0;
        const int tma_mode = (flags >> 2) & 3;
        const bool prefetch = !(flags & 16);  // claim the next item when this one starts (J3D_PREFETCH)
        const int total = n_items * ctl.n_iter;
        // lane 0 claims items and issues every TMA load; the whole warp polls the
        // persistent launch's dependency counters.  The next item is claimed when
        // the current one starts, so the claim's round trip overlaps its planes.
        int g = 0;
        if (lane == 0) g = (int)atomicAdd(&sched[0], 1u);
        g = __shfl_sync(0xffffffffu, g, 0);
        for (;;) {
            if (g >= total) g = -1;
            int gn = 0;
            if (lane == 0) {
                if (prefetch && g >= 0) gn = (int)atomicAdd(&sched[0], 1u);
                mbar_wait(&qempty[qs], qph ^ 1);
                queue[qs] = g;
                mbar_arrive(&qfull[qs]);
            }
            if (++qs == IQ) { qs = 0; qph ^= 1; }
            if (g < 0) break;
            const int k = g / n_items, it = g - k * n_items;
            // iteration 0 of a call waits only for peers (this GPU's previous
            // launch is complete in stream order)
            if (ctl.done && (k > 0 || ctl.sys)) wait_slabs(ctl, it, ctl.base + (uint32_t)k, lane, (flags & 32) != 0);
            if (lane == 0) {
                uint64_t pol_first = 0, pol_last = 0;
                if (tma_mode) {
                    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
                    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
                }
                const WorkItem w = items[it];
                const int bp = 2 * w.blk + (parity ^ (k & 1));
                const CUtensorMap* tm = tmaps + bp;
                const CUtensorMap* tx = tmapsx + bp;
                tmap_acquire(tm);
                tmap_acquire(tx);
                const int nxb = descs[bp].nx, nyb = descs[bp].ny, nzb = descs[bp].nz;
                // strategy C: ghost values the prologue takes from the receive buffers,
                // loaded here with TMA ("unpack ... in one kernel"): the
                // x ghost vectors, the y ghost rows (into the stage's y side rows) and
                // whole ghost planes, from maps over the receive buffers (setup.cu)
                const uint32_t ptma = (flags & 1) ? descs[bp].pro_tma : 0u;
                const CUtensorMap* pm = tmapsp + 6 * bp;
                // tiles at a block x edge also load the x ghost vectors of their rows
                const uint32_t xe = (w.tx == 0 ? 1u : 0u) | ((w.tx + 1) * T::TX >= nxb ? 2u : 0u);
                const uint32_t ye = (ptma & 4u) && w.ty == 0 ? 1u : 0u;
                const uint32_t ye2 = (ptma & 8u) && (w.ty + 1) * T::TY >= nyb ? 1u : 0u;
                const uint32_t bytes = T::TX_BYTES + (uint32_t)__popc(xe) * (T::TY * 8) + (ye + ye2) * (T::W * 8);
                const int c0 = w.tx * T::TX - T::HX, c1 = w.ty * T::TY;
                if (ptma) {
                    for (int f = 0; f < 6; ++f)
                        if (ptma & (1u << f)) tmap_acquire(pm + f);
                }
                for (int z = w.z0 - 1; z <= w.z1; ++z) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_expect_tx(&full[s], bytes);
                    unsigned char* dst = smem + s * T::STAGE_BYTES;
                    // receive buffers: x faces (y, z), y faces (x, z), z faces (x, y), owned
                    // coordinates only (ghost-plane / corner coordinates are zero-filled, unused)
                    if (xe & 1u) {
                        if (ptma & 1u) tma_load_2d(dst + T::SIDE_OFF, pm + 0, &full[s], c1, z);
                        else tma_load_3d(dst + T::SIDE_OFF, tx, &full[s], c1, z + 1, 0);
                    }
                    if (xe & 2u) {
                        if (ptma & 2u) tma_load_2d(dst + T::SIDE_OFF + T::SIDE_STRIDE, pm + 1, &full[s], c1, z);
                        else tma_load_3d(dst + T::SIDE_OFF + T::SIDE_STRIDE, tx, &full[s], c1, z + 1, 1);
                    }
                    if constexpr (T::YS) {
                        if (ye) tma_load_2d(dst + T::YSIDE_OFF, pm + 2, &full[s], c0, z);
                        if (ye2) tma_load_2d(dst + T::YSIDE_OFF + T::YSIDE_STRIDE, pm + 3, &full[s], c0, z);
                    }
                    const int zf = z < 0 ? 4 : z >= nzb ? 5 : -1;
                    if (zf >= 0 && (ptma & (1u << zf))) {
                        tma_load_2d(dst, pm + zf, &full[s], c0, c1 - 1);  // the ghost plane: neighbour's face
                    } else if (tma_mode == 0) {
                        tma_load_3d(dst, tm, &full[s], c0, c1, z + 1);
                    } else {
                        tma_load_3d_hint(dst, tm, &full[s], c0, c1, z + 1, tma_mode == 1 ? pol_first : pol_last);
                    }
                    if (++s == NSTAGE) { s = 0; ph ^= 1; }
                }
                if (!prefetch) gn = (int)atomicAdd(&sched[0], 1u);
            }
            g = __shfl_sync(0xffffffffu, gn, 0);
        }
        if (lane == 0) {
            __threadfence();
            if (atomicAdd(&sched[1], 1u) == gridDim.x - 1) {  // every CTA has taken its last item
                sched[0] = 0;
                sched[1] = 0;
                __threadfence();
            }
        }
        return;
    }

    // ---------------- consumer warps
    int s = 0, qs = 0;
    uint32_t ph = 0, qph = 0;
    auto stage = [&](int i) -> double* { return reinterpret_cast<double*>(smem + i * T::STAGE_BYTES); };
    auto advance = [&]() { if (++s == NSTAGE) { s = 0; ph ^= 1; } };

    for (;;) {
        mbar_wait(&qfull[qs], qph);
        const int g = queue[qs];
        __syncwarp();
        if (lane == 0) mbar_arrive(&qempty[qs]);
        if (++qs == IQ) { qs = 0; qph ^= 1; }
        if (g < 0) break;
        const int kit = g / n_items, it = g - kit * n_items;

        const WorkItem w = items[it];
        const StencilDesc* d = descs + (2 * w.blk + (parity ^ (kit & 1)));
        const int nx = d->nx, ny = d->ny, nz = d->nz;
        const int64_t pitch = d->pitch, zs = d->zs;
        const int x0 = w.tx * T::TX, y0 = w.ty * T::TY;
        const int xl = x0 + (T::MAP == 1 ? lane : 2 * lane), yl = y0 + warp * RPW;  // this thread's first cell
        double* obase = d->out + (int64_t)(yl + 1) * pitch + XOFF + xl;
        const uint32_t pro = faces ? d->pro_mask : 0u;   // ghost faces patched with generic loads (fallback)
        const uint32_t ptma = faces ? d->pro_tma : 0u;   // ghost faces the producer loaded from receive buffers
        const uint32_t epi = faces ? d->epi_mask : 0u;
        // block faces (bits 0..3 = -x,+x,-y,+y) this tile's cells touch
        const uint32_t touch = (x0 == 0 ? 1u : 0u) | (x0 + T::TX >= nx ? 2u : 0u) | (y0 == 0 ? 4u : 0u) |
                               (y0 + T::TY >= ny ? 8u : 0u);
        const bool whole = x0 + T::TX <= nx && y0 + T::TY <= ny;  // no cell of the tile is outside the block
        const bool fullw = T::MAP == 1 && whole && x0 == 0 && nx == T::TX;  // compute_plane_s FULL
        // x-face destinations of this tile: wide tiles load them once per item
        // (registers are plentiful there), narrow 2-CTA/SM tiles per plane
        constexpr bool HOISTX = T::TX >= 128;
        FaceRef fxm{nullptr, 0, 0}, fxp{nullptr, 0, 0};
        if (HOISTX && (epi & touch & 1u)) fxm = load_face(&d->epi[0]);
        if (HOISTX && (epi & touch & 2u)) fxp = load_face(&d->epi[1]);
        auto face_x = [&](int f) -> FaceRef {
            if constexpr (HOISTX) return f == 0 ? fxm : fxp;
            else return load_face(&d->epi[f]);
        };
        // one-cell map with 4+ rows per warp (register room): the x-face stores'
        // destinations once per item in compact form -- this warp's first row at
        // z = 0 and the plane stride (x faces are contiguous in y: sa == 1,
        // setup.cu checks) -- instead of three descriptor loads per plane
        constexpr bool HOISTX1 = T::MAP == 1 && RPW >= 4;
        double* xq0 = nullptr;
        double* xq1 = nullptr;
        int32_t xsb0 = 0, xsb1 = 0;
        if (HOISTX1 && (epi & touch & 1u)) {
            const FaceRef F = load_face(&d->epi[0]);
            xq0 = F.p + yl;
            xsb0 = (int32_t)F.sb;
        }
        if (HOISTX1 && (epi & touch & 2u)) {
            const FaceRef F = load_face(&d->epi[1]);
            xq1 = F.p + yl;
            xsb1 = (int32_t)F.sb;
        }
        const int sbase = (warp * RPW + 1) * W + (T::MAP == 1 ? lane : 2 * lane) + T::HX;  // smem offset of the first cell

        // wait for the stage of plane zz, patch its ghosts (fused prologue) if needed
        // block x edge: per plane, lane r < RPW copies its row's ghost values from
        // the stage's x ghost vectors into the row's halo column (offsets in
        // doubles from the stage base, fixed for the item)
        const int er = warp * RPW + lane;
        const int edl = (er + 1) * W + T::HX - 1, esl = T::SIDE_OFF / 8 + er;
        const int edr = (er + 1) * W + T::HX + (nx - x0), esr = (T::SIDE_OFF + T::SIDE_STRIDE) / 8 + er;
        const bool ecopy = (touch & 3u) && lane < RPW;
        // MAP 1 reads the x ghost vectors in place instead (xlb / xrb: offsets of
        // this thread's row-0 vector entries from its edge cell; see compute_plane_s)
        const int xlast_t = nx - 1 - x0, kedge = xlast_t >> 5;
        const bool xlf = (touch & 1u) && lane == 0;
        const bool xrf = (touch & 2u) && lane == (xlast_t & 31);
        const int xlb = T::SIDE_OFF / 8 + warp * RPW - sbase;
        const int xrb = (T::SIDE_OFF + T::SIDE_STRIDE) / 8 + warp * RPW - sbase - 32 * kedge;
        // strategy C, y ghost rows from the receive buffers (TMA-fed): the warp
        // reading the tile's -y ghost row (warp 0, tile row 0) / +y ghost row (the
        // warp owning the block's last row) copies the stage's y side row into it
        const int gly = ny - y0;  // tile-local row of the +y ghost
        const bool ycopy_lo = (ptma & 4u) && y0 == 0 && warp == 0;
        const bool ycopy_hi = (ptma & 8u) && gly <= T::TY && gly - 1 >= warp * RPW && gly - 1 < warp * RPW + RPW;
        auto acquire = [&](int zz) {
            mbar_wait(&full[s], ph);
            if (T::MAP == 0 && (touch & 3u)) {
                if (ecopy) {
                    double* st = stage(s);
                    if (touch & 1u) st[edl] = st[esl];
                    if (touch & 2u) st[edr] = st[esr];
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                __syncwarp();
            }
            if (T::YS && (ycopy_lo | ycopy_hi)) {
                double* st = stage(s);
                for (int i = lane; i < T::TX; i += 32) {
                    if (ycopy_lo) st[T::HX + i] = st[T::YSIDE_OFF / 8 + T::HX + i];
                    if (ycopy_hi) st[(gly + 1) * W + T::HX + i] = st[(T::YSIDE_OFF + T::YSIDE_STRIDE) / 8 + T::HX + i];
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
            }
            if ((pro & touch) || (zz < 0 && (pro & 16u)) || (zz >= nz && (pro & 32u))) {
                patch_stage<T>(d, stage(s), zz, x0, y0, warp, lane);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
            }
        };

        // One output plane z from the stages of planes z-1 (pm), z (pc), z+1
        // (pp), all at this thread's offset.  MODE 0: no face work; 1: x faces
        // only (the boundary values are captured in the hot loop and stored by
        // the owning lane afterwards); 2: any faces, stored inline (fused
        // epilogue, "pack fused into the update").  WHOLE: every cell of the
        // tile is inside the block (no store predicates).  The hot loop has no
        // branch; a quotient that is zero, subnormal or NaN (div7_rare: zero,
        // tiny or non-finite sums) flags the plane for a rare exact pass
        // (recompute from the same inputs, store again).
        auto compute_plane = [&](auto mode_tag, auto whole_tag, int z, uint32_t fm, const double* pm,
                                 const double* pc, const double* pp) {
            constexpr int MODE = decltype(mode_tag)::value;
            constexpr bool WHOLE = decltype(whole_tag)::value;
            constexpr bool FACES = MODE == 2;
            double* op = obase + (int64_t)(z + 1) * zs;
            double cap0[RPW], cap1[RPW];  // MODE 1: new values of the x = 0 / x = nx-1 cells of each row
            const int xlast = nx - 1 - x0;  // tile-local x of the last cell
            const int clast = xlast >> 6, lane_last = (xlast & 63) >> 1;
            const bool last_is_x = !(xlast & 1);
            double* zdst = nullptr;
            int64_t zsb = 0;
            double* ymd = nullptr;
            double* ypd = nullptr;
            double* xmd = nullptr;
            double* xpd = nullptr;
            int64_t xmsa = 0, xpsa = 0;
            uint32_t rare_faces = 0;
            if constexpr (FACES) {
                if (fm & 1u) {
                    const FaceRef F = face_x(0);
                    xmd = F.p + (int64_t)z * F.sb;
                    xmsa = F.sa;
                }
                if (fm & 2u) {
                    const FaceRef F = face_x(1);
                    xpd = F.p + (int64_t)z * F.sb;
                    xpsa = F.sa;
                }
                if ((fm & 48u) == 48u) {
                    rare_faces |= 48u;  // nz == 1: two z faces per cell
                } else if (fm & 48u) {
                    const FaceRef F = load_face(&d->epi[(fm & 16u) ? 4 : 5]);
                    zdst = F.p;
                    zsb = F.sb;
                }
                if (fm & 4u) {
                    const FaceRef F = load_face(&d->epi[2]);
                    ymd = F.p + (int64_t)z * F.sb;
                }
                if (fm & 8u) {
                    const FaceRef F = load_face(&d->epi[3]);
                    ypd = F.p + (int64_t)z * F.sb;
                }
            }
            bool rare = false;
#pragma unroll
            for (int r = 0; r < RPW; ++r) {
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int off = r * W + 64 * c;
                    const double* p = pc + off;
                    const double2 cc = *reinterpret_cast<const double2*>(p);
                    const double2 ym = *reinterpret_cast<const double2*>(p - W);
                    const double2 yp = *reinterpret_cast<const double2*>(p + W);
                    const double2 zm = *reinterpret_cast<const double2*>(pm + off);
                    const double2 zp = *reinterpret_cast<const double2*>(pp + off);
                    const double s0 = sum7(cc.x, p[-1], cc.y, ym.x, yp.x, zm.x, zp.x);
                    const double s1 = sum7(cc.y, cc.x, p[2], ym.y, yp.y, zm.y, zp.y);
                    const double vx = div7_fast(s0), vy = div7_fast(s1);
                    rare |= div7_rare(vx) | div7_rare(vy);
                    if constexpr (MODE == 1) {
                        if (c == 0) cap0[r] = vx;
                        if (c == clast) cap1[r] = last_is_x ? vx : vy;
                    }
                    double* o = op + r * pitch + 64 * c;
                    const int x = xl + 64 * c, y = yl + r;
                    bool v1 = true, v0 = true;
                    if constexpr (!WHOLE) {
                        v1 = y < ny && x + 1 < nx;
                        v0 = y < ny && x < nx;
                    }
                    if (v1) st_global_v2(o, vx, vy);
                    else if (v0) o[0] = vx;
                    if constexpr (FACES) {
                        if (xmd && x == 0 && v0) {
                            // my -x face feeds the neighbour's +x ghost
                            xmd[y * xmsa] = vx;
                        }
                        if (xpd && v0) {
                            const bool hit0 = x == nx - 1, hit1 = x + 1 == nx - 1;
                            if (hit0 || hit1) {
                                const double v = hit0 ? vx : vy;
                                xpd[y * xpsa] = v;
                            }
                        }
                        if (fm & ~3u) {
                            double* fd[3] = {zdst ? zdst + x + (int64_t)y * zsb : nullptr,
                                             (ymd && y == 0) ? ymd + x : nullptr,
                                             (ypd && y == ny - 1) ? ypd + x : nullptr};
#pragma unroll
                            for (int k = 0; k < 3; ++k) {
                                double* q = fd[k];
                                if (!q) continue;
                                if (v1 && !(reinterpret_cast<uintptr_t>(q) & 15)) {
                                    st_global_v2(q, vx, vy);
                                } else {
                                    if (v0) q[0] = vx;
                                    if (v1) q[1] = vy;
                                }
                            }
                        }
                    }
                }
            }
            if constexpr (MODE == 1) {
                if ((fm & 1u) && x0 == 0 && lane == 0) {
                    const FaceRef F = face_x(0);
                    double* q = F.p + (int64_t)z * F.sb;
#pragma unroll
                    for (int r = 0; r < RPW; ++r)
                        if (WHOLE || yl + r < ny) {
                            q[(int64_t)(yl + r) * F.sa] = cap0[r];
                        }
                }
                if ((fm & 2u) && clast < CPL && lane == lane_last) {
                    const FaceRef F = face_x(1);
                    double* q = F.p + (int64_t)z * F.sb;
#pragma unroll
                    for (int r = 0; r < RPW; ++r)
                        if (WHOLE || yl + r < ny) {
                            q[(int64_t)(yl + r) * F.sa] = cap1[r];
                        }
                }
            }
            if (rare || rare_faces) {
#pragma unroll
                for (int r = 0; r < RPW; ++r) {
#pragma unroll
                    for (int c = 0; c < CPL; ++c) {
                        const int x = xl + 64 * c, y = yl + r;
                        if (y >= ny || x >= nx) continue;
                        const bool has2 = x + 1 < nx;
                        const bool onb = (rare_faces & 48u) != 0;
                        if (!rare && !onb) continue;
                        const int off = r * W + 64 * c;
                        const double* p = pc + off;
                        const double2 cc = *reinterpret_cast<const double2*>(p);
                        const double2 ym = *reinterpret_cast<const double2*>(p - W);
                        const double2 yp = *reinterpret_cast<const double2*>(p + W);
                        const double2 zm = *reinterpret_cast<const double2*>(pm + off);
                        const double2 zp = *reinterpret_cast<const double2*>(pp + off);
                        const double vx = div7(sum7(cc.x, p[-1], cc.y, ym.x, yp.x, zm.x, zp.x));
                        const double vy = div7(sum7(cc.y, cc.x, p[2], ym.y, yp.y, zm.y, zp.y));
                        double* o = op + r * pitch + 64 * c;
                        o[0] = vx;
                        if (has2) o[1] = vy;
                        // rare quotients: redo every face store of this cell with the exact value
                        const uint32_t m = rare ? fm : (rare_faces & fm);
                        if (m) epi_store(d, m, x, y, z, vx, vy, has2);
                    }
                }
            }
        };

        // MAP 1: the same plane update with one cell per lane and column step 32
        // FULL: the tile spans the block's whole width (x0 == 0, nx == TX; e.g.
        // the 96^3 blocks of BASELINE configs[4]) and is whole: the x-edge cells
        // are lane 0 of k = 0 and lane 31 of k = KPL-1 at compile time, so the
        // x-neighbour offsets, the +x capture and the store predicates are
        // per-row constants instead of per-cell selects
        auto compute_plane_s = [&](auto mode_tag, auto whole_tag, auto full_tag, int z, uint32_t fm,
                                   const double* pm, const double* pc, const double* pp) {
            constexpr int MODE = decltype(mode_tag)::value;
            constexpr bool FULL = decltype(full_tag)::value;
            constexpr bool WHOLE = decltype(whole_tag)::value || FULL;
            constexpr int KPL = T::KPL;
            double* op = obase + (int64_t)(z + 1) * zs;
            double cap0[RPW], cap1[RPW];
            const int xlast = nx - 1 - x0;
            const int klast = FULL ? KPL - 1 : xlast >> 5, lane_last = FULL ? 31 : xlast & 31;
            const int kedge_ = FULL ? KPL - 1 : kedge;
            double* zdst = nullptr;
            int64_t zsb = 0;
            double* ymd = nullptr;
            double* ypd = nullptr;
            uint32_t rare_faces = 0;
            if constexpr (MODE == 2) {
                if ((fm & 48u) == 48u) {
                    rare_faces |= 48u;
                } else if (fm & 48u) {
                    const FaceRef F = load_face(&d->epi[(fm & 16u) ? 4 : 5]);
                    zdst = F.p;
                    zsb = F.sb;
                }
                if (fm & 4u) {
                    const FaceRef F = load_face(&d->epi[2]);
                    ymd = F.p + (int64_t)z * F.sb;
                }
                if (fm & 8u) {
                    const FaceRef F = load_face(&d->epi[3]);
                    ypd = F.p + (int64_t)z * F.sb;
                }
            }
            bool rare = false;
#pragma unroll
            for (int r = 0; r < RPW; ++r) {
#pragma unroll
                for (int k = 0; k < KPL; ++k) {
                    const int off = r * W + 32 * k;
                    const double* p = pc + off;
                    // block x edge: the neighbour outside the block comes from the
                    // stage's x ghost vector (offsets fixed for the item)
                    const int om = (k == 0 && xlf) ? xlb + r * (1 - W) : -1;
                    const int oq = (k == kedge_ && xrf) ? xrb + r * (1 - W) : 1;
                    const double sv = sum7(p[0], p[om], p[oq], p[-W], p[W], pm[off], pp[off]);
                    const double v = div7_fast(sv);
                    rare |= div7_rare(v);
                    if constexpr (MODE >= 1) {
                        if (k == 0) cap0[r] = v;
                        if (k == klast) cap1[r] = v;
                    }
                    const int x = xl + 32 * k, y = yl + r;
                    bool v0 = true;
                    if constexpr (!WHOLE) v0 = y < ny && x < nx;
                    if (v0) {
                        double* o = op + r * pitch + 32 * k;
                        asm volatile("st.global.f64 [%0], %1;" ::"l"(o), "d"(v) : "memory");
                        if constexpr (MODE == 2) {
                            if (zdst) zdst[x + (int64_t)y * zsb] = v;
                            if (ymd && y == 0) ymd[x] = v;
                            if (ypd && y == ny - 1) ypd[x] = v;
                        }
                    }
                }
            }
            if constexpr (MODE >= 1) {  // x faces: the lane owning x = 0 / x = nx-1
                if ((fm & 1u) && x0 == 0 && lane == 0) {
                    if constexpr (HOISTX1) {
                        double* q = xq0 + (int64_t)z * xsb0;
#pragma unroll
                        for (int r = 0; r < RPW; ++r)
                            if (WHOLE || yl + r < ny) q[r] = cap0[r];
                    } else {
                        const FaceRef F = face_x(0);
                        double* q = F.p + (int64_t)z * F.sb;
#pragma unroll
                        for (int r = 0; r < RPW; ++r)
                            if (WHOLE || yl + r < ny) {
                                q[(int64_t)(yl + r) * F.sa] = cap0[r];
                            }
                    }
                }
                if ((fm & 2u) && klast < KPL && lane == lane_last) {
                    if constexpr (HOISTX1) {
                        double* q = xq1 + (int64_t)z * xsb1;
#pragma unroll
                        for (int r = 0; r < RPW; ++r)
                            if (WHOLE || yl + r < ny) q[r] = cap1[r];
                    } else {
                        const FaceRef F = face_x(1);
                        double* q = F.p + (int64_t)z * F.sb;
#pragma unroll
                        for (int r = 0; r < RPW; ++r)
                            if (WHOLE || yl + r < ny) {
                                q[(int64_t)(yl + r) * F.sa] = cap1[r];
                            }
                    }
                }
            }
            if (rare || rare_faces) {
#pragma unroll
                for (int r = 0; r < RPW; ++r) {
#pragma unroll
                    for (int k = 0; k < KPL; ++k) {
                        const int x = xl + 32 * k, y = yl + r;
                        if (y >= ny || x >= nx) continue;
                        const int off = r * W + 32 * k;
                        const double* p = pc + off;
                        const int om = (k == 0 && xlf) ? xlb + r * (1 - W) : -1;
                        const int oq = (k == kedge_ && xrf) ? xrb + r * (1 - W) : 1;
                        const double v = div7(sum7(p[0], p[om], p[oq], p[-W], p[W], pm[off], pp[off]));
                        op[r * pitch + 32 * k] = v;
                        const uint32_t m = rare ? fm : (rare_faces & fm);
                        // epi_store writes pairs; pass (v, v) with has2 = false
                        if (m) epi_store(d, m, x, y, z, v, v, false);
                    }
                }
            }
        };

        // stages of planes z-1, z, z+1 are held; every value is read from smem
        acquire(w.z0 - 1);
        int sm = s;
        advance();
        acquire(w.z0);
        int sc = s;
        advance();
        for (int z = w.z0; z < w.z1; ++z) {
            acquire(z + 1);
            const int sp = s;
            advance();
            const double* pm = stage(sm) + sbase;
            const double* pc = stage(sc) + sbase;
            const double* pp = stage(sp) + sbase;
            const uint32_t fm = epi & (touch | (z == 0 ? 16u : 0u) | (z == nz - 1 ? 32u : 0u));
            using M0 = std::integral_constant<int, 0>;
            using M1 = std::integral_constant<int, 1>;
            using M2 = std::integral_constant<int, 2>;
            if constexpr (T::MAP == 1) {
                using F_ = std::false_type;
                using T_ = std::true_type;
                if (fullw) {
                    if (fm & ~3u) compute_plane_s(M2{}, T_{}, T_{}, z, fm, pm, pc, pp);
                    else if (fm) compute_plane_s(M1{}, T_{}, T_{}, z, fm, pm, pc, pp);
                    else compute_plane_s(M0{}, T_{}, T_{}, z, 0u, pm, pc, pp);
                } else {
                    if (fm & ~3u) compute_plane_s(M2{}, F_{}, F_{}, z, fm, pm, pc, pp);
                    else if (fm) compute_plane_s(M1{}, F_{}, F_{}, z, fm, pm, pc, pp);
                    else if (whole) compute_plane_s(M0{}, T_{}, F_{}, z, 0u, pm, pc, pp);
                    else compute_plane_s(M0{}, F_{}, F_{}, z, 0u, pm, pc, pp);
                }
            } else {
                if (fm & ~3u) compute_plane(M2{}, std::false_type{}, z, fm, pm, pc, pp);
                else if (fm && whole) compute_plane(M1{}, std::true_type{}, z, fm, pm, pc, pp);  // x faces only:
                else if (fm) compute_plane(M1{}, std::false_type{}, z, fm, pm, pc, pp);          // half the tiles at ODF >= 8
                else if (whole) compute_plane(M0{}, std::true_type{}, z, 0u, pm, pc, pp);
                else compute_plane(M0{}, std::false_type{}, z, 0u, pm, pc, pp);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[sm]);
            sm = sc;
            sc = sp;
        }
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&empty[sm]);  // plane z1-1
            mbar_arrive(&empty[sc]);  // plane z1
        }
        if (ctl.done) {  // persistent launch: publish this warp's part of the item (release)
            const int sv = ctl.item_slab[it];
            // slabs next to a peer GPU (they stored into its ghost layer; it reads their
            // counter over NVLink) release at system scope, the others at GPU scope
            if (sv & SLAB_PEER) __threadfence_system();
            else __threadfence();
            __syncwarp();
            if (lane == 0) atomicAdd(ctl.done + (sv & SLAB_MASK), 1u);
        }
    }
}

// ------------------------------------------------------------------ persistent: end of a call
// Wait until every peer counter this GPU's slabs depend on reached `need`:
// the peers' epilogue stores into this GPU's ghost layers for the call's
// iterations have all landed when this kernel completes.
__global__ void __launch_bounds__(32) wait_counters_kernel(const unsigned int* const* __restrict__ ptrs, int n,
                                                          uint32_t need, uint64_t limit_ns) {
    for (int i = threadIdx.x; i < n; i += 32) wait_counter(ptrs[i], need, true, limit_ns);
    __threadfence_system();
}

// ------------------------------------------------------------------ face copies
__global__ void __launch_bounds__(256) copy_faces_kernel(const CopyDesc* __restrict__ descs, int per_group) {
    const CopyDesc* g = descs + (int64_t)blockIdx.y * per_group;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // The paper's fused (un)pack: thread count = the largest face, each thread
    // looks at the faces in turn and copies when its index is inside that face
    // (PAPER.md L524).  per_group == 1 is the unfused one-face kernel.
    for (int k = 0; k < per_group; ++k) {
        const int64_t na = g[k].na, nb = g[k].nb;
        if (idx < na * nb) {
            const int64_t b = idx / na, a = idx - b * na;
            const FaceRef src = g[k].src, dst = g[k].dst;
            dst.p[a * dst.sa + b * dst.sb] = src.p[a * src.sa + b * src.sb];
        }
    }
}

// Host-staged exchange moves (exchange.cu host_exchange): the same strided
// copy, one side in pinned host memory mapped into the device.  To host:
// write-through stores (st.global.wt: straight to system memory); from host:
// cache-volatile loads (ld.global.cv: never a line cached from an earlier
// epoch of the staging area).
__global__ void __launch_bounds__(256) stage_copy_kernel(const CopyDesc* __restrict__ descs, int per_group,
                                                         int from_host) {
    const CopyDesc* g = descs + (int64_t)blockIdx.y * per_group;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int k = 0; k < per_group; ++k) {
        const int64_t na = g[k].na, nb = g[k].nb;
        if (idx < na * nb) {
            const int64_t b = idx / na, a = idx - b * na;
            const double* sp = g[k].src.p + a * g[k].src.sa + b * g[k].src.sb;
            double* dp = g[k].dst.p + a * g[k].dst.sa + b * g[k].dst.sb;
            double v;
            if (from_host) {
                asm volatile("ld.global.cv.f64 %0, [%1];" : "=d"(v) : "l"(sp) : "memory");
                *dp = v;
            } else {
                v = *sp;
                asm volatile("st.global.wt.f64 [%0], %1;" ::"l"(dp), "d"(v) : "memory");
            }
        }
    }
}

// ------------------------------------------------------------------ init
__global__ void __launch_bounds__(256) init_kernel(const BlockGeom* __restrict__ geoms, int kind, double p0, double p1,
                                                   double p2, double p3, uint64_t hseed, double boundary, int64_t gx,
                                                   int64_t gy, int64_t gz) {
    const BlockGeom b = geoms[blockIdx.z];
    const int64_t rows = (int64_t)(b.ny + 2) * (b.nz + 2);
    const int x = (int)(blockIdx.x * blockDim.x + threadIdx.x) - 1;
    if (x > b.nx) return;
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const int y = (int)(row % (b.ny + 2)) - 1;
        const int z = (int)(row / (b.ny + 2)) - 1;
        const int64_t gi = b.ox + x, gj = b.oy + y, gk = b.oz + z;
        const bool ghost = gi < 0 || gi >= gx || gj < 0 || gj >= gy || gk < 0 || gk >= gz;
        double v;
        if (kind == 1) {
            v = p0;
        } else if (kind == 2) {
            const double a = __dmul_rn(p0, (double)gi), bb = __dmul_rn(p1, (double)gj), c = __dmul_rn(p2, (double)gk);
            v = __dadd_rn(__dadd_rn(__dadd_rn(a, bb), c), p3);
        } else if (kind == 3) {
            if (ghost) v = boundary;
            else {
                const uint64_t gidx = (uint64_t)gi + (uint64_t)gx * ((uint64_t)gj + (uint64_t)gy * (uint64_t)gk);
                v = (double)(splitmix64(hseed ^ gidx) >> 11) * 0x1p-53;
            }
        } else {
            v = ghost ? boundary : 0.0;
        }
        if (x < 0 || x == b.nx) {  // x ghost arrays (layout: device.cuh)
            if (y >= 0 && y < b.ny) {
                const int64_t o = b.xg_off + (x < 0 ? 0 : b.xg_side) + (int64_t)(z + 1) * b.xg_pitch + y;
                b.buf[0][o] = v;
                b.buf[1][o] = v;
            }
            continue;
        }
        const int64_t o = (int64_t)(z + 1) * b.zs + (int64_t)(y + 1) * b.pitch + XOFF + x;
        b.buf[0][o] = v;
        b.buf[1][o] = v;
    }
}

// ------------------------------------------------------------------ reporting
__global__ void __launch_bounds__(256) checksum_kernel(const BlockGeom* __restrict__ geoms, int which, int64_t gx,
                                                       int64_t gy, unsigned long long* acc) {
    const BlockGeom b = geoms[blockIdx.y];
    const double* u = b.buf[which];
    const int64_t n = (int64_t)b.nx * b.ny * b.nz;
    uint64_t sum = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = i % b.nx, t = i / b.nx, y = t % b.ny, z = t / b.ny;
        const double v = u[(z + 1) * b.zs + (y + 1) * b.pitch + XOFF + x];
        const uint64_t gidx = (uint64_t)(b.ox + x) + (uint64_t)gx * ((uint64_t)(b.oy + y) + (uint64_t)gy * (uint64_t)(b.oz + z));
        sum += splitmix64((uint64_t)__double_as_longlong(v) ^ splitmix64(gidx));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(acc, (unsigned long long)sum);
}

__global__ void __launch_bounds__(256) residual_kernel(const BlockGeom* __restrict__ geoms, int which,
                                                       unsigned long long* acc) {
    const BlockGeom b = geoms[blockIdx.y];
    const double* u = b.buf[which];
    const double* v = b.buf[which ^ 1];
    const int64_t n = (int64_t)b.nx * b.ny * b.nz;
    // max over the bit patterns of |u - v|: non-negative doubles order like
    // their bit patterns, and a NaN difference (bits above +inf's) wins, so a
    // NaN anywhere makes the residual NaN (R11; fmax would drop it)
    unsigned long long m = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = i % b.nx, t = i / b.nx, y = t % b.ny, z = t / b.ny;
        const int64_t o = (z + 1) * b.zs + (y + 1) * b.pitch + XOFF + x;
        const unsigned long long d = (unsigned long long)__double_as_longlong(fabs(__dsub_rn(u[o], v[o])));
        m = d > m ? d : m;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, m, o);
        m = t > m ? t : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(acc, m);
}

// ------------------------------------------------------------------ division self-test
// Compares the stencil's division -- r = div7_fast(s), replaced by div7(s)
// when div7_rare(r) -- and div7 alone with the IEEE division routine on n
// inputs drawn from splitmix64: mode 0 = random bit patterns (every double:
// subnormals, +-inf and NaNs included), 1 = uniform in [0,7) (the workloads'
// range), 2 = small integers times 2^-k (exact / tie-prone quotients), 3 =
// |s| near the subnormal boundary, 4 = the special values +-0, +-inf, NaN,
// +-DBL_MAX and its neighbours, +-min normal, +-min subnormal, 5 = |s| in
// the top binades (sums near overflow), 6 = |s| within 2^-10 of
// 7*2^-1022 (the fast path's stated lower limit).  NaN results compare by
// NaN-ness only (NaN payloads are not part of the result).
__device__ __forceinline__ bool div7_same(double a, double b) {
    if (isnan(b)) return isnan(a);
    return __double_as_longlong(a) == __double_as_longlong(b);
}

__global__ void div7_selftest_kernel(uint64_t n, uint64_t seed, unsigned long long* bad, double* example) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h = splitmix64(seed ^ (i * 0x9E3779B97F4A7C15ULL));
        const int mode = (int)(i % 7);
        double s;
        if (mode == 0) {
            s = __longlong_as_double((long long)h);
        } else if (mode == 1) {
            s = (double)(h >> 11) * 0x1p-53 * 7.0;
        } else if (mode == 2) {
            s = ldexp((double)((long long)(h >> 40) - (1LL << 23)), -(int)((h >> 8) & 63));
        } else if (mode == 3) {
            s = ldexp((double)(h >> 11) * 0x1p-53 + 0.5, -1016 - (int)((h >> 4) & 63));
            if (h & 1) s = -s;
        } else if (mode == 4) {
            const uint64_t special[10] = {0x0ULL, 0x7ff0000000000000ULL, 0x7ff8000000000000ULL, 0x7fefffffffffffffULL,
                                          0x0010000000000000ULL, 0x1ULL, 0x7feffffffffffff0ULL, 0x7ff4000000000001ULL,
                                          0x000fffffffffffffULL, 0x001c000000000000ULL};
            uint64_t b = special[(h >> 1) % 10];
            if ((h >> 8) & 1) b = (b - ((h >> 16) & 15)) & 0x7fffffffffffffffULL;  // neighbours below
            s =__longlong_as_double((long long)(b | ((h & 1) << 63)));  // both signs
        } else if (mode == 5) {
            s = ldexp((double)(h >> 11) * 0x1p-53 + 0.5, 1024 - (int)((h >> 4) & 7));
            if (h & 1) s = -s;
        } else {
            s = __dmul_rn(0x1.cp-1020, 1.0 + ldexp((double)((long long)(h >> 32) - (1LL << 31)), -41));
            if (h & 1) s = -s;
        }
        const double b = __ddiv_rn(s, 7.0);
        double a = div7_fast(s);
        if (div7_rare(a)) a = div7(s);
        const double c = div7(s);
        if (!div7_same(a, b) || !div7_same(c, b)) {
            if (atomicAdd(bad, 1ULL) == 0) { example[0] = s; example[1] = div7_same(a, b) ? c : a; example[2] = b; }
        }
    }
}

cudaError_t launch_div7_selftest(uint64_t n, uint64_t seed, unsigned long long* bad, double* example, int sms,
                                 cudaStream_t st) {
    div7_selftest_kernel<<<sms * 8, 256, 0, st>>>(n, seed, bad, example);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ host launchers
// Tile configurations selectable at run time (kind index):
//          TX  NCW RPW NSTAGE MINB      tile     CTAs/SM (smem)
#define J3D_TILES(X)                                                    \
    X(0, 192, 11, 2, 5, 1)  /* 192x22, 5 x 38 KB stages, 1 CTA/SM       */ \
    X(1, 128, 15, 2, 5, 1)  /* 128x30, 5 x 35 KB, 1 CTA/SM               */ \
    X(2, 64, 8, 2, 7, 3)    /* 64x16, 7 x 10 KB, 3 CTAs/SM               */ \
    X(3, 128, 8, 2, 5, 2)   /* 128x16, 5 x 20 KB, 2 CTAs/SM              */ \
    X(4, 64, 8, 2, 6, 2)    /* 64x16, 6 stages, 2 CTAs/SM                */ \
    X(5, 128, 8, 1, 8, 2)   /* 128x8, 8 stages, 2 CTAs/SM                */ \
    X(6, 192, 15, 2, 4, 1)  /* 192x30, 4 x 51 KB                         */ \
    X(7, 128, 12, 2, 5, 1)  /* 128x24                                    */ \
    X(8, 128, 15, 2, 6, 1)  /* 128x30, 6 stages                          */ \
    X(9, 64, 6, 2, 6, 2)    /* 64x12, 2 CTAs/SM (7 warps)                */ \
    X(10, 64, 12, 2, 6, 1)  /* 64x24, 1 CTA/SM                           */ \
    X(11, 64, 7, 2, 6, 2)   /* 64x14, 2 CTAs/SM (8 warps)                */ \
    X(12, -96, 8, 2, 6, 2)  /* 96x16 one cell per lane (96-wide blocks)  */ \
    X(13, -96, 16, 2, 4, 1) /* 96x32 one cell per lane                   */ \
    X(14, -96, 8, 1, 8, 2)  /* 96x8 one cell per lane                    */ \
    X(15, -96, 8, 1, 6, 3)  /* 96x8, 3 CTAs/SM                           */ \
    X(16, -96, 12, 1, 8, 2) /* 96x12                                     */ \
    X(17, -192, 11, 2, 5, 1) /* 192x22 one cell per lane                 */ \
    X(18, -96, 6, 2, 8, 2)  /* 96x12 (RPW 2)                             */ \
    X(19, -96, 8, 2, 7, 2)  /* 96x16, 7 stages, 2 CTAs/SM                */ \
    X(20, 192, 8, 2, 5, 1)  /* 192x16, 5 x 29 KB stages                  */ \
    X(21, 192, 12, 2, 5, 1) /* 192x24, 5 stages                          */ \
    X(22, -96, 4, 4, 6, 2)  /* 96x16 one cell per lane, 4 rows per warp  */ \
    X(23, -96, 4, 4, 7, 2)  /* 96x16, RPW 4, 7 stages                    */ \
    X(24, -96, 4, 6, 5, 2)  /* 96x24, RPW 6                              */ \
    X(25, -96, 4, 4, 4, 3)  /* 96x16, RPW 4, 3 CTAs/SM                   */ \
    X(26, 192, 6, 4, 5, 1)  /* 192x24, 4 rows per warp                   */ \
    X(27, 192, 8, 3, 5, 1)  /* 192x24, 3 rows per warp                   */

template <class T>
static cudaError_t launch_t(const StencilLaunch& L, cudaStream_t st) {
    // once per device (the attribute belongs to the device's context); ranks may
    // be threads of one process, on one device or several
    static std::atomic<uint64_t> attr_set{0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_set.load(std::memory_order_acquire) & bit)) {
        e = cudaFuncSetAttribute(stencil_tma_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        attr_set.fetch_or(bit, std::memory_order_acq_rel);
    }
    if (L.n_items <= 0) return cudaSuccess;
    stencil_tma_kernel<T><<<L.grid, T::THREADS, T::SMEM_BYTES, st>>>(
        L.descs, L.tmaps, L.tmaps_pro, L.tmaps_x, L.items, L.n_items, L.parity,
        (L.faces ? 1 : 0) | ((L.tma_mode & 3) << 2) | (L.prefetch ? 0 : 16) | (L.depfence ? 32 : 0), L.sched, L.ctl);
    return cudaGetLastError();
}

template <class T>
static cudaError_t occ_t(int* blocks) {
    cudaError_t e = cudaFuncSetAttribute(stencil_tma_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         T::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, stencil_tma_kernel<T>, T::THREADS, T::SMEM_BYTES);
}

#define J3D_TYPE(k, tx, ncw, rpw, ns, mb) Tile<(tx > 0 ? tx : -tx), ncw, rpw, ns, mb, (tx > 0 ? 0 : 1)>
#define J3D_TYPE_YS(k, tx, ncw, rpw, ns, mb) Tile<(tx > 0 ? tx : -tx), ncw, rpw, ns, mb, (tx > 0 ? 0 : 1), true>

// The tile kinds strategy C uses by default (setup.cu) also get an instance with y
// side rows for its TMA-fed prologue (same parameters as in J3D_TILES).
#define J3D_TILES_YS(X)          \
    X(0, 192, 11, 2, 5, 1)       \
    X(1, 128, 15, 2, 5, 1)       \
    X(4, 64, 8, 2, 6, 2)         \
    X(12, -96, 8, 2, 6, 2)       \
    X(21, 192, 12, 2, 5, 1)      \
    X(26, 192, 6, 4, 5, 1)

int num_tile_kinds() { return 28; }

TileShape tile_shape(int kind) {
    switch (kind) {
#define X(k, tx, ncw, rpw, ns, mb) \
    case k: return TileShape{(tx > 0 ? tx : -tx), ncw * rpw, ncw};
        J3D_TILES(X)
#undef X
    }
    return TileShape{0, 0, 0};
}

cudaError_t launch_stencil(const StencilLaunch& L, cudaStream_t st) {
    if (L.yside) {
        switch (L.kind) {
#define X(k, tx, ncw, rpw, ns, mb) \
    case k: return launch_t<J3D_TYPE_YS(k, tx, ncw, rpw, ns, mb)>(L, st);
            J3D_TILES_YS(X)
#undef X
        }
        return cudaErrorInvalidValue;
    }
    switch (L.kind) {
#define X(k, tx, ncw, rpw, ns, mb) \
    case k: return launch_t<J3D_TYPE(k, tx, ncw, rpw, ns, mb)>(L, st);
        J3D_TILES(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

cudaError_t stencil_occupancy(int kind, bool ys, int* blocks_per_sm) {
    if (ys) {
        switch (kind) {
#define X(k, tx, ncw, rpw, ns, mb) \
    case k: return occ_t<J3D_TYPE_YS(k, tx, ncw, rpw, ns, mb)>(blocks_per_sm);
            J3D_TILES_YS(X)
#undef X
        }
        return cudaErrorInvalidValue;
    }
    switch (kind) {
#define X(k, tx, ncw, rpw, ns, mb) \
    case k: return occ_t<J3D_TYPE(k, tx, ncw, rpw, ns, mb)>(blocks_per_sm);
        J3D_TILES(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

// Load every kernel a context may launch now, at create time.  CUDA's lazy
// module loading would otherwise load a kernel at its first launch, and that
// load waits for kernels already running on the device -- a deadlock when a
// running kernel waits for another rank on the same GPU (a persistent launch
// spinning on a peer's slab counters while this rank's first end-of-call
// wait kernel is being loaded).
template <class T>
static cudaError_t preload_t() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, stencil_tma_kernel<T>);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(stencil_tma_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM_BYTES);
}

cudaError_t preload_kernels(int kind, bool ys) {
    cudaError_t e = cudaErrorInvalidValue;
    if (ys) {
        switch (kind) {
#define X(k, tx, ncw, rpw, ns, mb) \
    case k: e = preload_t<J3D_TYPE_YS(k, tx, ncw, rpw, ns, mb)>(); break;
            J3D_TILES_YS(X)
#undef X
        }
    } else {
        switch (kind) {
#define X(k, tx, ncw, rpw, ns, mb) \
    case k: e = preload_t<J3D_TYPE(k, tx, ncw, rpw, ns, mb)>(); break;
            J3D_TILES(X)
#undef X
        }
    }
    if (e != cudaSuccess) return e;
    cudaFuncAttributes a;
    const void* fns[] = {(const void*)wait_counters_kernel, (const void*)copy_faces_kernel,
                         (const void*)stage_copy_kernel, (const void*)init_kernel,
                         (const void*)checksum_kernel, (const void*)residual_kernel};
    for (const void* f : fns)
        if ((e = cudaFuncGetAttributes(&a, f)) != cudaSuccess) return e;
    return cudaSuccess;
}

bool tile_yside(int kind) {
    switch (kind) {
#define X(k, tx, ncw, rpw, ns, mb) \
    case k: return J3D_TYPE_YS(k, tx, ncw, rpw, ns, mb)::YS;
        J3D_TILES_YS(X)
#undef X
    }
    return false;
}

int stencil_box_w(int kind) { return tile_shape(kind).tx + 8; }
int stencil_box_h(int kind) { return tile_shape(kind).ty + 2; }

cudaError_t launch_wait_counters(const unsigned int* const* ptrs, int n, uint32_t need, uint64_t limit_ns,
                                 cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    wait_counters_kernel<<<1, 32, 0, st>>>(ptrs, n, need, limit_ns);
    return cudaGetLastError();
}

cudaError_t launch_copy_faces(const CopyDesc* d, int per_group, int groups, int64_t max_cells, cudaStream_t st) {
    if (groups <= 0 || max_cells <= 0) return cudaSuccess;
    const int64_t nblk = (max_cells + 255) / 256;
    if (nblk > 0x7fffffff || groups > 65535) return cudaErrorInvalidValue;
    copy_faces_kernel<<<dim3((unsigned)nblk, (unsigned)groups), 256, 0, st>>>(d, per_group);
    return cudaGetLastError();
}

cudaError_t launch_stage_copy(const CopyDesc* d, int per_group, int groups, int64_t max_cells, bool from_host,
                              cudaStream_t st) {
    if (groups <= 0 || max_cells <= 0) return cudaSuccess;
    const int64_t nblk = (max_cells + 255) / 256;
    if (nblk > 0x7fffffff || groups > 65535) return cudaErrorInvalidValue;
    stage_copy_kernel<<<dim3((unsigned)nblk, (unsigned)groups), 256, 0, st>>>(d, per_group, from_host ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_init(const BlockGeom* g, int nblocks, int max_nx, int64_t max_rows, int kind, const double* p,
                        uint64_t seed, double boundary, int64_t gx, int64_t gy, int64_t gz, cudaStream_t st) {
    if (nblocks <= 0) return cudaSuccess;
    const unsigned gxd = (unsigned)((max_nx + 2 + 255) / 256);
    const unsigned gyd = (unsigned)(max_rows < 65535 ? max_rows : 65535);
    // the hash init seeds each cell with splitmix64(splitmix64(seed) ^ gidx)
    uint64_t z = seed + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    const uint64_t hs = z ^ (z >> 31);
    init_kernel<<<dim3(gxd, gyd, (unsigned)nblocks), 256, 0, st>>>(g, kind, p[0], p[1], p[2], p[3], hs, boundary, gx,
                                                                     gy, gz);
    return cudaGetLastError();
}

cudaError_t launch_checksum(const BlockGeom* g, int nblocks, int which, int64_t gx, int64_t gy, unsigned long long* acc,
                            int sms, cudaStream_t st) {
    if (nblocks <= 0) return cudaSuccess;
    checksum_kernel<<<dim3((unsigned)(sms * 4), (unsigned)nblocks), 256, 0, st>>>(g, which, gx, gy, acc);
    return cudaGetLastError();
}

cudaError_t launch_residual(const BlockGeom* g, int nblocks, int which, unsigned long long* acc, int sms,
                            cudaStream_t st) {
    if (nblocks <= 0) return cudaSuccess;
    residual_kernel<<<dim3((unsigned)(sms * 4), (unsigned)nblocks), 256, 0, st>>>(g, which, acc);
    return cudaGetLastError();
}

}  // namespace j3d
