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
// a list of work items (block, xy tile, z range).  Per CTA one producer warp
// streams (TX+4) x (TY+2) xy-planes of the input buffer -- the tile plus its
// 1-cell halo, ghost cells included -- into an NSTAGE-deep shared-memory ring
// with TMA (cp.async.bulk.tensor.3d, mbarrier complete_tx).  Eight consumer
// warps march up z: each thread keeps the centre values of planes z-1, z,
// z+1 for its 2*CPL x RPW cells in registers, reads the four in-plane
// neighbours of plane z from shared memory, and writes 16-byte vector stores
// of the new plane to HBM.  Every input plane is fetched once per tile (plus
// the 1-cell halo, which neighbouring tiles fetch concurrently and therefore
// hit in L2), every output cell written once: the compulsory 16 B/LUP.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tmap_acquire(const CUtensorMap* m) {
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(m))
                 : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// The update itself: SPEC.md L388, summed left to right, IEEE division.
__device__ __forceinline__ double jacobi7(double c, double xm, double xp, double ym, double yp, double zm, double zp) {
    double s = __dadd_rn(c, xm);
    s = __dadd_rn(s, xp);
    s = __dadd_rn(s, ym);
    s = __dadd_rn(s, yp);
    s = __dadd_rn(s, zm);
    s = __dadd_rn(s, zp);
    return __ddiv_rn(s, 7.0);
}

// ------------------------------------------------------------------ stencil
template <int TX, int TY, int NSTAGE>
struct StencilShape {
    static constexpr int NCW = 8;  // consumer warps
    static constexpr int RPW = TY / NCW;
    static constexpr int CPL = TX / 64;  // double2 column groups per lane
    static constexpr int W = TX + 4;     // smem row: x0-2 .. x0+TX+1
    static constexpr int H = TY + 2;
    static constexpr uint32_t TX_BYTES = W * H * 8;
    static constexpr int STAGE_BYTES = (W * H * 8 + 127) / 128 * 128;
    static constexpr int SMEM_BYTES = NSTAGE * STAGE_BYTES + 2 * NSTAGE * 8 + 128;
    static constexpr int THREADS = 32 * (NCW + 1);
    static_assert(TY % NCW == 0 && TX % 64 == 0 && W <= 256, "tile shape");
};

template <int TX, int TY, int NSTAGE, bool FACES>
__global__ void __launch_bounds__(StencilShape<TX, TY, NSTAGE>::THREADS, FACES ? 1 : 2)
    stencil_tma_kernel(const StencilDesc* __restrict__ descs, const CUtensorMap* __restrict__ tmaps,
                       const WorkItem* __restrict__ items, int n_items, int parity) {
    using S = StencilShape<TX, TY, NSTAGE>;
    constexpr int NCW = S::NCW, RPW = S::RPW, CPL = S::CPL, W = S::W;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * S::STAGE_BYTES);
    uint64_t* empty = full + NSTAGE;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NCW) {  // ---------------- producer warp: TMA plane loads
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
                const WorkItem w = items[it];
                const CUtensorMap* tm = tmaps + (2 * w.blk + parity);
                tmap_acquire(tm);
                const int c0 = XOFF + w.tx * TX - 2, c1 = w.ty * TY;
                for (int z = w.z0 - 1; z <= w.z1; ++z) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_expect_tx(&full[s], S::TX_BYTES);
                    tma_load_3d(smem + s * S::STAGE_BYTES, tm, &full[s], c0, c1, z + 1);
                    if (++s == NSTAGE) { s = 0; ph ^= 1; }
                }
            }
        }
        return;
    }

    // ---------------- consumer warps
    int s = 0;
    uint32_t ph = 0;
    auto advance = [&]() { if (++s == NSTAGE) { s = 0; ph ^= 1; } };
    auto stage = [&](int i) { return reinterpret_cast<const double*>(smem + i * S::STAGE_BYTES); };

    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const WorkItem w = items[it];
        const StencilDesc* d = descs + (2 * w.blk + parity);
        const int nx = d->nx, ny = d->ny, nz = d->nz;
        const int64_t pitch = d->pitch, zs = d->zs;
        double* __restrict__ out = d->out;
        const uint32_t epi = FACES ? d->epi_mask : 0u, pro = FACES ? d->pro_mask : 0u;
        const int x0 = w.tx * TX, y0 = w.ty * TY;
        const bool edge_xy = FACES && (epi | pro) &&
                             (x0 == 0 || x0 + TX >= nx - 1 || y0 == 0 || y0 + TY >= ny);

        double2 prev[RPW][CPL], cur[RPW][CPL], nxt[RPW][CPL];
        auto read_centres = [&](const double* st, double2 (&v)[RPW][CPL]) {
#pragma unroll
            for (int r = 0; r < RPW; ++r)
#pragma unroll
                for (int c = 0; c < CPL; ++c)
                    v[r][c] = *reinterpret_cast<const double2*>(st + (warp * RPW + r + 1) * W + 64 * c + 2 * lane + 2);
        };
        // face (z-plane) prologue: centre values of a ghost plane from a receive buffer
        auto read_face_plane = [&](const FaceRef& f, double2 (&v)[RPW][CPL]) {
#pragma unroll
            for (int r = 0; r < RPW; ++r) {
                const int y = y0 + warp * RPW + r;
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int x = x0 + 64 * c + 2 * lane;
                    if (y < ny && x < nx) {
                        v[r][c].x = f.p[x * f.sa + y * f.sb];
                        if (x + 1 < nx) v[r][c].y = f.p[(x + 1) * f.sa + y * f.sb];
                    }
                }
            }
        };

        // plane z0-1: only its centre values are needed (as -z neighbours)
        mbar_wait(&full[s], ph);
        read_centres(stage(s), prev);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        advance();
        if (FACES && w.z0 == 0 && (pro & (1u << 4))) read_face_plane(d->pro[4], prev);
        // plane z0
        mbar_wait(&full[s], ph);
        read_centres(stage(s), cur);
        int scur = s;
        advance();

        for (int z = w.z0; z < w.z1; ++z) {
            mbar_wait(&full[s], ph);
            read_centres(stage(s), nxt);
            if (FACES && z + 1 == nz && (pro & (1u << 5))) read_face_plane(d->pro[5], nxt);
            const double* st = stage(scur);
            const bool face_here = FACES && (epi | pro) && (edge_xy || z == 0 || z == nz - 1);
#pragma unroll
            for (int r = 0; r < RPW; ++r) {
                const int ly = warp * RPW + r;
                const int y = y0 + ly;
                if (y >= ny) continue;
                double* orow = out + (int64_t)(z + 1) * zs + (int64_t)(y + 1) * pitch + XOFF;
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int lx = 64 * c + 2 * lane;
                    const int x = x0 + lx;
                    if (x >= nx) continue;
                    const double* p = st + (ly + 1) * W + lx + 2;
                    double2 cc = cur[r][c];
                    double L = p[-1];
                    double R = p[2];
                    double2 ym = *reinterpret_cast<const double2*>(p - W);
                    double2 yp = *reinterpret_cast<const double2*>(p + W);
                    const double2 zm = prev[r][c], zp = nxt[r][c];
                    const bool has2 = x + 1 < nx;
                    if (FACES && face_here && pro) {  // prologue: ghosts from receive buffers
                        if ((pro & 1u) && x == 0) { const FaceRef f = d->pro[0]; L = f.p[y * f.sa + z * f.sb]; }
                        if (pro & 2u) {
                            const FaceRef f = d->pro[1];
                            if (x + 1 == nx) cc.y = f.p[y * f.sa + z * f.sb];
                            else if (x + 2 == nx) R = f.p[y * f.sa + z * f.sb];
                        }
                        if ((pro & 4u) && y == 0) {
                            const FaceRef f = d->pro[2];
                            ym.x = f.p[x * f.sa + z * f.sb];
                            if (has2) ym.y = f.p[(x + 1) * f.sa + z * f.sb];
                        }
                        if ((pro & 8u) && y == ny - 1) {
                            const FaceRef f = d->pro[3];
                            yp.x = f.p[x * f.sa + z * f.sb];
                            if (has2) yp.y = f.p[(x + 1) * f.sa + z * f.sb];
                        }
                    }
                    const double vx = jacobi7(cc.x, L, cc.y, ym.x, yp.x, zm.x, zp.x);
                    const double vy = jacobi7(cc.y, cc.x, R, ym.y, yp.y, zm.y, zp.y);
                    if (has2) *reinterpret_cast<double2*>(orow + x) = make_double2(vx, vy);
                    else orow[x] = vx;
                    if (FACES && face_here && epi) {  // epilogue: new boundary layer -> face destinations
                        if ((epi & 1u) && x == 0) { const FaceRef f = d->epi[0]; f.p[y * f.sa + z * f.sb] = vx; }
                        if (epi & 2u) {
                            const FaceRef f = d->epi[1];
                            if (x == nx - 1) f.p[y * f.sa + z * f.sb] = vx;
                            else if (x + 1 == nx - 1) f.p[y * f.sa + z * f.sb] = vy;
                        }
                        if ((epi & 4u) && y == 0) {
                            const FaceRef f = d->epi[2];
                            f.p[x * f.sa + z * f.sb] = vx;
                            if (has2) f.p[(x + 1) * f.sa + z * f.sb] = vy;
                        }
                        if ((epi & 8u) && y == ny - 1) {
                            const FaceRef f = d->epi[3];
                            f.p[x * f.sa + z * f.sb] = vx;
                            if (has2) f.p[(x + 1) * f.sa + z * f.sb] = vy;
                        }
                        if ((epi & 16u) && z == 0) {
                            const FaceRef f = d->epi[4];
                            f.p[x * f.sa + y * f.sb] = vx;
                            if (has2) f.p[(x + 1) * f.sa + y * f.sb] = vy;
                        }
                        if ((epi & 32u) && z == nz - 1) {
                            const FaceRef f = d->epi[5];
                            f.p[x * f.sa + y * f.sb] = vx;
                            if (has2) f.p[(x + 1) * f.sa + y * f.sb] = vy;
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[scur]);
            scur = s;
            advance();
#pragma unroll
            for (int r = 0; r < RPW; ++r)
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    prev[r][c] = cur[r][c];
                    cur[r][c] = nxt[r][c];
                }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[scur]);  // plane z1
    }
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
    double m = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = i % b.nx, t = i / b.nx, y = t % b.ny, z = t / b.ny;
        const int64_t o = (z + 1) * b.zs + (y + 1) * b.pitch + XOFF + x;
        m = fmax(m, fabs(u[o] - v[o]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    // non-negative doubles order like their bit patterns
    if ((threadIdx.x & 31) == 0) atomicMax(acc, (unsigned long long)__double_as_longlong(m));
}

// ------------------------------------------------------------------ host launchers
template <int TX, int TY, int NSTAGE, bool FACES>
static cudaError_t launch_stencil_t(const StencilLaunch& L, cudaStream_t st) {
    using S = StencilShape<TX, TY, NSTAGE>;
    auto kern = stencil_tma_kernel<TX, TY, NSTAGE, FACES>;
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    if (L.n_items <= 0) return cudaSuccess;
    kern<<<L.grid, S::THREADS, S::SMEM_BYTES, st>>>(L.descs, L.tmaps, L.items, L.n_items, L.parity);
    return cudaGetLastError();
}

template <int TX, int TY, int NSTAGE, bool FACES>
static cudaError_t occupancy_t(int* blocks) {
    using S = StencilShape<TX, TY, NSTAGE>;
    auto kern = stencil_tma_kernel<TX, TY, NSTAGE, FACES>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, kern, S::THREADS, S::SMEM_BYTES);
}

// Tile configurations (TX, TY, NSTAGE).  Kind 0: wide blocks, kind 1: narrow.
#define J3D_TILE0 128, 16, 4
#define J3D_TILE1 64, 16, 4

TileShape tile_shape(int kind) {
    if (kind == 0) return TileShape{128, 16};
    return TileShape{64, 16};
}

cudaError_t launch_stencil(const StencilLaunch& L, cudaStream_t st) {
    if (L.kind == 0) return L.faces ? launch_stencil_t<J3D_TILE0, true>(L, st) : launch_stencil_t<J3D_TILE0, false>(L, st);
    return L.faces ? launch_stencil_t<J3D_TILE1, true>(L, st) : launch_stencil_t<J3D_TILE1, false>(L, st);
}

cudaError_t stencil_occupancy(int kind, bool faces, int* blocks_per_sm) {
    if (kind == 0) return faces ? occupancy_t<J3D_TILE0, true>(blocks_per_sm) : occupancy_t<J3D_TILE0, false>(blocks_per_sm);
    return faces ? occupancy_t<J3D_TILE1, true>(blocks_per_sm) : occupancy_t<J3D_TILE1, false>(blocks_per_sm);
}

int stencil_box_w(int kind) { return tile_shape(kind).tx + 4; }
int stencil_box_h(int kind) { return tile_shape(kind).ty + 2; }

cudaError_t launch_copy_faces(const CopyDesc* d, int per_group, int groups, int64_t max_cells, cudaStream_t st) {
    if (groups <= 0 || max_cells <= 0) return cudaSuccess;
    const int64_t nblk = (max_cells + 255) / 256;
    if (nblk > 0x7fffffff || groups > 65535) return cudaErrorInvalidValue;
    copy_faces_kernel<<<dim3((unsigned)nblk, (unsigned)groups), 256, 0, st>>>(d, per_group);
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
