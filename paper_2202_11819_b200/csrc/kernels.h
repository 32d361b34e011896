// kernels.h -- host-side launch interface of the sm_100a kernels (kernels.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"

namespace j3d {

struct TileShape {
    int tx, ty;
    int ncw;  // consumer warps per CTA
};

struct StencilLaunch {
    const StencilDesc* descs;  // device, [2*n_local_blocks]
    const CUtensorMap* tmaps;  // device, [2*n_local_blocks], 64-B aligned
    const CUtensorMap* tmaps_pro;    // device, [2*n_local_blocks][6]: strategy C's receive buffers per face
    const CUtensorMap* tmaps_x;      // device, [2*n_local_blocks]: x ghost vectors (y, z, side), box TY x 1 x 1
    int tma_mode;            // L2 policy of the plane loads: 0 plain, 1 evict_first, 2 evict_last (default)
    const WorkItem* items;     // device
    int n_items;
    int parity;  // input buffer parity
    int grid;    // persistent CTAs
    int kind;    // tile configuration (kernels.cu J3D_TILES)
    bool faces;  // any prologue/epilogue faces in this launch
    bool yside = false;      // launch the tile's instance with y side rows (strategy C)
    bool prefetch = false;   // the producer claims its next item when the current one starts
    bool depfence = false;   // persistent: a gpu/sys fence after the dependency polling (experiment)
    unsigned int* sched;     // device [2] scheduler counters (zero on entry; reset by the kernel)
    IterCtl ctl;             // iterations in this launch + slab dependency tracking (persistent)
};

int num_tile_kinds();
TileShape tile_shape(int kind);
int stencil_box_w(int kind);
bool tile_yside(int kind);  // the kind has an instance whose stages carry y side rows (strategy C's TMA-fed y ghost rows)
int stencil_box_h(int kind);
cudaError_t launch_stencil(const StencilLaunch& L, cudaStream_t st);
cudaError_t stencil_occupancy(int kind, bool ys, int* blocks_per_sm);
cudaError_t preload_kernels(int kind, bool ys);  // defeat lazy loading (see kernels.cu)
cudaError_t launch_div7_selftest(uint64_t n, uint64_t seed, unsigned long long* bad, double* example, int sms,
                                 cudaStream_t st);
cudaError_t launch_wait_counters(const unsigned int* const* ptrs, int n, uint32_t need, uint64_t limit_ns,
                                 cudaStream_t st);
cudaError_t launch_stage_copy(const CopyDesc* d, int per_group, int groups, int64_t max_cells, bool from_host,
                              cudaStream_t st);
cudaError_t launch_copy_faces(const CopyDesc* d, int per_group, int groups, int64_t max_cells, cudaStream_t st);
cudaError_t launch_init(const BlockGeom* g, int nblocks, int max_nx, int64_t max_rows, int kind, const double* p,
                        uint64_t seed, double boundary, int64_t gx, int64_t gy, int64_t gz, cudaStream_t st);
cudaError_t launch_checksum(const BlockGeom* g, int nblocks, int which, int64_t gx, int64_t gy,
                            unsigned long long* acc, int sms, cudaStream_t st);
cudaError_t launch_residual(const BlockGeom* g, int nblocks, int which, unsigned long long* acc, int sms,
                            cudaStream_t st);

}  // namespace j3d
