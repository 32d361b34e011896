// plan.h -- host-only decomposition planner.
//
// "the grid is decomposed in a way that minimizes the
// aggregate surface area, which is tied to communication volume";
// L566-568: ODF = chares per PE and GPU.  Tie-break / divisibility:
// SPEC.md L358-361, L376-384 (reading R9).  Mapping: GPU grid
// first, then the block grid inside each GPU (reading R10).
#pragma once
#include <array>
#include <cstdint>
#include <string>
#include <vector>

namespace j3d {

// face index f: 0 -x, 1 +x, 2 -y, 3 +y, 4 -z, 5 +z ; opposite = f ^ 1
enum Face { XM = 0, XP = 1, YM = 2, YP = 3, ZM = 4, ZP = 5 };

struct BlockPlan {
    int64_t id;                   // x-fastest index on the global block grid
    std::array<int64_t, 3> gpos;  // position on the global block grid
    std::array<int64_t, 3> origin;// global coordinate of owned cell (0,0,0)
    int32_t owner;                // rank
    int32_t local;                // index among the owner's blocks (x-fastest inside the GPU)
    std::array<int64_t, 6> nbr;   // neighbour block id or -1 (global Dirichlet boundary)
    std::array<int32_t, 6> nbr_rank;
};

struct Plan {
    std::array<int64_t, 3> gdim;      // global owned cells
    std::array<int32_t, 3> gpu_grid;  // (px,py,pz)
    std::array<int32_t, 3> blk_grid;  // blocks per GPU per axis
    std::array<int64_t, 3> ext;       // block extent
    std::array<int64_t, 3> nblk;      // global block grid = gpu_grid * blk_grid
    int32_t n_gpus = 1, odf = 1;
    std::vector<BlockPlan> blocks;    // all blocks, by id
    std::vector<std::vector<int64_t>> by_rank;  // block ids per rank, local order
};

// Returns 0 or a J3D_E* code; msg receives the reason.
int decompose(const std::array<int64_t, 3>& dims, int64_t n, std::array<int32_t, 3>& out, std::string& msg);
int make_plan(const std::array<int64_t, 3>& gdim, const std::array<int64_t, 3>& bdim, int32_t odf,
              int32_t n_gpus, Plan& plan, std::string& msg);

inline int64_t face_cells(const std::array<int64_t, 3>& e, int f) {
    return (f < 2) ? e[1] * e[2] : (f < 4) ? e[0] * e[2] : e[0] * e[1];
}

}  // namespace j3d
