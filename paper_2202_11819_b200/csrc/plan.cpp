// plan.cpp -- decomposition planner (see plan.h for the cited passages).
#include "plan.h"

#include "../../include/jacobi3d.h"

namespace j3d {

int decompose(const std::array<int64_t, 3>& d, int64_t n, std::array<int32_t, 3>& out, std::string& msg) {
    if (n < 1 || d[0] < 1 || d[1] < 1 || d[2] < 1) {
        msg = "extents and part count must be >= 1";
        return J3D_EINVAL;
    }
    bool found = false;
    int64_t best_area = 0;
    std::array<int64_t, 3> best{0, 0, 0};
    bool fail[3] = {false, false, false};
    // ordered factor triples, enumerated lexicographically so that the first
    // minimum found is the lexicographically smallest
    for (int64_t px = 1; px <= n; ++px) {
        if (n % px) continue;
        for (int64_t py = 1; py <= n / px; ++py) {
            if ((n / px) % py) continue;
            const int64_t pz = n / px / py;
            const int64_t p[3] = {px, py, pz};
            bool ok = true;
            for (int a = 0; a < 3; ++a)
                if (d[a] % p[a]) { fail[a] = true; ok = false; }
            if (!ok) continue;
            const int64_t bx = d[0] / px, by = d[1] / py, bz = d[2] / pz;
            const int64_t area = n * 2 * (bx * by + by * bz + bx * bz);
            if (!found || area < best_area) {
                found = true;
                best_area = area;
                best = {px, py, pz};
            }
        }
    }
    if (!found) {
        msg = "no divisible factorisation of " + std::to_string(n) + " parts; failing dimension(s):";
        const char* nm = "xyz";
        for (int a = 0; a < 3; ++a)
            if (fail[a]) msg += std::string(" ") + nm[a];
        return J3D_EDECOMP;
    }
    out = {(int32_t)best[0], (int32_t)best[1], (int32_t)best[2]};
    return J3D_OK;
}

int make_plan(const std::array<int64_t, 3>& gdim, const std::array<int64_t, 3>& bdim, int32_t odf,
              int32_t n_gpus, Plan& P, std::string& msg) {
    if (odf < 1 || n_gpus < 1) {
        msg = "odf and n_gpus must be >= 1";
        return J3D_EINVAL;
    }
    for (int a = 0; a < 3; ++a)
        if (gdim[a] < 1) {
            msg = "global extent must be >= 1 on every axis";
            return J3D_EINVAL;
        }
    int rc = decompose(gdim, n_gpus, P.gpu_grid, msg);
    if (rc) return rc;
    std::array<int64_t, 3> per;
    for (int a = 0; a < 3; ++a) per[a] = gdim[a] / P.gpu_grid[a];
    const bool user_blocks = bdim[0] || bdim[1] || bdim[2];
    if (user_blocks) {
        const char* nm = "xyz";
        for (int a = 0; a < 3; ++a) {
            if (bdim[a] < 1) {
                msg = "block extents must all be >= 1 (or all 0 for automatic)";
                return J3D_EINVAL;
            }
            if (per[a] % bdim[a]) {
                msg = std::string("block extent does not divide the per-GPU extent along ") + nm[a];
                return J3D_EDECOMP;
            }
            P.blk_grid[a] = (int32_t)(per[a] / bdim[a]);
        }
        if ((int64_t)P.blk_grid[0] * P.blk_grid[1] * P.blk_grid[2] != odf) {
            msg = "blocks per GPU (" + std::to_string((int64_t)P.blk_grid[0] * P.blk_grid[1] * P.blk_grid[2]) +
                  ") != ODF (" + std::to_string(odf) + ")";
            return J3D_EDECOMP;
        }
    } else {
        rc = decompose(per, odf, P.blk_grid, msg);
        if (rc) return rc;
    }
    P.gdim = gdim;
    P.n_gpus = n_gpus;
    P.odf = odf;
    for (int a = 0; a < 3; ++a) {
        P.ext[a] = per[a] / P.blk_grid[a];
        P.nblk[a] = (int64_t)P.gpu_grid[a] * P.blk_grid[a];
    }
    const int64_t nb = P.nblk[0] * P.nblk[1] * P.nblk[2];
    P.blocks.assign(nb, BlockPlan{});
    P.by_rank.assign(n_gpus, {});
    for (int64_t k = 0; k < P.nblk[2]; ++k)
        for (int64_t j = 0; j < P.nblk[1]; ++j)
            for (int64_t i = 0; i < P.nblk[0]; ++i) {
                const int64_t id = i + P.nblk[0] * (j + P.nblk[1] * k);
                BlockPlan& b = P.blocks[id];
                b.id = id;
                b.gpos = {i, j, k};
                b.origin = {i * P.ext[0], j * P.ext[1], k * P.ext[2]};
                const int64_t gi = i / P.blk_grid[0], gj = j / P.blk_grid[1], gk = k / P.blk_grid[2];
                b.owner = (int32_t)(gi + P.gpu_grid[0] * (gj + P.gpu_grid[1] * gk));
                const int64_t li = i % P.blk_grid[0], lj = j % P.blk_grid[1], lk = k % P.blk_grid[2];
                b.local = (int32_t)(li + P.blk_grid[0] * (lj + P.blk_grid[1] * lk));
            }
    for (auto& b : P.blocks) {
        for (int f = 0; f < 6; ++f) {
            const int a = f / 2, dir = (f & 1) ? 1 : -1;
            std::array<int64_t, 3> q = b.gpos;
            q[a] += dir;
            if (q[a] < 0 || q[a] >= P.nblk[a]) {
                b.nbr[f] = -1;
                b.nbr_rank[f] = -1;
            } else {
                b.nbr[f] = q[0] + P.nblk[0] * (q[1] + P.nblk[1] * q[2]);
                b.nbr_rank[f] = -2;  // filled below
            }
        }
    }
    for (auto& b : P.blocks)
        for (int f = 0; f < 6; ++f)
            if (b.nbr[f] >= 0) b.nbr_rank[f] = P.blocks[b.nbr[f]].owner;
    for (int r = 0; r < n_gpus; ++r) P.by_rank[r].assign(odf, -1);
    for (auto& b : P.blocks) P.by_rank[b.owner][b.local] = b.id;
    return J3D_OK;
}

}  // namespace j3d
