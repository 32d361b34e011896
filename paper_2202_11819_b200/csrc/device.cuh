// device.cuh -- layouts and descriptors shared by the host orchestrator and
// the sm_100a kernels of the Jacobi3D hot path.
//
// HBM layout of one block buffer:
//   a ghosted 3D array of (nz+2) planes x (ny+2) rows x pitch doubles.  Owned
//   cell (x,y,z), x in [0,nx), lives at
//       base[(z+1)*zs + (y+1)*pitch + XOFF + x],   zs = pitch*(ny+2)
//   XOFF = 16 doubles puts every owned row on a 128-byte boundary (pitch is a
//   multiple of 16 doubles and buffers are 256-byte aligned), so warps read
//   and write whole 128-byte lines and 16-byte vector accesses are aligned.
//   The y and z ghost layers are rows / planes of this array (y = -1, ny;
//   z = -1, nz).  The x ghost layers are NOT columns of it: each buffer is
//   followed by two x ghost arrays (-x, +x), element (y, z) at
//       xg[side][(z+1)*xg_pitch + y],   xg_pitch = ny rounded up to even,
//   so a ghost column costs no partially used 128-byte line per row (on
//   96-wide blocks those lines were a third of the DRAM reads) and the
//   neighbour's epilogue stores it contiguously in y.  The stencil's TMA
//   map starts at the owned column 0 and ends at nx - 1 (the halo columns
//   beyond a block edge are zero-filled out of bounds) and a second map
//   loads the x ghost vectors of the tile's rows.
#pragma once
#include <cstdint>

namespace j3d {

#ifndef J3D_XOFF
#define J3D_XOFF 16
#endif
constexpr int XOFF = J3D_XOFF;  // even (16-byte aligned cell pairs); -DJ3D_XOFF only for layout experiments
constexpr int PITCH_ALIGN = 16;  // doubles

struct FaceRef {  // element (a,b) of a 2D face lives at p[a*sa + b*sb]
    double* p;
    int64_t sa, sb;
};

// One (block, buffer parity) as seen by the stencil kernel.
struct StencilDesc {
    const double* in;   // ghosted input buffer  (u^n)
    double* out;        // ghosted output buffer (u^{n+1})
    int32_t nx, ny, nz;
    uint32_t epi_mask;  // faces whose new boundary layer the epilogue stores to epi[f]
    int64_t pitch, zs;
    uint32_t pro_mask;  // faces whose ghost values the prologue patches from pro[f] with generic loads
    uint32_t pro_tma;   // faces whose ghost values the producer loads from pro[f] with TMA (strategy C)
    FaceRef epi[6];
    FaceRef pro[6];
};

// A unit of stencil work: one (TX x TY) tile of one block over planes [z0,z1).
struct WorkItem {
    int32_t blk;    // local block index (descriptor = 2*blk + parity)
    int16_t tx, ty; // tile coordinates
    int32_t z0, z1;
};

// Multi-iteration (persistent) stencil launches, J3D_PERSISTENT: launch item g
// is item (g mod n_items) of relative iteration k = g / n_items.  A slab is
// one row of tiles (all tx) of one block over one z chunk; done[s] counts
// consumer-warp completions of slab s (mod 2^32, never reset).  An item of
// iteration k > 0 may start once every slab in slab_deps[item_slab[i]] -- the
// slabs whose iteration-k-1 writes it reads (own slab, the adjacent chunks
// and tile rows, the x neighbours' same slab, the y / z neighbours' edge
// slab; setup.cu build_persist_deps) and, by symmetry, those whose
// iteration-k-1 reads its writes would clobber -- has done >= (base+k)*target.
constexpr int MAX_DEPS = 12;
constexpr int32_t SLAB_PEER = 1 << 30;      // item_slab flag: the slab touches a peer GPU's face
constexpr int32_t SLAB_MASK = SLAB_PEER - 1;
struct IterCtl {
    const int32_t* item_slab;               // [n_items] slab index | SLAB_PEER
    const unsigned int* const* slab_deps;   // [n_slabs][MAX_DEPS] counters, null padded; bit 0 set: a peer's
    unsigned int* done;                     // [n_slabs]; nullptr: one iteration, no tracking
    int32_t n_iter;                         // iterations in this launch
    uint32_t target;                        // completions per slab per iteration (consumer warps x tiles per slab)
    uint32_t base;                          // iterations counted in done[] before this launch
    int32_t sys;                            // 1: some slabs wait on peer counters (iteration 0 waits too)
    uint64_t timeout_ns;                    // a counter wait longer than this traps (J3D_TIMEOUT_S)
};

// A strided 2D face copy (pack: owned layer -> send buffer / peer receive
// buffer; unpack: receive buffer -> ghost layer).  na == 0 marks an unused slot.
struct CopyDesc {
    FaceRef src;
    FaceRef dst;
    int32_t na, nb;
};

// Per-block geometry for init / checksum / residual.
struct BlockGeom {
    double* buf[2];
    int64_t ox, oy, oz;  // global origin of owned cell (0,0,0)
    int32_t nx, ny, nz, pad;
    int64_t pitch, zs;
    int64_t xg_off, xg_side, xg_pitch;  // x ghost arrays: buf + xg_off + side*xg_side (doubles)
};

}  // namespace j3d
