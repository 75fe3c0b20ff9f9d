// dev_types.h — plain-old-data tables shared by the host engine and the kernels.
#pragma once
#include <cstdint>

namespace mpmb {

enum : int {
    GEOM_PLANE = 0, GEOM_SPHERE = 1, GEOM_BOX = 2, GEOM_QUAD_SLICER = 3,
    GEOM_TRI_MESH_SLICER = 4, GEOM_ARC = 5, GEOM_POLYLINE = 6
};
enum : int { REGION_BULK = 0, REGION_SURFACE = 1, REGION_EDGE = 2, REGION_SPINE = 3, REGION_CURVE = 4 };
enum : int { MOTION_FIXED = 0, MOTION_KINEMATIC = 1, MOTION_FREE = 2 };
enum : int { BC_SLIP = 0, BC_STICKY = 1 };

// Particle slot flags (word 2 of the R plane).
constexpr uint32_t kActiveBit = 0x80000000u;
constexpr uint32_t kMatMask = 0xFFu;
constexpr int kSceneShift = 8;
constexpr uint32_t kSceneMask = 0x3FFFFFu;
// set at upload on a particle given inactive together with an explicit stress: the reference
// never updates an inactive particle's cached stress, so downloads return the uploaded value
constexpr uint32_t kKeepStressBit = 0x40000000u;

constexpr float kMassEps = 1e-9f;  // state.hpp:13
constexpr int kBrick = 4;          // nodes (and cells) per brick edge
constexpr int kBrickNodes = 64;

// Per-scene grid + shape range (one entry per scene of a batch).
struct DevScene {
    float origin[3];
    float dx;
    float inv_dx;      // 1.0f / dx, as the reference computes it (math.hpp:219)
    float m_inv;       // 4 / (dx*dx) (solvers.hpp:149)
    int dims[3];
    int nb[3];         // bricks per axis = ceil(dims / 4)
    uint64_t node_base;   // first node of this scene in the bricked node pool
    uint32_t brick_base;  // first brick of this scene in the global brick space
    int shape_begin;
    int shape_count;
    int pad;
};

// Grid geometry shared by every scene of an engine (one SceneConfig per batch): kernels
// read it from the parameter bank (constant cache), never per particle from memory.
// origin / dims are the GLOBAL grid (keys, node positions, BC, deactivation are the
// reference's arithmetic on global indices); the node STORAGE of a slab domain (slab
// decomposition) covers global x nodes [goff, goff + lx) in nb bricks.
struct Geo {
    float origin[3];
    float dx;
    float inv_dx;
    float m_inv;
    int dims[3];
    int nb[3];
    uint64_t nodes_per_scene;
    uint32_t bricks_per_scene;
    int goff;            // global x index of local node 0 (0 without a slab)
    int lx;              // local storage width in x (nodes)
    int own_lo, own_hi;  // local x range of the nodes this domain owns (contact sums)
    int pad;
};

constexpr int kMaxConstMats = 16;  // materials carried in the kernel parameter bank

// Flattened mpm::Shape minus pose (rigid_dynamics.hpp:107-117, geometry.hpp:44-86).
struct DevShape {
    int geom;
    int motion;
    int vtx_begin, n_vtx;      // vertex pool (float3)
    int idx_begin, n_idx;      // int pool: triangle indices
    int spine_begin, n_spine;  // int pool: spine edge pairs
    float gp[4];
    float mu_k, c_d, hw, body_mass;
    float inertia[3];
    int scene;
    // local-frame box (center, half extents) outside which the shape can neither contact a
    // node nor push a particle (every region's band included, conservative margin);
    // lbox_h[0] < 0 for unbounded shapes (plane).  A cull, never a change of result.
    float lbox_c[3];
    float lbox_h[3];
};

// mpm::ShapePose (geometry.hpp:14-27), padded to 64 B.
struct DevPose {
    float pos[3];
    float rot[4];
    float lin[3];
    float ang[3];
    float pad[3];
};

}  // namespace mpmb
