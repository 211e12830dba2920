// mrv_internal.h -- device scene layout shared by scene.cpp (host precompute) and
// kernels.cu (sm_100a).  Not part of the ABI.
//
// The scene is ONE contiguous blob (16-byte aligned sections) that every CTA
// stages into shared memory with a 1-D TMA bulk copy (cp.async.bulk) at kernel
// start.  All offsets below are byte offsets into the blob.
#pragma once
#include <stdint.h>

namespace mrv {

constexpr int kMaxGroupSpheres = 32;   // spheres per collision group (one warp round in the narrow phase)
constexpr int kMaxWarpsPerCta = 16;    // the launcher picks 1..16 warps per CTA (FFC: kMaxWarpsFfc) for the best residency
constexpr int kFfcWarpsFull = 18;      // FFC keeps no per-group bounds in smem: more, smaller warps fit (18 = its smem limit on cfg5; 20 measured 0.9 % slower)
constexpr int kMaxWarpsFfc = 20;       // FFC's launch bound: 20 warps (5 per SM sub-partition at 96 registers) where the lean instance stores compact link frames (kernels.cu frame_off)
constexpr int kQueueCap = 256;         // narrow-phase queue entries per warp (flushed before it can overflow)
constexpr int kFrameWords = 9;         // stored link frame: rotation columns 0, 1 and translation
constexpr int kSuperMax = 3;           // groups per supergroup (first-level robot-robot bound)
constexpr int kNarrowCap = 128;        // second-level survivors (group pairs) queued for the sphere tests
constexpr int kSegLen = 8;             // candidates per broad-phase segment
constexpr int kRRSegLen = 5;           // candidates per robot-robot level-1 segment (unrolled tests per lane)
static_assert(kQueueCap >= 32 * kSegLen, "one broad-phase iteration must fit an empty queue");
constexpr int kWpCapFloats = 2048;     // motion waypoint block staged in smem if it fits (8 KB)
constexpr float kBoundEps = 1e-4f;     // broad-phase inflation

// Packed table records (see scene.cpp for how they are filled).
//   robot  int4 A: {kind, dof, link_begin, n_links}
//          int4 B: {group_begin, n_groups, sphere_begin, n_spheres}
//          int4 C: {super_begin, n_super, fast_dh, 0}
//   super  int4:  {robot, group_begin, n_groups (<= kSuperMax), 0}: supergroup = consecutive groups
//   group_super int32 per group: its supergroup | 0x80000000 if it is the supergroup's last member
//          | 0x40000000 if it is the first
//   dhrec  3 x float4 per link (fast-DH robots): {a, cos alpha, sin alpha, d}, group bound,
//          {group, group_super code, 0, 0} as int bits
//   dhbase 3 x float4 per robot (fast-DH robots): base * Tz(d_0) Tx(a_0) Rx(alpha_0) rows,
//          so that the chain walk's first joint is Rz(q_0) alone
//          float4 x3: base rows (3x4), identity for SE2/SE3
//   link   int4:  {robot, joint_type | dh_form << 1, group_begin, n_groups}
//          float4 x3: joint origin O_j rows (3x4)
//   group  int4:  {link, sphere_begin, n_spheres, robot}
//          float4: {cx, cy, cz, R} local bounding sphere (R inflated)
//   sphere float4: {ox, oy, oz, r} in group order
//   obs    float4 x2 per obstacle: {lo, r}, {hi, 0} -- sphere obstacles (lo = hi = centre,
//          rounding radius r) first, then boxes (r = 0)
//   grid   2 x float4: {origin xyz, 1/h}, {nx, ny, nz, 0 as int bits}; cell_start uint16
//          [cells + 1], cell_list uint16 [entries]: obstacles within Rmax + eps of each
//          cell (Rmax = the largest group bound), cells x-fastest
//   self segments (4 x uint4 = 64 B): {hdr, 0, 0, 0}, {8 x uint16 candidate group},
//          {8 x float (R_a + R_k)^2 of the inflated bounds, rounded up}; hdr = group a |
//          (count << 16): group a vs the groups of its link's self-collision partners
//   rr segments (2 x uint4 = 32 B): {supergroup a | count << 16, rank_min, c0, c1},
//          {c2, c3, c4, 0}: a vs <= kRRSegLen supergroups of other robots (pairs owned
//          by either end, balanced); supergroup bounds are derived per state
//   link_off[4][n_links]: per-W (4, 8, 16, 32) smem word offset of each link's
//          frame block inside the per-warp frame area (bank-staggered by robot)
//   gcap   2 x float4 per group: {p0, rc}, {p1, 1}: a capsule (segment p0-p1 in the link
//          frame, radius rc, inflated like the bound) holding every sphere of the group;
//          {centre, R}, {centre, 0} (the bound sphere, flag 0) when a capsule is not tighter
//   sphere_index: int32 per sphere (group order) -> scene order index
struct DevScene {
  int32_t n_robots, n_links, n_groups, n_spheres;
  int32_t n_osph, n_box, n_cells, n_cell_entries;   // obstacle grid: cells, total list entries
  int32_t n_rr_items, n_pairs, max_link_per_robot, rr_seg_len;   // rr_seg_len: candidates per rr segment (<= kSegLen)
  int32_t fixed_layout, use_caps, n_rr_segs, n_super;   // fixed_layout: FixedLayout prefix (see below); use_caps:
                                                        // some group's capsule is tighter than its bound sphere
  int32_t n_self_segs, n_self_items, group_lg, rr_prefix_bytes;   // group_lg: log2 of the common group size if every
                                                        // group has the same power-of-two sphere count, else -1;
                                                        // rr_prefix_bytes: the blob prefix FFC reads (robots, links,
                                                        // groups, spheres, supergroups, rr segments, frame offsets)
  int32_t frame_words[4];      // per-W frame area size (words) incl. bank staggering
  uint32_t blob_bytes;
  uint32_t off_robot, off_link, off_group, off_gbound, off_sphere;
  uint32_t off_obs, off_grid, off_cell_start, off_cell_list, off_rr_segs, off_link_off, off_sphere_index;
  uint32_t off_robot_base, off_link_origin, off_super, off_group_super, off_self_segs, off_dhrec, off_gcap;
  uint32_t off_dhbase;
  uint32_t off_rr_segs_all;    // MRV_DIAG_NO_BROADPHASE: rr segments over every supergroup pair (no reach pruning)
  int32_t n_rr_segs_all;
  int32_t l1tile, l1tile_pad;  // l1tile bit 0: 4 robots x 3 supergroups (supergroup 3r + k): the tiled
                               // level 1; bit 1: fast-DH arms, group g = link g, x-axis group bounds;
                               // bit 2: sphere centres and capsule endpoints on the link x axes too
  uint64_t l1tile_masks;       // 15-bit pair mask of lane role r at bit 16 r
};

__host__ __device__ inline uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

// Fixed-offset layout of the FFC prefix, used when the scene fits these caps (cfg2/cfg5
// class teams): every table FFC reads then sits at a compile-time offset of the staged
// blob, so the W = 8 FFC kernel addresses them as immediates instead of re-deriving
// per-launch table pointers (ds.fixed_layout = 1; link_off rows are kFixLinks apart).
struct FixedLayout {
  static constexpr int kRobots = 4, kLinks = 32, kGroups = 32, kSpheres = 256, kRRSegs = 16, kSuper = 16;
  static constexpr uint32_t robot = 0;
  static constexpr uint32_t robot_base = robot + kRobots * 48;
  static constexpr uint32_t link = robot_base + kRobots * 48;
  static constexpr uint32_t link_origin = link + kLinks * 16;
  static constexpr uint32_t group = link_origin + kLinks * 48;
  static constexpr uint32_t gbound = group + kGroups * 16;
  static constexpr uint32_t sphere = gbound + kGroups * 16;
  static constexpr uint32_t rr_segs = sphere + kSpheres * 16;
  static constexpr uint32_t super = rr_segs + kRRSegs * 32;
  static constexpr uint32_t group_super = super + kSuper * 16;
  static constexpr uint32_t dhrec = group_super + kGroups * 4;
  static constexpr uint32_t dhbase = dhrec + kLinks * 48;
  static constexpr uint32_t link_off = dhbase + kRobots * 48;
  static constexpr uint32_t gcap = link_off + 4 * kLinks * 4;
  static constexpr uint32_t end = gcap + kGroups * 32;
};

}  // namespace mrv
