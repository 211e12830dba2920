// kernels.cu -- sm_100a kernels of libmrv: batched multi-robot MotVal (K1), FFC (K2)
// and the SpheresFK export (K3), plus their C-ABI launchers.
//
// One fused persistent kernel per query (one CTA of up to 16 / 18 warps per SM).  Each
// warp pulls motions from a global work counter and walks the motion's timesteps in
// batches of W states (W = 8 by default: the paper's SIMD batch B_i, PAPER.md:246;
// compile-time W = 8 instance) -- MotVal's production launch instead fills its batch
// from up to 8 motions, one state each, in a golden-ratio timestep order (run_spread,
// DESIGN.md reading c.28).  Per batch:
//   1. interpolate every robot's configuration at the batch's W timesteps
//      (rake order for MotVal; linear for FFC)
//      and run SpheresFK: lanes = (robot, state) pairs; link frames
//      and supergroup world bounds (Ritter-merged group bounds) go to the warp's smem;
//   2. CC(S_i, E) (MotVal): group bounds against a uniform obstacle grid
//      -- fused into the FK lanes for fast-DH teams (fk_env_fused), else a separate
//      pass -- then sphere-vs-obstacle narrow phase on the survivors;
//   3. CC(S_i, S_j): supergroup pairs (level 1, lanes = (segment,
//      state), balanced 5-candidate segments; for 4-robot x 3-supergroup teams at W = 8
//      the tiled level 1, lanes = the FK lanes (robot, state), rr_stage_tile) -> group
//      pairs (level 2) -> a capsule
//      prefilter (certified segment-distance lower bound) -> sphere pairs (narrow
//      phase: lanes = spheres of one group, the other group's world centres in a
//      per-warp scratch); survivors are compacted into smem queues by ballots;
//   4. reduction: MotVal -- any hit ends the motion (early termination,
//      PAPER.md:298, :310, :320); FFC -- per-state keys t*P + rank reduced with
//      a warp min; a batch that contains a conflict is the last one
//      (PAPER.md:361-363); with several warps per motion an atomicMin on the
//      per-motion key lets later batches skip.
// All geometry is fp32; all indices, keys and flags are integers.
// describe the layouts and the measured trade-offs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/mrv.h"
#include "mrv_internal.h"
#include "scene_impl.h"

// Opt-in bounds checking (compute-sanitizer is unavailable on the GPU pool): build
// with -DMRV_DEBUG_BOUNDS to trap on any out-of-range queue / table / smem index.
#ifdef MRV_DEBUG_BOUNDS
#include <cstdio>
#define MRV_CHECK(cond)                                                        \
  do {                                                                         \
    if (!(cond)) {                                                             \
      printf("MRV_CHECK failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);     \
      __trap();                                                                \
    }                                                                          \
  } while (0)
#else
#define MRV_CHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace mrv {

enum { Q_MOTVAL = 0, Q_FFC = 1 };
// per-warp queue capacities: FFC's level 1 adds at most 32 x kRRSegLen survivors per
// iteration and its level 2 few group pairs, so its queues are smaller (more warps fit)
template <int QUERY>
constexpr int kQCap = QUERY == Q_FFC ? 32 * kRRSegLen : kQueueCap;
template <int QUERY>
constexpr int kNCap = kNarrowCap;
// MotVal spread packing's queues (run_spread): one level-1 round, and 120 group pairs
constexpr int kSpreadQCap = 32 * kRRSegLen, kSpreadNCap = 120;
static_assert(kSpreadQCap >= 32 * 4 && kSpreadQCap >= 32 + 32, "an obstacle round fits the spread queue");
// Per-group world bounds per state are kept in smem (w.bc) only where a broad phase
// reads them many times: MotVal's separate obstacle / self stages.  FFC and the fused
// MotVal path (fk_env_fused) need them only in the second robot-robot level for the few
// surviving supergroup pairs and derive them from the link frames there (w.bc == null),
// which frees 16 B x W per group of per-warp scratch (more resident warps).
constexpr unsigned FULL = 0xFFFFFFFFu;

constexpr int kPPSegs = 64;   // PP-ST-RRT: most (focus, partner) level-1 segments of a launch

struct KParams {
  DevScene sc;
  const uint8_t* blob;
  const float* wp;
  const int32_t* Tm;
  const int32_t* Trob;       // [M][n] per-robot lengths or null
  int64_t M;
  int32_t Tfix, K, S, nKS;
  uint32_t flags;
  int32_t lgW, W, wi;
  int32_t n_slices, grab;
  uint8_t* out_valid;
  uint32_t* out_key;
  unsigned long long* work;
  unsigned long long* counters;
  uint32_t* effort;
  uint32_t* dev_status;       // the scene's device status word (MRV_DEVERR_* bits, atomicOr)
  uint32_t warp_bytes, off_frames, off_bc, off_sbc, off_queue, off_nq, off_nsc, off_wp;
  uint32_t stage_bytes;       // blob bytes staged into smem (FFC: the rr prefix)
  int32_t wp_in_smem;
  int32_t fuse_env;           // MotVal: obstacle broad phase fused into the FK lanes (fk_env_fused)
  int32_t t_begin, t_end;    // time window (t_end <= 0: T)
  int32_t focus;             // PP-ST-RRT variant: focus robot, -1 = all robots
  unsigned long long partners;
  // PP-ST-RRT with shared fixed partner paths (mrv_pp_motval_batch): the partners' geometry
  // comes from a per-timestep table instead of FK; null otherwise
  const float4* pp_table;
  const int32_t* pp_t0;      // [M] absolute start timestep of each candidate
  int32_t pp_H, pp_rec;      // table rows (horizon) and float4s per row
  int32_t pp_fbase, pp_gbase;   // link_off of the focus robot's first link at this W; its first group
  int32_t pp_nseg;           // > 0: level-1 segments of the (focus, partner) supergroup pairs only,
  const uint32_t* pp_segs;   //   DEVICE [pp_nseg][8] in the rr segment record format (copied to smem)
  // MotVal spread packing (run_spread): a warp's W state slots are shared by up to W motions,
  // each walking its timesteps in the order t_b = (T / 2 + b * step) mod T
  int32_t spread;
  int32_t sp_slots;          // motions a warp keeps in flight (<= W; fewer for small batches)
  uint32_t sp_step;          // step of a fixed T (per-motion T: spread_step on the device)
  // MotVal queue capacities (entries) of this launch's per-warp layout: broad-phase survivors
  // (>= 32 * kRRSegLen; kQueueCap with self-collision segments) and group pairs (<= kNarrowCap)
  int32_t qcap, ncap;
};

// queue capacities of a launch: FFC's are compile-time, MotVal's follow its layout
template <int QUERY>
__device__ __forceinline__ int qcap(const KParams& p) { return QUERY == Q_FFC ? kQCap<Q_FFC> : p.qcap; }
template <int QUERY>
__device__ __forceinline__ int ncap(const KParams& p) { return QUERY == Q_FFC ? kNCap<Q_FFC> : p.ncap; }

// ------------------------------------------------------------------ scene view
struct SV {
  const int4* robot;       // 3 records per robot
  const float4* robot_base;
  const int4* super;
  const int32_t* group_super;   // supergroup of each group, sign bit = last member
  const float4* dhrec;          // fast-DH per-link records (3 x float4)
  const float4* dhbase;         // fast-DH robots: base * (link 0's fixed DH part), 3 x float4
  const int4* link;
  const float4* link_origin;
  const int4* group;
  const float4* gbound;
  const float4* sphere;
  const float4* obs;          // 2 x float4 per obstacle: {lo, r}, {hi, 0}
  const float4* grid;         // {origin, 1/h}, {nx, ny, nz} (int bits)
  const uint16_t* cell_start;
  const uint16_t* cell_list;
  const uint4* rr_segs;
  const uint4* self_segs;
  const int32_t* link_off;
  const int32_t* sphere_index;
  const float4* gcap;         // 2 x float4 per group: capsule {p0, rc}, {p1, flag} in the link frame
};

// b: the staged prefix (tables every query reads); t: where the tail tables live (the
// obstacles, grid, self segments, unpruned robot-robot segments): the same smem copy when
// the whole blob was staged, else the blob in global memory (MotVal scenes whose obstacle
// tables would crowd out the per-warp scratch).  Offsets are blob offsets either way.
__device__ __forceinline__ SV make_sv(const uint8_t* b, const uint8_t* t, const DevScene& d, int wi) {
  SV v;
  v.robot = reinterpret_cast<const int4*>(b + d.off_robot);
  v.super = reinterpret_cast<const int4*>(b + d.off_super);
  v.group_super = reinterpret_cast<const int32_t*>(b + d.off_group_super);
  v.dhrec = reinterpret_cast<const float4*>(b + d.off_dhrec);
  v.dhbase = reinterpret_cast<const float4*>(b + d.off_dhbase);
  v.robot_base = reinterpret_cast<const float4*>(b + d.off_robot_base);
  v.link = reinterpret_cast<const int4*>(b + d.off_link);
  v.link_origin = reinterpret_cast<const float4*>(b + d.off_link_origin);
  v.group = reinterpret_cast<const int4*>(b + d.off_group);
  v.gbound = reinterpret_cast<const float4*>(b + d.off_gbound);
  v.sphere = reinterpret_cast<const float4*>(b + d.off_sphere);
  v.obs = reinterpret_cast<const float4*>(t + d.off_obs);
  v.grid = reinterpret_cast<const float4*>(t + d.off_grid);
  v.cell_start = reinterpret_cast<const uint16_t*>(t + d.off_cell_start);
  v.cell_list = reinterpret_cast<const uint16_t*>(t + d.off_cell_list);
  v.rr_segs = reinterpret_cast<const uint4*>(b + d.off_rr_segs);
  v.self_segs = reinterpret_cast<const uint4*>(t + d.off_self_segs);
  v.link_off = reinterpret_cast<const int32_t*>(b + d.off_link_off) +
               (size_t)wi * (d.fixed_layout ? FixedLayout::kLinks : d.n_links);
  v.sphere_index = reinterpret_cast<const int32_t*>(t + d.off_sphere_index);
  v.gcap = reinterpret_cast<const float4*>(b + d.off_gcap);
  return v;
}

// The same view at FixedLayout's compile-time offsets (ds.fixed_layout): only the FFC
// prefix tables are valid (FFC never reads the obstacle / self sections).
template <bool FIXED>
__device__ __forceinline__ SV make_sv_q(const uint8_t* b, const uint8_t* t, const DevScene& d, int wi) {
  if (!FIXED) return make_sv(b, t, d, wi);
  typedef FixedLayout FL;
  SV v = make_sv(b, t, d, wi);   // obstacle / self / export tables keep their runtime offsets
  v.robot = reinterpret_cast<const int4*>(b + FL::robot);
  v.robot_base = reinterpret_cast<const float4*>(b + FL::robot_base);
  v.link = reinterpret_cast<const int4*>(b + FL::link);
  v.link_origin = reinterpret_cast<const float4*>(b + FL::link_origin);
  v.group = reinterpret_cast<const int4*>(b + FL::group);
  v.gbound = reinterpret_cast<const float4*>(b + FL::gbound);
  v.sphere = reinterpret_cast<const float4*>(b + FL::sphere);
  v.rr_segs = reinterpret_cast<const uint4*>(b + FL::rr_segs);
  v.super = reinterpret_cast<const int4*>(b + FL::super);
  v.group_super = reinterpret_cast<const int32_t*>(b + FL::group_super);
  v.dhrec = reinterpret_cast<const float4*>(b + FL::dhrec);
  v.dhbase = reinterpret_cast<const float4*>(b + FL::dhbase);
  v.link_off = reinterpret_cast<const int32_t*>(b + FL::link_off) + (size_t)wi * FL::kLinks;
  v.gcap = reinterpret_cast<const float4*>(b + FL::gcap);
  return v;
}

// ------------------------------------------------------------------ predicates (strict, reading c.1/c.2)
__device__ __forceinline__ bool sph_sph(float ax, float ay, float az, float ar, float4 b) {
  const float dx = ax - b.x, dy = ay - b.y, dz = az - b.z;
  const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  const float rs = ar + b.w;
  return d2 < rs * rs;
}

// sphere (c, r) vs obstacle {lo, r_o}, {hi, 0} (reading c.2): e_k = max(lo_k - c_k, 0,
// c_k - hi_k), hit iff sum e_k^2 < (r + r_o)^2.  For a sphere obstacle (lo = hi = o)
// e_k = |c_k - o_k| exactly, so this is sph_sph bit for bit; for a box (r_o = 0) it is
// the clamped-distance test.
__device__ __forceinline__ float d2_obs(float cx, float cy, float cz, float4 lo, float4 hi) {
  const float ex = fmaxf(fmaxf(lo.x - cx, cx - hi.x), 0.0f);
  const float ey = fmaxf(fmaxf(lo.y - cy, cy - hi.y), 0.0f);
  const float ez = fmaxf(fmaxf(lo.z - cz, cz - hi.z), 0.0f);
  return fmaf(ex, ex, fmaf(ey, ey, ez * ez));
}

__device__ __forceinline__ bool sph_obs(float cx, float cy, float cz, float r, float4 lo, float4 hi) {
  const float rs = r + lo.w;
  return d2_obs(cx, cy, cz, lo, hi) < rs * rs;
}

// squared centre distance (the broad phases compare it with (R_a + R_b)^2 of the
// inflated bounds: formed per test for robot-robot bounds, precomputed and rounded up
// in the self-collision segments)
__device__ __forceinline__ float d2_sph(float4 a, float4 b) {
  const float dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
  return fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}

// MUFU square root (~2 ulp): only used for supergroup radii, which carry a 1e-5 m pad
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// MUFU reciprocal (~1 ulp): only used for supergroup centres, covered by the same pad
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// c = M * o (M row-major 3x4)
__device__ __forceinline__ void xform(const float* M, float ox, float oy, float oz, float& x, float& y, float& z) {
  x = fmaf(M[0], ox, fmaf(M[1], oy, fmaf(M[2], oz, M[3])));
  y = fmaf(M[4], ox, fmaf(M[5], oy, fmaf(M[6], oz, M[7])));
  z = fmaf(M[8], ox, fmaf(M[9], oy, fmaf(M[10], oz, M[11])));
}

// ------------------------------------------------------------------ interpolation (reading c.4)
struct Interp {
  int seg, seg1;   // knot segment; seg1 = seg + 1, or seg itself at an exact knot (u = 0)
  float u;
  bool exact;
};

// t (K - 1) / (T - 1) for products beyond 32 bits, without the runtime's 64-bit division
// (a subroutine CALL: after it the compiler cannot prove the warp converged and wraps every
// later warp collective of the kernel in WARPSYNC ... ENDCOLLECTIVE -- +20 % code, −4 % on
// cfg3 / cfg4): the quotient is < K <= 2^20, so a float estimate is within a few units and
// exact 64-bit remainder corrections finish it.
__device__ __forceinline__ uint32_t knot_div64(uint64_t num, uint32_t den, float rd, int* rem) {
  uint32_t q = (uint32_t)((float)num * rd);
  int64_t r = (int64_t)(num - (uint64_t)q * den);
  while (r < 0) { --q; r += den; }
  while (r >= (int64_t)den) { ++q; r -= den; }
  *rem = (int)r;
  return q;
}

// WIDE = false: the launcher guarantees (T - 1)(K - 1) < 2^32 (the lean instance: fixed T)
template <bool WIDE = true>
__device__ __forceinline__ Interp interp_setup(int t, int T, int K) {
  Interp ip;
  if (T <= 1 || K <= 1) {
    ip.seg = 0; ip.seg1 = 0; ip.u = 0.0f; ip.exact = true;
    return ip;
  }
  const uint32_t den = (uint32_t)(T - 1);
  const float rd = rcp_approx((float)den);
  const uint64_t num64 = (uint64_t)(uint32_t)t * (uint64_t)(uint32_t)(K - 1);
  uint32_t seg;
  int rem;
  if (WIDE && (num64 >> 32)) {   // (T - 1)(K - 1) >= 2^32 (long horizons with many knots): exact 64-bit division
    seg = knot_div64(num64, den, rd, &rem);
  } else {
    const uint32_t num = (uint32_t)num64;
    // exact integer quotient from a float estimate: the quotient is <= K - 1 and the
    // estimate's relative error a few ulp, so it is off by at most one and
    // one correction each way fixes it (validate_batch: K <= MRV_MAX_KNOTS = 2^20); rem in uint32 arithmetic, its sign read as int32
    // (|rem| < 2 den < 2^31).  u = rem / den with the MUFU reciprocal (<= 2 ulp; rem = 0
    // still gives u = 0 exactly).
    seg = (uint32_t)((float)num * rd);
    rem = (int)(num - seg * den);
    if (rem < 0) { --seg; rem += (int)den; }
    if (rem >= (int)den) { ++seg; rem -= (int)den; }
  }
  ip.seg = (int)seg;
  ip.exact = rem == 0;
  ip.seg1 = ip.exact ? ip.seg : ip.seg + 1;
  ip.u = (float)rem * rd;
  return ip;
}

// branch-free: at an exact knot u = 0 and seg1 = seg, so the result is w0 bit for bit
__device__ __forceinline__ float lerp_dof(const float* wr, int S, const Interp& ip, int d) {
  const float w0 = wr[ip.seg * S + d];
  const float w1 = wr[ip.seg1 * S + d];
  return fmaf(ip.u, w1 - w0, w0);
}

// sin/cos of a joint angle: the MUFU approximations (abs error ~4e-7 for |q| <= 2 pi;
// 7 chained joints x 1.75 m lever stay < 5e-6 m, inside the 1e-5 m parity budget),
// the accurate libdevice path for larger angles.
// wrap = false: the caller knows |q| <= 3 (every waypoint of the motion is, and q is
// their convex combination), where k = 0 and r = q bit for bit, so the reduction is skipped.
__device__ __forceinline__ void fast_sincos(float q, float& sn, float& cs, bool wrap = true) {
  // Cody-Waite reduction by 2*pi (two-constant split; exact for |q| <= pi, where k = 0),
  // then the MUFU approximations (abs error ~4e-7 on [-pi, pi]; 7 chained joints x
  // 1.75 m lever stay < 5e-6 m, inside the 1e-5 m parity budget)
  float r = q;
  if (wrap) {
    const float k = rintf(q * 0.159154943f);
    r = fmaf(-k, -1.74845553e-7f, fmaf(-k, 6.28318548f, q));
  }
  __sincosf(r, &sn, &cs);
}

// sin(x) for x in [0, pi] (the slerp angles; with knots pre-aligned to dot >= 0, Omega
// <= pi/2): reflect to [0, pi/2] and evaluate the Taylor series to x^11 -- relative error
// <= 1.7e-7 on [0, pi/2] in fp32 (near 0 too, unlike the MUFU sine, whose absolute error
// would dominate sin(Omega) for nearly equal orientations).  Replaces the general sinf and
// its slow-path range reduction.
__device__ __forceinline__ float sin_0pi(float x) {
  const float y = fminf(x, 3.14159265f - x);
  const float p = y * y;
  float t = fmaf(p, -2.50521084e-8f, 2.75573192e-6f);
  t = fmaf(p, t, -1.98412698e-4f);
  t = fmaf(p, t, 8.33333333e-3f);
  t = fmaf(p, t, -1.66666667e-1f);
  return fmaf(y * p, t, y);
}

// atan2(a, b) for a, b >= 0 (the slerp half angle): z = min/max in [0, 1], atan(z) =
// pi/4 + atan((z - 1)/(z + 1)) above tan(pi/8), then the odd series to y^15 on
// |y| <= 0.4143 -- absolute error <= 1e-7 in fp32 (reading c.8's formula, fewer
// instructions than the general atan2f).  a = b = 0 gives 0.
__device__ __forceinline__ float atan2_pos(float a, float b) {
  const float mx = fmaxf(a, b), mn = fminf(a, b);
  const float z = mx > 0.0f ? mn * rcp_approx(mx) : 0.0f;
  const bool big = z > 0.41421356f;
  const float y = big ? (z - 1.0f) * rcp_approx(z + 1.0f) : z;
  const float p = y * y;
  float t = fmaf(p, -6.66666667e-2f, 7.69230769e-2f);
  t = fmaf(p, t, -9.09090909e-2f);
  t = fmaf(p, t, 1.11111111e-1f);
  t = fmaf(p, t, -1.42857143e-1f);
  t = fmaf(p, t, 2.0e-1f);
  t = fmaf(p, t, -3.33333333e-1f);
  float r = fmaf(y * p, t, y);
  if (big) r += 0.785398163f;
  return a > b ? 1.57079633f - r : r;
}

// SE(3) pose at the interpolated state: position lerp, quaternion slerp (reading c.8),
// R from q with s = 2 / (q.q).  Out of line (atan2f / sinf are large).
__device__ __forceinline__ void se3_pose(const float* wr, int S, const Interp& ip, float* M) {
  const float px = lerp_dof(wr, S, ip, 0), py = lerp_dof(wr, S, ip, 1), pz = lerp_dof(wr, S, ip, 2);
  float qw, qx, qy, qz;
  const float* w0 = wr + ip.seg * S;
  if (ip.exact) {
    qw = w0[3]; qx = w0[4]; qy = w0[5]; qz = w0[6];
  } else {
    const float* w1 = w0 + S;
    const float a0 = w0[3], a1 = w0[4], a2 = w0[5], a3 = w0[6];
    const float b0 = w1[3], b1 = w1[4], b2 = w1[5], b3 = w1[6];
    const float m0 = b0 - a0, m1 = b1 - a1, m2 = b2 - a2, m3 = b3 - a3;
    const float p0 = b0 + a0, p1 = b1 + a1, p2 = b2 + a2, p3 = b3 + a3;
    const float dm = fmaf(m0, m0, fmaf(m1, m1, fmaf(m2, m2, m3 * m3)));
    const float dp = fmaf(p0, p0, fmaf(p1, p1, fmaf(p2, p2, p3 * p3)));
    const float om = 2.0f * atan2_pos(sqrtf(dm), sqrtf(dp));
    const float so = sin_0pi(om);
    float ca, cb;
    if (so < 1e-6f) {
      ca = 1.0f - ip.u; cb = ip.u;
    } else {
      const float inv = rcp_approx(so);
      ca = sin_0pi((1.0f - ip.u) * om) * inv;
      cb = sin_0pi(ip.u * om) * inv;
    }
    qw = fmaf(ca, a0, cb * b0); qx = fmaf(ca, a1, cb * b1);
    qy = fmaf(ca, a2, cb * b2); qz = fmaf(ca, a3, cb * b3);
  }
  const float s = 2.0f * rcp_approx(fmaf(qw, qw, fmaf(qx, qx, fmaf(qy, qy, qz * qz))));
  M[0] = 1.0f - s * (qy * qy + qz * qz); M[1] = s * (qx * qy - qw * qz); M[2] = s * (qx * qz + qw * qy); M[3] = px;
  M[4] = s * (qx * qy + qw * qz); M[5] = 1.0f - s * (qx * qx + qz * qz); M[6] = s * (qy * qz - qw * qx); M[7] = py;
  M[8] = s * (qx * qz - qw * qy); M[9] = s * (qy * qz + qw * qx); M[10] = 1.0f - s * (qx * qx + qy * qy); M[11] = pz;
}

// ------------------------------------------------------------------ SpheresFK (reading c.9)
// Calls sink(link, M) for every link frame of robot r (M: row-major 3x4 world<-link).
template <class Sink>
__device__ __forceinline__ void robot_fk(const SV& sv, int r, const Interp& ip, const float* wr, int S, Sink& sink) {
  const int4 ra = sv.robot[3 * r];
  const int kind = ra.x, dof = ra.y, lb = ra.z;
  float M[12];
  if (kind == MRV_CHAIN) {
    {
      const float4 b0 = sv.robot_base[3 * r], b1 = sv.robot_base[3 * r + 1], b2 = sv.robot_base[3 * r + 2];
      M[0] = b0.x; M[1] = b0.y; M[2] = b0.z; M[3] = b0.w;
      M[4] = b1.x; M[5] = b1.y; M[6] = b1.z; M[7] = b1.w;
      M[8] = b2.x; M[9] = b2.y; M[10] = b2.z; M[11] = b2.w;
    }
    for (int j = 0; j < dof; ++j) {
      const int link = lb + j;
      const float4 o0 = sv.link_origin[3 * link], o1 = sv.link_origin[3 * link + 1], o2 = sv.link_origin[3 * link + 2];
      const float q = lerp_dof(wr, S, ip, j);
      const int lt = sv.link[link].y;   // joint_type | dh_form << 1
      float A[12];
      if (lt & 2) {  // O = Tz(d) Tx(a) Rx(alpha): a = o0.w, c = o1.y, s = o2.y, d = o2.w
        const float ca = o1.y, sa = o2.y, ta = o0.w, td = o2.w;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const float m0 = M[4 * i], m1 = M[4 * i + 1], m2 = M[4 * i + 2], m3 = M[4 * i + 3];
          A[4 * i + 0] = m0;
          A[4 * i + 1] = fmaf(m1, ca, m2 * sa);
          A[4 * i + 2] = fmaf(m2, ca, -(m1 * sa));
          A[4 * i + 3] = fmaf(m0, ta, fmaf(m2, td, m3));
        }
      } else {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const float m0 = M[4 * i], m1 = M[4 * i + 1], m2 = M[4 * i + 2], m3 = M[4 * i + 3];
          A[4 * i + 0] = fmaf(m0, o0.x, fmaf(m1, o1.x, m2 * o2.x));
          A[4 * i + 1] = fmaf(m0, o0.y, fmaf(m1, o1.y, m2 * o2.y));
          A[4 * i + 2] = fmaf(m0, o0.z, fmaf(m1, o1.z, m2 * o2.z));
          A[4 * i + 3] = fmaf(m0, o0.w, fmaf(m1, o1.w, fmaf(m2, o2.w, m3)));
        }
      }
      if ((lt & 1) == 0) {  // revolute: A * Rz(q)
        float sn, cs;
        fast_sincos(q, sn, cs);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          M[4 * i + 0] = fmaf(cs, A[4 * i], sn * A[4 * i + 1]);
          M[4 * i + 1] = fmaf(cs, A[4 * i + 1], -sn * A[4 * i]);
          M[4 * i + 2] = A[4 * i + 2];
          M[4 * i + 3] = A[4 * i + 3];
        }
      } else {  // prismatic: A * Tz(q)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          M[4 * i + 0] = A[4 * i];
          M[4 * i + 1] = A[4 * i + 1];
          M[4 * i + 2] = A[4 * i + 2];
          M[4 * i + 3] = fmaf(q, A[4 * i + 2], A[4 * i + 3]);
        }
      }
      sink(link, M);
    }
  } else if (kind == MRV_SE2) {
    const float x = lerp_dof(wr, S, ip, 0), y = lerp_dof(wr, S, ip, 1), th = lerp_dof(wr, S, ip, 2);
    float sn, cs;
    fast_sincos(th, sn, cs);
    M[0] = cs; M[1] = -sn; M[2] = 0.0f; M[3] = x;
    M[4] = sn; M[5] = cs; M[6] = 0.0f; M[7] = y;
    M[8] = 0.0f; M[9] = 0.0f; M[10] = 1.0f; M[11] = 0.0f;
    sink(lb, M);
  } else {  // SE3: position lerp, quaternion slerp (reading c.8)
    se3_pose(wr, S, ip, M);
    sink(lb, M);
  }
}

// ------------------------------------------------------------------ per-warp state
struct Counters {
  unsigned long long v[MRV_NUM_COUNTERS];
};

struct Warp {
  float* frames;       // link blocks at link_off[l] (FrameSink layout)
  float4* bc;          // bc[g*W + s]: world bounding sphere of group g at state s
  float4* sbc;         // sbc[sg*W + s]: world bounding sphere of supergroup sg at state s
  uint32_t* queue;     // broad-phase survivors: s | k << 5 | segment << 8
  float4* nsc;         // narrow-phase scratch: 32 world sphere centres of the round's groups O
  uint2* nq;           // robot-robot group pairs for the sphere tests: {s | ga << 5, gb | rank << 16}
  const float* wp;     // motion waypoint block [n][K][S] (smem copy or global)
  const float* wp_smem;  // the smem copy (valid when p.wp_in_smem)
  bool wrap;             // some waypoint of the motion has |w| > 3: joint angles need range reduction
  int lane;
  int T, c, nb;
  int tb, te;          // evaluated timesteps [tb, te)
  const int32_t* Tr;   // this motion's per-robot lengths (global), or null
  int t0;              // PP table mode: the candidate's absolute start timestep
  bool rake;
  uint32_t amask;      // active states of the batch
  // spread packing: this lane's motion slot (its waypoints), timestep, and the batch slots
  // its motion owns
  const float* mwp;
  int mt, mT;          // (and its motion's T)
  uint32_t gmask;
  __device__ __forceinline__ int t_of(int s, int lgW) const { return rake ? c + s * nb : (c << lgW) + s; }
};

// Writes the link frame and the world bound of each of the link's groups, and grows
// each supergroup's bound incrementally (Ritter-style): adding ball (c, r) to (C, R)
// either leaves it unchanged (c inside) or replaces it by the smallest sphere holding
// both, R' = (R + |c - C| + r) / 2, C' = C + (R' - R) (c - C) / |c - C|.  Exact
// enclosure in exact arithmetic; padded by 1e-5 m + 1e-6 relative for fp32 rounding and
// the MUFU sqrt / reciprocal (each <= 2 ulp: < 1e-6 m over a supergroup's <= 2 merges)
// so the first level never culls what the second level keeps.  Branch-free: the first
// member meets R = -1e30 and is taken whole.
//
// Frame layout (per link block of 9W words at link_off[link], 16-B aligned):
//   [W x float4 {c0x, c0y, c0z, tx}] [W x float4 {c1x, c1y, c1z, ty}] [W x float tz]
// (rotation columns 0 and 1 and the translation; column 2 = c0 x c1 for proper rotations).
// Eight lanes of one robot store eight consecutive float4s: conflict-free 128-B wavefronts.
struct FrameSink {
  const SV* sv;
  float* frames;
  float4* bc;
  float4* sbc;
  int W, s;
  float cx, cy, cz, cr;
  __device__ __forceinline__ void reset() {
    cx = cy = cz = 0.0f;
    cr = -1e30f;
  }
  __device__ __forceinline__ void store_frame(int link, const float* M) {
    float* f = frames + sv->link_off[link];
    MRV_CHECK(link >= 0 && s >= 0 && s < W);
    reinterpret_cast<float4*>(f)[s] = make_float4(M[0], M[4], M[8], M[3]);
    reinterpret_cast<float4*>(f + 4 * W)[s] = make_float4(M[1], M[5], M[9], M[7]);
    f[8 * W + s] = M[11];
  }
  // world bound of group g (local bound gb) -> bc, grown into its supergroup's bound
  __device__ __forceinline__ void group(const float* M, float4 gb, int g, int gsup) {
    MRV_CHECK(g >= 0);
    group_at(bc + g * W + s, M, gb, gsup);
  }
  // (first / last membership is the same for every lane when the robots share a supergroup
  // partition -- identical arms -- so these branches are warp-uniform there)
  // XAXIS: the bound's centre is on the link's x axis (fast-DH robots, scene.cpp), placed
  // with column 0 and the translation alone (the same values xform gives for y = z = 0)
  template <bool XAXIS = false>
  __device__ __forceinline__ void group_at(float4* bcp, const float* M, float4 gb, int gsup) {
    float x, y, z;
    if (XAXIS) {
      x = fmaf(M[0], gb.x, M[3]);
      y = fmaf(M[4], gb.x, M[7]);
      z = fmaf(M[8], gb.x, M[11]);
    } else {
      xform(M, gb.x, gb.y, gb.z, x, y, z);
    }
    if (bc) *bcp = make_float4(x, y, z, gb.w);
    if (gsup & 0x40000000) {   // first member of its supergroup: taken whole
      cx = x; cy = y; cz = z; cr = gb.w;
    } else {
      const float dx = x - cx, dy = y - cy, dz = z - cz;
      const float d = sqrt_approx(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
      const bool contains = cr + d <= gb.w;        // the new ball holds the current sphere
      const bool grow = d + gb.w > cr;             // the new ball pokes out of the current sphere
      const float nr = 0.5f * (cr + d + gb.w);
      const float f = (nr - cr) * rcp_approx(d);   // d > 0 whenever grow && !contains
      const float gx = fmaf(f, dx, cx), gy = fmaf(f, dy, cy), gz = fmaf(f, dz, cz);
      cx = contains ? x : grow ? gx : cx;
      cy = contains ? y : grow ? gy : cy;
      cz = contains ? z : grow ? gz : cz;
      cr = contains ? gb.w : grow ? nr : cr;
    }
    if (gsup < 0)   // last member of its supergroup: sbc[sg * W + s] (the 32-bit byte offset drops the flag bits)
      *reinterpret_cast<float4*>(reinterpret_cast<char*>(sbc + s) + (uint32_t)gsup * (16u * (uint32_t)W)) =
          make_float4(cx, cy, cz, fmaf(cr, 1.0f + 1e-6f, 1e-5f));
  }
  __device__ __forceinline__ void operator()(int link, const float* M) {
    store_frame(link, M);
    const int4 L = sv->link[link];
    for (int g = L.z; g < L.z + L.w; ++g) group(M, sv->gbound[g], g, sv->group_super[g]);
  }
};

// link frame of (link block at word offset off, state s) -> row-major 3x4 F
__device__ __forceinline__ void load_frame(const float* frames, int off, int s, int W, float* F) {
  const float4 a = reinterpret_cast<const float4*>(frames + off)[s];
  const float4 b = reinterpret_cast<const float4*>(frames + off + 4 * W)[s];
  F[0] = a.x; F[4] = a.y; F[8] = a.z; F[3] = a.w;
  F[1] = b.x; F[5] = b.y; F[9] = b.z; F[7] = b.w;
  F[2] = fmaf(a.y, b.z, -a.z * b.y);
  F[6] = fmaf(a.z, b.x, -a.x * b.z);
  F[10] = fmaf(a.x, b.y, -a.y * b.x);
  F[11] = frames[off + 8 * W + s];
}

// point o of a link frame (block at word offset off, state s) -> world.  The third
// rotation column (c0 x c1) is only formed when o has a z component: sphere and bound
// offsets along the link's x-y plane (DH arms) skip the cross product.
__device__ __forceinline__ void xform_frame(const float* frames, int off, int s, int W, float ox, float oy, float oz,
                                            float& x, float& y, float& z) {
  const float4 a = reinterpret_cast<const float4*>(frames + off)[s];
  const float4 b = reinterpret_cast<const float4*>(frames + off + 4 * W)[s];
  const float tz = frames[off + 8 * W + s];
  x = fmaf(a.x, ox, fmaf(b.x, oy, a.w));
  y = fmaf(a.y, ox, fmaf(b.y, oy, b.w));
  z = fmaf(a.z, ox, fmaf(b.z, oy, tz));
  if (oz != 0.0f) {
    x = fmaf(fmaf(a.y, b.z, -a.z * b.y), oz, x);
    y = fmaf(fmaf(a.z, b.x, -a.x * b.z), oz, y);
    z = fmaf(fmaf(a.x, b.y, -a.y * b.x), oz, z);
  }
}

// ------------------------------------------------------------------ PP table mode accessors
// In the PP instance (mrv_pp_motval_batch) a warp's smem holds only the focus robot's link
// frames and group bounds; a partner's come from the partner table row of the state's
// absolute timestep t0 + t (held at the horizon's last row), streamed from L2/HBM.
__device__ __forceinline__ const float4* pp_row(const KParams& p, const Warp& w, int s) {
  int t = w.t_of(s, p.lgW);
  if (t >= w.T) t = w.T - 1;
  return p.pp_table + (size_t)min((int64_t)w.t0 + t, (int64_t)p.pp_H - 1) * p.pp_rec;
}

// rotation columns 0, 1 (+ translation x, y) and translation z of link `link` at state s
template <bool PP>
__device__ __forceinline__ void frame_cols(const KParams& p, const SV& sv, const Warp& w, int link, int s, float4& a,
                                           float4& b, float& tz) {
  if (PP && sv.link[link].x != p.focus) {
    if (p.counters) atomicAdd(p.counters + MRV_CNT_TABLE_BYTES, 48ull);   // (COUNT launches only)
    const float4* f = pp_row(p, w, s) + p.sc.n_super + 3 * link;
    a = __ldg(f);
    b = __ldg(f + 1);
    tz = __ldg(f + 2).x;
  } else {
    const int off = sv.link_off[link];
    a = reinterpret_cast<const float4*>(w.frames + off)[s];
    b = reinterpret_cast<const float4*>(w.frames + off + 4 * p.W)[s];
    tz = w.frames[off + 8 * p.W + s];
  }
}

template <bool PP>
__device__ __forceinline__ void load_frame_any(const KParams& p, const SV& sv, const Warp& w, int link, int s, float* F) {
  if (!PP) {
    load_frame(w.frames, sv.link_off[link], s, p.W, F);
    return;
  }
  float4 a, b;
  float tz;
  frame_cols<PP>(p, sv, w, link, s, a, b, tz);
  F[0] = a.x; F[4] = a.y; F[8] = a.z; F[3] = a.w;
  F[1] = b.x; F[5] = b.y; F[9] = b.z; F[7] = b.w;
  F[2] = fmaf(a.y, b.z, -a.z * b.y);
  F[6] = fmaf(a.z, b.x, -a.x * b.z);
  F[10] = fmaf(a.x, b.y, -a.y * b.x);
  F[11] = tz;
}

// world bound of group g at state s as stored by FK (smem bc) or the partner table
template <bool PP>
__device__ __forceinline__ float4 group_bound_any(const KParams& p, const SV& sv, const Warp& w, int g, int s) {
  if (PP && sv.group[g].w != p.focus) {
    if (p.counters) atomicAdd(p.counters + MRV_CNT_TABLE_BYTES, 16ull);   // (COUNT launches only)
    return __ldg(pp_row(p, w, s) + p.sc.n_super + 3 * p.sc.n_links + g);
  }
  return w.bc[(g << p.lgW) + s];
}

// world bounding sphere of group g at state s from its link frame (FFC: xform_frame;
// MotVal measured faster with the full frame load)
template <int QUERY>
__device__ __forceinline__ float4 group_world_bound(const SV& sv, const float* frames, int g, int s, int W) {
  const int4 G = sv.group[g];
  const float4 gb = sv.gbound[g];
  float x, y, z;
  if (QUERY == Q_FFC) {
    xform_frame(frames, sv.link_off[G.x], s, W, gb.x, gb.y, gb.z, x, y, z);
  } else {
    float F[12];
    load_frame(frames, sv.link_off[G.x], s, W, F);
    xform(F, gb.x, gb.y, gb.z, x, y, z);
  }
  return make_float4(x, y, z, gb.w);
}

// the same bound on a tiled-level-1 scene of fast-DH arms (ds.l1tile bit 1): group g is
// link g's only group, centred on the link's x axis -- the FK sink's 3-FMA placement
// (FrameSink::group_at<true>) from the stored column 0 and translation, bit for bit
// Compact link frames (FFC's lean instance on ds.l1tile bit-2 scenes, where every stored
// point lies on its link's x axis, so column 1 is never read): per link block of 6W words,
// [W x float4 {c0x, c0y, c0z, tx}] [W x float2 {ty, tz}], block l at word 6 W l.  Block
// offset and the translation's y, z in either layout:
__device__ __forceinline__ int frame_off(const SV& sv, int link, int W, bool cf) {
  return cf ? link * 6 * W : sv.link_off[link];
}
__device__ __forceinline__ float2 frame_tyz(const float* frames, int off, int s, int W, bool cf) {
  if (cf) return reinterpret_cast<const float2*>(frames + off + 4 * W)[s];
  return make_float2(frames[off + 4 * W + 4 * s + 3], frames[off + 8 * W + s]);
}

__device__ __forceinline__ float4 group_bound_xaxis(const SV& sv, const float* frames, int g, int s, int W, bool cf) {
  const int off = frame_off(sv, g, W, cf);
  const float4 gb = sv.gbound[g];
  const float4 a = reinterpret_cast<const float4*>(frames + off)[s];
  const float2 t = frame_tyz(frames, off, s, W, cf);
  return make_float4(fmaf(a.x, gb.x, a.w), fmaf(a.y, gb.x, t.x), fmaf(a.z, gb.x, t.y), gb.w);
}

// SpheresFK of a fast-DH robot (every joint revolute with a DH-form origin
// Tz(d) Tx(a) Rx(alpha), one collision group per link, links and groups consecutive):
// one packed record per link, no per-joint type branches (same arithmetic as
// robot_fk's DH path); frame and bound addresses advance by a constant stride.
// CF: compact link frames (frame_off / frame_tyz), the lean FFC instance on l1tile bit-2 scenes
template <int UNROLL, bool WRAP, bool CF = false>
__device__ __forceinline__ void robot_fk_dh(const SV& sv, int r, int lb, int dof, const Interp& ip, const float* wr,
                                            int S, FrameSink& sink) {
  float M[12];
  {   // base * Tz(d_0) Tx(a_0) Rx(alpha_0), folded on the host (sv.dhbase)
    const float4 b0 = sv.dhbase[3 * r], b1 = sv.dhbase[3 * r + 1], b2 = sv.dhbase[3 * r + 2];
    M[0] = b0.x; M[1] = b0.y; M[2] = b0.z; M[3] = b0.w;
    M[4] = b1.x; M[5] = b1.y; M[6] = b1.z; M[7] = b1.w;
    M[8] = b2.x; M[9] = b2.y; M[10] = b2.z; M[11] = b2.w;
  }
  const int W = sink.W, s = sink.s;
  constexpr int kStride = CF ? 6 : kFrameWords;   // words per link and state
  float* fp = sink.frames + frame_off(sv, lb, W, CF);
  float4* bp = sink.bc + sv.link[lb].z * W + s;
  const float4* rec = sv.dhrec + 3 * lb;
  const float* w0 = wr + ip.seg * S;    // the two knots' joint values (lerp_dof, with the
  const float* w1 = wr + ip.seg1 * S;   // addresses advanced per joint instead of re-derived)
  {   // joint 0: Rz(q_0) alone
    const float4 GB = rec[1];
    const int gsup = reinterpret_cast<const int*>(rec + 2)[1];
    const float q = fmaf(ip.u, *w1 - *w0, *w0);
    float sn, cs;
    fast_sincos(q, sn, cs, WRAP);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const float m0 = M[4 * i], a1 = M[4 * i + 1];
      M[4 * i + 0] = fmaf(cs, m0, sn * a1);
      M[4 * i + 1] = fmaf(cs, a1, -sn * m0);
    }
    reinterpret_cast<float4*>(fp)[s] = make_float4(M[0], M[4], M[8], M[3]);
    if (CF) {
      reinterpret_cast<float2*>(fp + 4 * W)[s] = make_float2(M[7], M[11]);
    } else {
      reinterpret_cast<float4*>(fp + 4 * W)[s] = make_float4(M[1], M[5], M[9], M[7]);
      fp[8 * W + s] = M[11];
    }
    sink.group_at<true>(bp, M, GB, gsup);
    fp += kStride * W;
    bp += W;
    rec += 3;
    ++w0;
    ++w1;
  }
#pragma unroll UNROLL
  for (int j = 1; j < dof; ++j, fp += kStride * W, bp += W, rec += 3, ++w0, ++w1) {
    const float4 P = rec[0], GB = rec[1];
    const int gsup = reinterpret_cast<const int*>(rec + 2)[1];
    const float q = fmaf(ip.u, *w1 - *w0, *w0);
    float sn, cs;
    fast_sincos(q, sn, cs, WRAP);
    const float ta = P.x, ca = P.y, sa = P.z, td = P.w;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const float m0 = M[4 * i], m1 = M[4 * i + 1], m2 = M[4 * i + 2], m3 = M[4 * i + 3];
      const float a1 = fmaf(m1, ca, m2 * sa);          // A = M * Tz(d) Tx(a) Rx(alpha)
      const float a2 = fmaf(m2, ca, -(m1 * sa));
      M[4 * i + 3] = fmaf(m0, ta, fmaf(m2, td, m3));
      M[4 * i + 0] = fmaf(cs, m0, sn * a1);             // M = A * Rz(q)
      M[4 * i + 1] = fmaf(cs, a1, -sn * m0);
      M[4 * i + 2] = a2;
    }
    reinterpret_cast<float4*>(fp)[s] = make_float4(M[0], M[4], M[8], M[3]);
    if (CF) {
      reinterpret_cast<float2*>(fp + 4 * W)[s] = make_float2(M[7], M[11]);
    } else {
      reinterpret_cast<float4*>(fp + 4 * W)[s] = make_float4(M[1], M[5], M[9], M[7]);
      fp[8 * W + s] = M[11];
    }
    sink.group_at<true>(bp, M, GB, gsup);
  }
}

// PP table mode: the focus robot's FK on lanes 0..W-1 (every FK lane busy at W = 32),
// then the partners' supergroup bounds at each state's absolute timestep t0 + t (held at
// the horizon's last row) from the table, lanes = (supergroup, state) -- level 1 needs
// nothing else; frames and group bounds are fetched only for surviving pairs (pp_fetch)
// the partners' supergroup rows of the batch's states, requested (cp.async, global -> smem,
// 16 B per item) before the focus robot's chain walk so the L2 / HBM latency of the table
// overlaps it; the caller waits (cp.async.wait_all) after the walk
template <bool COUNT>
__device__ __forceinline__ void pp_request_rows(const KParams& p, const SV& sv, Warp& w, Counters& cnt) {
  const int r = p.focus;
  for (int j = 0; j < p.sc.n_robots; ++j) {
    if (j == r || !((p.partners >> j) & 1ull)) continue;
    const int4 rc = sv.robot[3 * j + 2];
    const int items = rc.y << p.lgW;
    for (int i = w.lane; i < items; i += 32) {
      const int sg = rc.x + (i >> p.lgW), s = i & (p.W - 1);
      int t = w.t_of(s, p.lgW);
      if (t >= w.T) t = w.T - 1;
      const float4* src = p.pp_table + (size_t)min((int64_t)w.t0 + t, (int64_t)p.pp_H - 1) * p.pp_rec + sg;
      const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(w.sbc + sg * p.W + s));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
      if (COUNT && ((w.amask >> s) & 1u)) cnt.v[MRV_CNT_TABLE_BYTES] += 16;
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <bool COUNT>
__device__ __forceinline__ void fk_stage_pp(const KParams& p, const SV& sv, Warp& w, Counters& cnt) {
  const int r = p.focus;
  pp_request_rows<COUNT>(p, sv, w, cnt);
  for (int s = w.lane; s < p.W; s += 32) {
    int t = w.t_of(s, p.lgW);
    if (t >= w.T) t = w.T - 1;
    const Interp ip = interp_setup(t, w.T, p.K);
    FrameSink sink;
    sink.sv = &sv; sink.frames = w.frames; sink.sbc = w.sbc; sink.W = p.W; sink.s = s;
    sink.bc = w.bc;
    sink.reset();
    const int4 rc = sv.robot[3 * r + 2];
    if (rc.z && p.wp_in_smem) {   // fast-DH chain
      const int4 ra = sv.robot[3 * r];
      robot_fk_dh<1, true>(sv, r, ra.z, ra.y, ip, w.wp_smem, p.S, sink);
    } else if (p.wp_in_smem) {
      robot_fk(sv, r, ip, w.wp_smem, p.S, sink);
    } else {
      robot_fk(sv, r, ip, w.wp, p.S, sink);
    }
    if (COUNT && ((w.amask >> s) & 1u)) {
      const int4 ra = sv.robot[3 * r];
      cnt.v[MRV_CNT_SUPER_BOUNDS] += rc.y;
      cnt.v[MRV_CNT_ROBOT_STATES] += 1;
      if (ra.x == MRV_CHAIN) cnt.v[MRV_CNT_JOINTS] += ra.y;
      cnt.v[MRV_CNT_STATES] += 1;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");   // (the caller's __syncwarp publishes the rows)
}

template <int QUERY, bool COUNT, bool LEAN = false, bool PP = false>
__device__ __forceinline__ void fk_stage(const KParams& p, const SV& sv, Warp& w, Counters& cnt) {
  if (PP) {
    fk_stage_pp<COUNT>(p, sv, w, cnt);
    return;
  }
  const int total = p.sc.n_robots << p.lgW;
  for (int x = w.lane; x < total; x += 32) {
    const int r = x >> p.lgW, s = x & (p.W - 1);
    if (p.focus >= 0 && r != p.focus && !((p.partners >> r) & 1ull)) continue;   // ignored robot
    // robot r stays at its goal after its own path; spread packing: this
    // lane's state (s = lane % W at W = 8) belongs to the motion in slot w.mwp
    const int Tr = w.Tr ? w.Tr[r] : p.spread ? w.mT : w.T;
    int t = p.spread ? w.mt : w.t_of(s, p.lgW);
    if (t >= Tr) t = Tr - 1;
    const Interp ip = interp_setup<!LEAN>(t, Tr, p.K);
    const float* wsm = p.spread ? w.mwp : w.wp_smem;
    FrameSink sink;
    sink.sv = &sv; sink.frames = w.frames; sink.sbc = w.sbc; sink.W = p.W; sink.s = s;
    sink.bc = w.bc;
    sink.reset();
    const int4 rc = sv.robot[3 * r + 2];
    if (rc.z && p.wp_in_smem) {   // fast-DH chain
      const int4 ra = sv.robot[3 * r];
      // two joints per trip overlap one joint's bound with the next joint's chain; MotVal,
      // whose hot loop also holds the obstacle stage, measured faster without it
      // lean instance: motions whose waypoints all lie in [-3, 3] skip the angle range
      // reduction (a separate loop copy: a predicated reduction would still issue; the
      // general instances keep one copy -- the second cost cfg3's SE(3) loop 9 %)
      const float* wr = wsm + r * p.K * p.S;
      if (QUERY == Q_FFC && LEAN && (p.sc.l1tile & 4)) {   // compact frames (the launcher sized them)
        if (!w.wrap) robot_fk_dh<2, false, true>(sv, r, ra.z, ra.y, ip, wr, p.S, sink);
        else robot_fk_dh<2, true, true>(sv, r, ra.z, ra.y, ip, wr, p.S, sink);
      } else if (LEAN && !w.wrap) {
        robot_fk_dh<QUERY == Q_FFC ? 2 : 1, false>(sv, r, ra.z, ra.y, ip, wr, p.S, sink);
      } else {
        robot_fk_dh<QUERY == Q_FFC ? 2 : 1, true>(sv, r, ra.z, ra.y, ip, wr, p.S, sink);
      }
    } else if (p.wp_in_smem) {    // two inlined copies so the smem copy gets LDS addressing
      robot_fk(sv, r, ip, wsm + r * p.K * p.S, p.S, sink);
    } else {
      robot_fk(sv, r, ip, w.wp + (size_t)r * p.K * p.S, p.S, sink);
    }
    if (COUNT && ((w.amask >> s) & 1u)) cnt.v[MRV_CNT_SUPER_BOUNDS] += sv.robot[3 * r + 2].y;
    if (COUNT && ((w.amask >> s) & 1u)) {
      cnt.v[MRV_CNT_ROBOT_STATES] += 1;
      const int4 ra = sv.robot[3 * r];
      if (ra.x == MRV_CHAIN) cnt.v[MRV_CNT_JOINTS] += ra.y;
      if (r == (p.focus >= 0 ? p.focus : 0)) cnt.v[MRV_CNT_STATES] += 1;   // (the focus robot is always evaluated)
    }
  }
}

// lanes -> queue entries packing: entry sizes na (1..32); returns per-lane entry
// (index into [e0, e0+nfit)), the lane's offset inside the entry, lanes used, entries consumed
struct Pack {
  int my, k, used, nfit;
};

// every entry has 1 << lg lanes (the scene's groups all have the same power-of-two size):
// entry = lane >> lg, no scan
__device__ __forceinline__ Pack pack_uniform(int lane, int lg, int remaining) {
  Pack pk;
  const int per = 32 >> lg;
  pk.nfit = min(per, remaining);
  pk.used = pk.nfit << lg;
  pk.my = lane >> lg;
  pk.k = lane & ((1 << lg) - 1);
  return pk;
}

__device__ __forceinline__ Pack pack_round(int lane, bool valid, int na) {
  int incl = valid ? na : 64;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += v;
  }
  const int mine = valid ? na : 64;
  const bool fits = valid && incl <= 32;
  const unsigned fitm = __ballot_sync(FULL, fits);
  Pack pk;
  pk.nfit = __popc(fitm);
  const unsigned starts = __reduce_or_sync(FULL, fits ? (1u << (incl - mine)) : 0u);
  pk.used = __shfl_sync(FULL, incl, pk.nfit - 1);
  pk.my = __popc(starts & (FULL >> (31 - lane))) - 1;
  const int excl = __shfl_sync(FULL, incl - mine, pk.my < 0 ? 0 : pk.my);
  pk.k = lane - excl;
  return pk;
}

// ------------------------------------------------------------------ broad-phase segments
// A segment = one bound a (in registers) vs a short candidate list: robot-robot level 1
// (supergroup a vs <= kRRSegLen supergroups of other robots) and self-collision (group
// a vs <= kSegLen groups of its partner links).  Broad-phase lanes are (segment slot
// gi, state s), s = lane % W fixed for the whole stage, so the state's activity, t * P
// and bound row are loop invariants and a lane's tests are independent and branch-free
// (the latency-bound kernel needs that ILP).  Survivors are a per-lane bit mask,
// compacted into the warp's queue by per-bit ballots.  Queue entry: s | k << 5 |
// segment << 8.

__device__ __forceinline__ uint32_t seg_idx(const uint4& ix, int k) {
  const uint32_t w = k < 2 ? ix.x : k < 4 ? ix.y : k < 6 ? ix.z : ix.w;
  return (k & 1) ? (w >> 16) : (w & 0xFFFFu);
}

__device__ __forceinline__ uint32_t seg_idx_smem(const uint4* segs, int seg, int k) {
  return reinterpret_cast<const uint16_t*>(segs + 4 * seg + 1)[k];
}

// exclusive prefix of the per-lane survivor counts popc(bits) and their total, from one
// ballot per bit position present in the warp (survivors are sparse: usually one or two
// positions, each a VOTE + two POPC -- no dependent shuffle chain)
__device__ __forceinline__ int scan_bits(int lane, uint32_t bits, int& total) {
  const unsigned lt = (1u << lane) - 1u;
  unsigned present = __reduce_or_sync(FULL, bits);
  int excl = 0;
  total = 0;
  while (present) {
    const int k = __ffs(present) - 1;
    present &= present - 1u;
    const unsigned bal = __ballot_sync(FULL, (bits >> k) & 1u);
    excl += __popc(bal & lt);
    total += __popc(bal);
  }
  return excl;
}

__device__ __forceinline__ void enqueue_bits(Warp& w, uint32_t bits, int s, int seg, int& qn, int excl, int total) {
  int pos = qn + excl;
  MRV_CHECK(qn + total <= kQueueCap && seg >= 0 && seg < (1 << 24));
  while (bits) {
    const int k = __ffs(bits) - 1;
    bits &= bits - 1u;
    w.queue[pos++] = (uint32_t)s | ((uint32_t)k << 5) | ((uint32_t)seg << 8);
  }
  qn += total;
}


// MotVal (warp-uniform `hits`): may the batch stop?  Any hit ends a one-motion batch;
// under spread packing, only a hit for every motion that has states in the batch.
__device__ __forceinline__ uint32_t dead_states(const Warp& w, uint32_t hits) {
  return __reduce_or_sync(FULL, (hits & w.gmask) ? w.gmask : 0u);
}

__device__ __forceinline__ bool mv_done(const KParams& p, const Warp& w, uint32_t hits) {
  if (!p.spread) return hits != 0;
  return hits != 0 && (w.amask & ~dead_states(w, hits)) == 0;
}

// ------------------------------------------------------------------ robot-obstacle: CC(S_i, E)
// Env queue entry: s | group << 5 | cell-list position << 16 (the obstacle is
// cell_list[position]); needs n_groups < 2048 (checked at scene creation).  Returns
// nonzero on a hit: under spread packing the mask of the batch states with a hit.
template <bool COUNT>
__device__ uint32_t flush_env(const KParams& p, const SV& sv, Warp& w, int qn, Counters& cnt) {
  bool hit = false;
  uint32_t hs = 0;
  const int glg = p.sc.group_lg;
  for (int e0 = 0; e0 < qn;) {
    Pack pk;
    uint32_t ment;
    int gl, gs;
    if (glg >= 0) {   // uniform group size: each lane reads its own entry (broadcast LDS)
      pk = pack_uniform(w.lane, glg, qn - e0);
      ment = w.queue[min(e0 + pk.my, qn - 1)];
      const int4 G = sv.group[(ment >> 5) & 0x7FFu];
      gl = G.x;
      gs = G.y;
    } else {
      const int e = e0 + w.lane;
      const bool valid = e < qn;
      uint32_t ent = 0;
      int na = 1;
      int4 G = make_int4(0, 0, 0, 0);
      if (valid) {
        ent = w.queue[e];
        MRV_CHECK(e < kQueueCap && (int)((ent >> 5) & 0x7FFu) < p.sc.n_groups);
        G = sv.group[(ent >> 5) & 0x7FFu];
        MRV_CHECK(G.z >= 1 && G.z <= 32);
        na = G.z;
      }
      pk = pack_round(w.lane, valid, na);
      ment = __shfl_sync(FULL, ent, pk.my);
      gl = __shfl_sync(FULL, G.x, pk.my);
      gs = __shfl_sync(FULL, G.y, pk.my);
    }
    if (w.lane < pk.used) {
      const int s = ment & 31;
      // queue entries carry a cell-list position, or the obstacle itself without the grid
      const bool nobp = (p.flags & MRV_DIAG_NO_BROADPHASE) != 0;
      MRV_CHECK(nobp || (int)(ment >> 16) < p.sc.n_cell_entries);
      const uint32_t o = nobp ? (ment >> 16) : sv.cell_list[ment >> 16];
      MRV_CHECK((int)o < p.sc.n_osph + p.sc.n_box);
      float F[12];
      load_frame(w.frames, sv.link_off[gl], s, p.W, F);
      const float4 sp = sv.sphere[gs + pk.k];
      float x, y, z;
      xform(F, sp.x, sp.y, sp.z, x, y, z);
      const bool h = sph_obs(x, y, z, sp.w, sv.obs[2 * o], sv.obs[2 * o + 1]);
      hit |= h;
      hs |= h ? 1u << s : 0u;
      if (COUNT) {
        cnt.v[MRV_CNT_ENV_NARROW] += 1;
        cnt.v[MRV_CNT_SPHERE_XFORM] += 1;
      }
    }
    e0 += pk.nfit;
  }
  return p.spread ? __reduce_or_sync(FULL, hs) : (uint32_t)__any_sync(FULL, hit);
}

// Broad phase of CC(S_i, E) on the obstacle grid: lanes = (group,
// state); each lane finds its bound centre's cell and tests the bound against the cell's
// list, four candidates per trip (independent tests), until every lane's list is done;
// survivors go to w.queue (flushed to the narrow phase when it could overflow).
template <bool COUNT>
__device__ __forceinline__ bool env_grid_pass(const KParams& p, const SV& sv, Warp& w, bool stop_on_hit, int& qn,
                                              uint32_t& any, Counters& cnt) {
  if (p.sc.n_cells == 0) return false;
  const bool nobp = (p.flags & MRV_DIAG_NO_BROADPHASE) != 0;
  const float4 g0 = sv.grid[0];
  const int4 gn = *reinterpret_cast<const int4*>(sv.grid + 1);
  int x_lo = 0, total = p.sc.n_groups << p.lgW;
  if (p.focus >= 0) {   // PP-ST-RRT variant: only the focus robot's groups
    const int4 rb = sv.robot[3 * p.focus + 1];
    x_lo = rb.x << p.lgW;
    total = (rb.x + rb.y) << p.lgW;
  }
  for (int x0 = x_lo; x0 < total; x0 += 32) {
    const int x = x0 + w.lane;
    const int g = x >> p.lgW, s = x & (p.W - 1);
    int beg = 0, cnt_o = 0;
    float4 A = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    if (x < total && ((w.amask >> s) & 1u) && (p.focus < 0 || sv.group[g].w == p.focus)) {
      A = w.bc[x];   // bc[g * W + s]
      if (nobp) {   // diagnostic: no grid either -- every obstacle is a candidate
        cnt_o = p.sc.n_osph + p.sc.n_box;
      } else {
        const float fx = (A.x - g0.x) * g0.w, fy = (A.y - g0.y) * g0.w, fz = (A.z - g0.z) * g0.w;
        const int ix = (int)floorf(fx), iy = (int)floorf(fy), iz = (int)floorf(fz);
        if (ix >= 0 && iy >= 0 && iz >= 0 && ix < gn.x && iy < gn.y && iz < gn.z) {   // else: no obstacle within Rmax
          const int c = (iz * gn.y + iy) * gn.x + ix;
          beg = sv.cell_start[c];
          cnt_o = (int)sv.cell_start[c + 1] - beg;
        }
      }
    }
    for (int i0 = 0; __any_sync(FULL, i0 < cnt_o); i0 += 4) {
      uint32_t bits = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool v = i0 + u < cnt_o;
        const uint32_t o = nobp ? (uint32_t)(v ? i0 + u : 0) : sv.cell_list[v ? beg + i0 + u : 0];
        const float4 lo = sv.obs[2 * o], hi = sv.obs[2 * o + 1];
        const float rs = A.w + lo.w;
        const bool t = nobp || d2_obs(A.x, A.y, A.z, lo, hi) < rs * rs;
        bits |= (v && t ? 1u : 0u) << u;
      }
      if (COUNT) cnt.v[MRV_CNT_ENV_BROAD] += (uint64_t)max(0, min(4, cnt_o - i0));
      if (__any_sync(FULL, bits != 0u)) {
        int tot;
        const int excl = scan_bits(w.lane, bits, tot);
        if (qn + tot > p.qcap) {   // tot <= 32 * 4 <= p.qcap
          __syncwarp();
          any |= flush_env<COUNT>(p, sv, w, qn, cnt);
          qn = 0;
          __syncwarp();
          if (stop_on_hit && mv_done(p, w, any)) return true;   // (spread: every motion has a hit)
        }
        int pos = qn + excl;
        MRV_CHECK(qn + tot <= p.qcap);
        while (bits) {
          const int u = __ffs(bits) - 1;
          bits &= bits - 1u;
          w.queue[pos++] = (uint32_t)s | ((uint32_t)g << 5) | ((uint32_t)(beg + i0 + u) << 16);
        }
        qn += tot;
      }
    }
  }
  return false;
}

// ------------------------------------------------------------------ robot-robot: CC(S_i, S_j)
// Level 1: supergroup pairs (segments over sbc) -> w.queue.  Level 2: each surviving
// supergroup pair expands to its <= 9 group pairs (lanes packed by a warp scan),
// tested on the group bounds -> w.nq.  Level 3: sphere tests of surviving group pairs.
// MotVal: hit flag (0/1); FFC: minimum key t*P + rank (NONE if no hit).

// Capsule prefilter of a group pair (ga, gb) at state s: false only if the two groups'
// capsules (sv.gcap, each holding all of its group's spheres with the bound's inflation)
// are certainly disjoint.  Closest points (s~, t~) of the two world segments by one
// clamped alternation (Ericson's segment-segment step; any (s~, t~) in [0,1]^2 is
// acceptable), then a certificate that does not trust them: h(s,t) = |P(s) - Q(t)|^2 is
// a convex quadratic, so for the minimiser x* in the unit square
//   h(x*) >= h(x~) + grad h(x~) . (x* - x~) >= h(x~) + sum_i min(-g_i x~_i, g_i (1 - x~_i)),
// a lower bound LB on the squared segment distance that holds however inexact x~ is
// (near-parallel segments, degenerate capsules).  Reject iff LB (less a relative rounding
// margin) >= (rc_a + rc_b)^2.  Not a step of the method: a cull like the bound levels,
// so the sphere predicate still decides every result.
__device__ __forceinline__ void frame_pt(const float4& a, const float4& b, float tz, float4 o, float& x, float& y,
                                         float& z) {
  x = fmaf(a.x, o.x, fmaf(b.x, o.y, a.w));
  y = fmaf(a.y, o.x, fmaf(b.y, o.y, b.w));
  z = fmaf(a.z, o.x, fmaf(b.z, o.y, tz));
  if (o.z != 0.0f) {
    x = fmaf(fmaf(a.y, b.z, -a.z * b.y), o.z, x);
    y = fmaf(fmaf(a.z, b.x, -a.x * b.z), o.z, y);
    z = fmaf(fmaf(a.x, b.y, -a.y * b.x), o.z, z);
  }
}

// a point (o.x, 0, 0) of a link frame: frame_pt / xform_frame for an offset on the link's
// x axis (ds.l1tile bit 2), bit for bit -- column 0 and the translation only
__device__ __forceinline__ void frame_pt_x(const float* frames, int off, int s, int W, float ox, float& x, float& y,
                                           float& z, bool cf) {
  const float4 a = reinterpret_cast<const float4*>(frames + off)[s];
  const float2 t = frame_tyz(frames, off, s, W, cf);
  x = fmaf(a.x, ox, a.w);
  y = fmaf(a.y, ox, t.x);
  z = fmaf(a.z, ox, t.y);
}

template <bool PP, bool XAX = false, bool CF = false>
__device__ __forceinline__ void capsule_world(const KParams& p, const SV& sv, const Warp& w, int g, int s, float* P,
                                              float& rc) {
  if (!PP && XAX && (p.sc.l1tile & 4)) {   // endpoints on the link's x axis, group g = link g
    const int off = frame_off(sv, g, p.W, CF);
    const float4 c0 = sv.gcap[2 * g], c1 = sv.gcap[2 * g + 1];
    const float4 a = reinterpret_cast<const float4*>(w.frames + off)[s];
    const float2 t = frame_tyz(w.frames, off, s, p.W, CF);
    const float ty = t.x, tz = t.y;
    P[0] = fmaf(a.x, c0.x, a.w);
    P[1] = fmaf(a.y, c0.x, ty);
    P[2] = fmaf(a.z, c0.x, tz);
    P[3] = fmaf(a.x, c1.x, a.w);
    P[4] = fmaf(a.y, c1.x, ty);
    P[5] = fmaf(a.z, c1.x, tz);
    rc = c0.w;
    return;
  }
  float4 a, b;
  float tz;
  frame_cols<PP>(p, sv, w, sv.group[g].x, s, a, b, tz);
  const float4 c0 = sv.gcap[2 * g], c1 = sv.gcap[2 * g + 1];
  frame_pt(a, b, tz, c0, P[0], P[1], P[2]);
  frame_pt(a, b, tz, c1, P[3], P[4], P[5]);
  rc = c0.w;
}

template <bool PP, bool XAX = false, bool CF = false>
__device__ __forceinline__ bool capsules_may_touch(const KParams& p, const SV& sv, const Warp& w, int ga, int gb, int s) {
  float A[6], B[6], ra, rb;
  capsule_world<PP, XAX, CF>(p, sv, w, ga, s, A, ra);
  capsule_world<PP, XAX, CF>(p, sv, w, gb, s, B, rb);
  const float d1x = A[3] - A[0], d1y = A[4] - A[1], d1z = A[5] - A[2];
  const float d2x = B[3] - B[0], d2y = B[4] - B[1], d2z = B[5] - B[2];
  const float rx = A[0] - B[0], ry = A[1] - B[1], rz = A[2] - B[2];
  const float a = fmaf(d1x, d1x, fmaf(d1y, d1y, d1z * d1z));
  const float e = fmaf(d2x, d2x, fmaf(d2y, d2y, d2z * d2z));
  const float b = fmaf(d1x, d2x, fmaf(d1y, d2y, d1z * d2z));
  const float c = fmaf(d1x, rx, fmaf(d1y, ry, d1z * rz));
  const float f = fmaf(d2x, rx, fmaf(d2y, ry, d2z * rz));
  const float den = fmaf(a, e, -b * b);
  // __saturatef maps NaN (0 * inf from a degenerate segment) to 0
  const float s0 = __saturatef(fmaf(b, f, -c * e) * rcp_approx(den));
  const float t = __saturatef(fmaf(b, s0, f) * rcp_approx(e));
  const float u = __saturatef(fmaf(b, t, -c) * rcp_approx(a));
  const float Dx = fmaf(u, d1x, fmaf(-t, d2x, rx));
  const float Dy = fmaf(u, d1y, fmaf(-t, d2y, ry));
  const float Dz = fmaf(u, d1z, fmaf(-t, d2z, rz));
  const float h = fmaf(Dx, Dx, fmaf(Dy, Dy, Dz * Dz));
  const float gs = 2.0f * fmaf(Dx, d1x, fmaf(Dy, d1y, Dz * d1z));
  const float gt = -2.0f * fmaf(Dx, d2x, fmaf(Dy, d2y, Dz * d2z));
  const float lb = h + fminf(-gs * u, gs * (1.0f - u)) + fminf(-gt * t, gt * (1.0f - t));
  const float tol = 1e-6f * (h + fabsf(gs) + fabsf(gt));
  const float R = ra + rb;
  return lb - tol < R * R;
}

// Compacts w.nq[0, nn) in place to the entries whose capsules may touch (FFC: and whose
// key can still win); returns the new count.
template <int QUERY, bool COUNT, bool PP = false, bool XAX = false, bool CF = false>
__device__ int capsule_pass(const KParams& p, const SV& sv, Warp& w, int nn, uint32_t kprune, Counters& cnt) {
  const uint32_t P = (uint32_t)p.sc.n_pairs;
  int out = 0;
  for (int e0 = 0; e0 < nn; e0 += 32) {
    const int e = e0 + w.lane;
    bool keep = false;
    uint2 ent = make_uint2(0, 0);
    if (e < nn) {
      ent = w.nq[e];
      const int s = (int)(ent.x & 31u);
      const bool live = QUERY == Q_MOTVAL || (uint32_t)w.t_of(s, p.lgW) * P + (ent.y >> 16) < kprune;
      const int ga = (int)(ent.x >> 5), gb = (int)(ent.y & 0xFFFFu);
      keep = live;
      // a pair of two capsule-less groups (flag {p1, flag}.w == 0) gains nothing over level 2
      if (live && sv.gcap[2 * ga + 1].w + sv.gcap[2 * gb + 1].w > 0.0f) {
        keep = capsules_may_touch<PP, XAX, CF>(p, sv, w, ga, gb, s);
        if (COUNT) cnt.v[MRV_CNT_RR_CAPSULE] += 1;
      }
    }
    const unsigned m = __ballot_sync(FULL, keep);
    __syncwarp();
    if (keep) w.nq[out + __popc(m & ((1u << w.lane) - 1u))] = ent;
    out += __popc(m);
  }
  __syncwarp();
  return out;
}

// XAX: instantiated from the tiled level 1 only (rr_stage_tile, flush_l1<DIRECT>), where the
// x-axis placements (ds.l1tile bit 2) apply; the other instances keep their code unchanged
// (the general FFC / MotVal kernels measured 9-15 % slower with the runtime branch in them)
template <int QUERY, bool COUNT, bool PP = false, bool XAX = false, bool CF = false>
__device__ uint32_t flush_narrow(const KParams& p, const SV& sv, Warp& w, int nn, uint32_t kprune, Counters& cnt) {
  uint32_t best = MRV_NO_CONFLICT;
  bool hit = false;
  uint32_t hs = 0;   // MotVal spread packing: the states with a hit
  const uint32_t P = (uint32_t)p.sc.n_pairs;
  const int glg = p.sc.group_lg;
  if (p.sc.use_caps && !(p.flags & MRV_DIAG_NO_BROADPHASE)) nn = capsule_pass<QUERY, COUNT, PP, XAX, CF>(p, sv, w, nn, kprune, cnt);
  for (int e0 = 0; e0 < nn;) {
    Pack pk;
    uint32_t ms, mrank;
    int ll, ls, ol, os, on;
    if (glg >= 0) {   // uniform group size: each lane reads its own entry (broadcast LDS)
      pk = pack_uniform(w.lane, glg, nn - e0);
      const uint2 ent = w.nq[min(e0 + pk.my, nn - 1)];
      MRV_CHECK(e0 + pk.my < kNarrowCap);
      const int4 GA = sv.group[ent.x >> 5], GB = sv.group[ent.y & 0xFFFFu];
      ms = ent.x & 31u;
      mrank = ent.y >> 16;
      ll = GA.x; ls = GA.y; ol = GB.x; os = GB.y; on = GB.z;
    } else {
      const int e = e0 + w.lane;
      const bool valid = e < nn;
      uint2 ent = make_uint2(0, 0);
      int4 GL = make_int4(0, 0, 1, 0), GO = make_int4(0, 0, 1, 0);
      if (valid) {
        ent = w.nq[e];
        MRV_CHECK(e < kNarrowCap && (int)(ent.x >> 5) < p.sc.n_groups && (int)(ent.y & 0xFFFFu) < p.sc.n_groups);
        const int4 GA = sv.group[ent.x >> 5], GB = sv.group[ent.y & 0xFFFFu];
        // the group with more spheres goes on the lanes, the other one is looped over
        if (GB.z > GA.z) { GL = GB; GO = GA; } else { GL = GA; GO = GB; }
      }
      pk = pack_round(w.lane, valid, GL.z);
      ms = __shfl_sync(FULL, ent.x, pk.my) & 31u;
      mrank = __shfl_sync(FULL, ent.y, pk.my) >> 16;
      ll = __shfl_sync(FULL, GL.x, pk.my);
      ls = __shfl_sync(FULL, GL.y, pk.my);
      ol = __shfl_sync(FULL, GO.x, pk.my);
      os = __shfl_sync(FULL, GO.y, pk.my);
      on = __shfl_sync(FULL, GO.z, pk.my);
    }
    // lane = sphere pk.k of the entry's group L; the entry's lanes are contiguous, so the
    // lane also transforms sphere pk.k of group O (pk.k < on, as on <= na) into
    // w.nsc[lane], and the loop reads O's world centres from w.nsc[lane - pk.k + l]
    bool live = false;
    uint32_t key = 0;
    float ax = 0.0f, ay = 0.0f, az = 0.0f, ar = 0.0f;
    if (w.lane < pk.used) {
      const int s = (int)ms;
      key = (uint32_t)w.t_of(s, p.lgW) * P + mrank;
      live = QUERY == Q_MOTVAL || key < kprune;
      if (XAX && live && QUERY == Q_FFC && (p.sc.l1tile & 4)) {   // centres on the link x axes
        const float4 sa = sv.sphere[ls + pk.k];
        frame_pt_x(w.frames, frame_off(sv, ll, p.W, CF), s, p.W, sa.x, ax, ay, az, CF);
        ar = sa.w;
        if (pk.k < on) {
          const float4 sb = sv.sphere[os + pk.k];
          float bx, by, bz;
          frame_pt_x(w.frames, frame_off(sv, ol, p.W, CF), s, p.W, sb.x, bx, by, bz, CF);
          w.nsc[w.lane] = make_float4(bx, by, bz, sb.w);
        }
      } else if (live && QUERY == Q_FFC) {   // (MotVal measured faster with the full frame load)
        const float4 sa = sv.sphere[ls + pk.k];
        xform_frame(w.frames, sv.link_off[ll], s, p.W, sa.x, sa.y, sa.z, ax, ay, az);
        ar = sa.w;
        if (pk.k < on) {
          const float4 sb = sv.sphere[os + pk.k];
          float bx, by, bz;
          xform_frame(w.frames, sv.link_off[ol], s, p.W, sb.x, sb.y, sb.z, bx, by, bz);
          w.nsc[w.lane] = make_float4(bx, by, bz, sb.w);
        }
      } else if (live) {
        float F[12];
        load_frame_any<PP>(p, sv, w, ll, s, F);
        const float4 sa = sv.sphere[ls + pk.k];
        xform(F, sa.x, sa.y, sa.z, ax, ay, az);
        ar = sa.w;
        if (pk.k < on) {
          load_frame_any<PP>(p, sv, w, ol, s, F);
          const float4 sb = sv.sphere[os + pk.k];
          float bx, by, bz;
          xform(F, sb.x, sb.y, sb.z, bx, by, bz);
          w.nsc[w.lane] = make_float4(bx, by, bz, sb.w);
        }
      }
    }
    __syncwarp();
    if (live) {
      const float4* ob = w.nsc + (w.lane - pk.k);
      bool h = false;
#pragma unroll 8
      for (int l = 0; l < on; ++l) h |= sph_sph(ax, ay, az, ar, ob[l]);
      if (COUNT) {
        cnt.v[MRV_CNT_RR_NARROW] += on;
        cnt.v[MRV_CNT_SPHERE_XFORM] += 1 + (pk.k < on ? 1 : 0);
      }
      if (h) {
        hit = true;
        hs |= 1u << ms;
        best = min(best, key);
      }
    }
    __syncwarp();
    e0 += pk.nfit;
  }
  if (QUERY == Q_MOTVAL) return p.spread ? __reduce_or_sync(FULL, hs) : __any_sync(FULL, hit) ? 1u : 0u;
  return __reduce_min_sync(FULL, best);
}

// ------------------------------------------------------------------ self-collision
// Queued self pairs (s | k << 5 | segment << 8) become group pairs for the narrow phase,
// kNarrowCap at a time.
template <bool COUNT>
__device__ bool flush_self(const KParams& p, const SV& sv, Warp& w, int qn, Counters& cnt) {
  bool hit = false;
  for (int c0 = 0; c0 < qn; c0 += p.ncap) {
    const int nn = min(p.ncap, qn - c0);
    for (int e = w.lane; e < nn; e += 32) {
      const uint32_t ent = w.queue[c0 + e];
      const int seg = ent >> 8;
      MRV_CHECK(seg < p.sc.n_self_segs);
      const uint32_t ga = sv.self_segs[4 * seg].x & 0xFFFFu;
      const uint32_t gb = seg_idx_smem(sv.self_segs, seg, (ent >> 5) & 7);
      w.nq[e] = make_uint2((ent & 31u) | (ga << 5), gb);
    }
    __syncwarp();
    hit |= flush_narrow<Q_MOTVAL, COUNT>(p, sv, w, nn, MRV_NO_CONFLICT, cnt) != 0;
    __syncwarp();
  }
  return hit;
}

// Broad phase over the self-collision segments (group bound vs the groups of the
// paired links, precomputed (R_a + R_b)^2): lanes = (segment slot, state).
template <bool COUNT>
__device__ bool self_pass(const KParams& p, const SV& sv, Warp& w, bool stop_on_hit, bool& any, Counters& cnt) {
  const bool nobp = (p.flags & MRV_DIAG_NO_BROADPHASE) != 0;
  const int s = w.lane & (p.W - 1), gi = w.lane >> p.lgW, G = 32 >> p.lgW;
  const bool act = (w.amask >> s) & 1u;
  const float4* bcs = w.bc + s;
  const int nseg = p.sc.n_self_segs;
  int qn = 0;
  for (int b0 = 0; b0 < nseg; b0 += G) {
    const int sg = b0 + gi;
    uint32_t bits = 0;
    if (act && sg < nseg) {
      const uint4* rec = sv.self_segs + 4 * sg;
      const uint4 h = rec[0], ix = rec[1];
      // PP-ST-RRT variant: only the focus robot's own checks (n = 0 leaves bits empty)
      const bool mine = p.focus < 0 || sv.group[h.x & 0xFFFFu].w == p.focus;
      const float4 r2a = *reinterpret_cast<const float4*>(rec + 2), r2b = *reinterpret_cast<const float4*>(rec + 3);
      const float r2[8] = {r2a.x, r2a.y, r2a.z, r2a.w, r2b.x, r2b.y, r2b.z, r2b.w};
      const int n = mine ? (h.x >> 16) & 15 : 0;
      const float4 A = bcs[(h.x & 0xFFFFu) << p.lgW];
#pragma unroll
      for (int k = 0; k < kSegLen; ++k) {
        const float4 B = bcs[seg_idx(ix, k) << p.lgW];
        bits |= (d2_sph(A, B) < r2[k] ? 1u : 0u) << k;
      }
      const uint32_t m = (1u << n) - 1u;
      bits = nobp ? m : (bits & m);
      if (COUNT) cnt.v[MRV_CNT_SELF_BROAD] += n;
    }
    if (__any_sync(FULL, bits != 0u)) {
      int total;
      const int excl = scan_bits(w.lane, bits, total);
      if (qn + total > p.qcap) {   // (p.qcap = kQueueCap >= 32 * kSegLen with self segments)
        __syncwarp();
        any |= flush_self<COUNT>(p, sv, w, qn, cnt);
        qn = 0;
        __syncwarp();
        if (any && stop_on_hit) return true;
      }
      enqueue_bits(w, bits, s, sg, qn, excl, total);
    }
  }
  if (qn) {
    __syncwarp();
    any |= flush_self<COUNT>(p, sv, w, qn, cnt);
    __syncwarp();
  }
  return any && stop_on_hit;
}

// CC(S_i, E) of Alg. 1: robot-obstacle (MRV_CHECK_ENV) and the
// robot's self-collision pairs (MRV_CHECK_SELF).  Returns nonzero on a hit (under spread
// packing, which runs without self pairs: the mask of the states with an obstacle hit).
template <bool COUNT>
__device__ uint32_t env_stage(const KParams& p, const SV& sv, Warp& w, bool stop_on_hit, Counters& cnt) {
  uint32_t any = 0;
  if (p.flags & MRV_CHECK_ENV) {
    int qn = 0;
    if (env_grid_pass<COUNT>(p, sv, w, stop_on_hit, qn, any, cnt)) return any;
    if (qn) {
      __syncwarp();
      any |= flush_env<COUNT>(p, sv, w, qn, cnt);
      __syncwarp();
    }
    if (stop_on_hit && mv_done(p, w, any)) return any;
  }
  if (p.flags & MRV_CHECK_SELF) {
    bool sany = any != 0;
    if (self_pass<COUNT>(p, sv, w, stop_on_hit, sany, cnt)) return 1u;
    any |= sany ? 1u : 0u;
  }
  return any;
}

template <int QUERY>
__device__ __forceinline__ void merge(uint32_t& res, uint32_t r) {
  if (QUERY == Q_MOTVAL) res |= r;
  else res = min(res, r);
}

// Level 2 on qn queued supergroup pairs, one lane per pair: the <= 3 x 3 group bounds
// are tested branch-free into a 9-bit mask, survivors are compacted into w.nq by a
// warp scan (w.nq is flushed first if it could overflow).  Returns true if MotVal may stop.
// FFC level 2 with three lanes per queued supergroup pair (lane = one group of a, tested
// against the <= 3 groups of b): a batch's ~10 surviving pairs fill one round of 30
// lanes instead of a third of a round, and each lane derives 4 group bounds and runs 3
// tests instead of 6 and 9.  Same tests, same survivors (in a different queue order;
// the narrow phase's min-reduction does not depend on it).
template <bool COUNT>
__device__ void flush_l1_rows(const KParams& p, const SV& sv, Warp& w, int qn, int& nn, uint32_t& res,
                              bool stop_on_hit, Counters& cnt) {
  const bool nobp = (p.flags & MRV_DIAG_NO_BROADPHASE) != 0;
  const uint32_t P = (uint32_t)p.sc.n_pairs;
  const int n = p.sc.n_robots;
  for (int c0 = 0; c0 < 3 * qn; c0 += 32) {
    const int e = c0 + w.lane;
    const int pr = (e * 0xAAABu) >> 17, ka = e - 3 * pr;   // e / 3, e % 3 (e < 3 * kQueueCap)
    uint32_t bits = 0, s = 0, rank = 0;
    int ga = 0, gb0 = 0;
    if (pr < qn) {
      const uint32_t ent = w.queue[pr];
      const int seg = ent >> 8;
      MRV_CHECK(pr < kQueueCap && seg < p.sc.n_rr_segs);
      const uint32_t* rs = reinterpret_cast<const uint32_t*>(sv.rr_segs + 2 * seg);
      const int4 SA = sv.super[rs[0] & 0xFFFFu];
      const int4 SB = sv.super[rs[2 + ((ent >> 5) & 7)]];
      s = ent & 31;
      const int i = min(SA.x, SB.x), j = max(SA.x, SB.x);
      rank = (uint32_t)(i * n - i * (i + 1) / 2 + (j - i - 1));
      ga = SA.y + ka;
      gb0 = SB.y;
      if (ka < SA.z) {
        const float4 A = group_world_bound<Q_FFC>(sv, w.frames, ga, s, p.W);
#pragma unroll
        for (int kb = 0; kb < 3; ++kb) {
          const float4 B = group_world_bound<Q_FFC>(sv, w.frames, min(gb0 + kb, gb0 + SB.z - 1), s, p.W);
          const float rsum = A.w + B.w;
          bits |= (d2_sph(A, B) < rsum * rsum ? 1u : 0u) << kb;
        }
        const uint32_t valid = (1u << SB.z) - 1u;
        bits = nobp ? valid : (bits & valid);
        if (COUNT) cnt.v[MRV_CNT_RR_BROAD] += (uint64_t)SB.z;
      }
    }
    if (__any_sync(FULL, bits != 0u)) {
      int total;
      static_assert(32 * kSuperMax <= kNarrowCap, "one round of rows fits an empty group-pair queue");
      const int excl = scan_bits(w.lane, bits, total);
      if (nn + total > kNCap<Q_FFC>) {
        __syncwarp();
        merge<Q_FFC>(res, flush_narrow<Q_FFC, COUNT>(p, sv, w, nn, stop_on_hit ? res : MRV_NO_CONFLICT, cnt));
        nn = 0;
        __syncwarp();
      }
      int pos = nn + excl;
      MRV_CHECK(nn + total <= kNCap<Q_FFC>);
      while (bits) {
        const int kb = __ffs(bits) - 1;
        bits &= bits - 1u;
        w.nq[pos++] = make_uint2(s | ((uint32_t)ga << 5), (uint32_t)(gb0 + kb) | (rank << 16));
      }
      nn += total;
    }
  }
}

// DIRECT: queue entries name the two supergroups, s | a << 5 | b << 10 (rr_stage_tile),
// instead of a segment slot
template <int QUERY, bool COUNT, bool LEAN = false, bool PP = false, bool DIRECT = false>
__device__ bool flush_l1(const KParams& p, const SV& sv, Warp& w, int qn, int& nn, uint32_t& res, bool stop_on_hit,
                         Counters& cnt) {
  static_assert(kSuperMax == 3, "level-2 tile is 3 x 3");
  if (QUERY == Q_FFC && !LEAN && !DIRECT) {   // (the lean cfg5 instance measured 5.6 % slower with rows)
    flush_l1_rows<COUNT>(p, sv, w, qn, nn, res, stop_on_hit, cnt);
    return false;
  }
  const bool nobp = (p.flags & MRV_DIAG_NO_BROADPHASE) != 0;
  const uint32_t P = (uint32_t)p.sc.n_pairs;
  const int n = p.sc.n_robots;
  for (int c0 = 0; c0 < qn; c0 += 32) {
    const int e = c0 + w.lane;
    uint32_t bits = 0, s = 0, rank = 0;
    int ga0 = 0, gb0 = 0;
    if (e < qn) {
      const uint32_t ent = w.queue[e];
      int4 SA, SB;
      if (DIRECT) {
        MRV_CHECK(e < kQueueCap && (int)((ent >> 5) & 31) < p.sc.n_super && (int)((ent >> 10) & 31) < p.sc.n_super);
        SA = sv.super[(ent >> 5) & 31];
        SB = sv.super[(ent >> 10) & 31];
      } else {
        const int seg = ent >> 8;
        MRV_CHECK(e < kQueueCap && seg < p.sc.n_rr_segs);
        const uint32_t* rs = reinterpret_cast<const uint32_t*>(sv.rr_segs + 2 * seg);
        SA = sv.super[rs[0] & 0xFFFFu];
        SB = sv.super[rs[2 + ((ent >> 5) & 7)]];
        MRV_CHECK((int)(rs[0] & 0xFFFFu) < p.sc.n_super && (int)rs[2 + ((ent >> 5) & 7)] < p.sc.n_super);
      }
      s = ent & 31;
      const int i = min(SA.x, SB.x), j = max(SA.x, SB.x);   // segments own pairs in either order
      rank = (uint32_t)(i * n - i * (i + 1) / 2 + (j - i - 1));
      ga0 = SA.y;
      gb0 = SB.y;
      {
        float4 A[3], B[3];
        if (PP) {   // the partner side's bounds from the table row
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            A[q] = group_bound_any<PP>(p, sv, w, min(ga0 + q, ga0 + SA.z - 1), s);
            B[q] = group_bound_any<PP>(p, sv, w, min(gb0 + q, gb0 + SB.z - 1), s);
          }
        } else if (w.bc) {
          const float4* bcs = w.bc + s;
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            A[q] = bcs[min(ga0 + q, ga0 + SA.z - 1) << p.lgW];
            B[q] = bcs[min(gb0 + q, gb0 + SB.z - 1) << p.lgW];
          }
        } else if (DIRECT && (p.sc.l1tile & 2)) {
          const bool cf = QUERY == Q_FFC && LEAN && (p.sc.l1tile & 4);   // compact frames: FFC's lean instance
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            A[q] = group_bound_xaxis(sv, w.frames, min(ga0 + q, ga0 + SA.z - 1), s, p.W, cf);
            B[q] = group_bound_xaxis(sv, w.frames, min(gb0 + q, gb0 + SB.z - 1), s, p.W, cf);
          }
        } else {   // world bound = link frame x local bound (the FK sink's arithmetic)
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            A[q] = group_world_bound<QUERY>(sv, w.frames, min(ga0 + q, ga0 + SA.z - 1), s, p.W);
            B[q] = group_world_bound<QUERY>(sv, w.frames, min(gb0 + q, gb0 + SB.z - 1), s, p.W);
          }
        }
#pragma unroll
        for (int ka = 0; ka < 3; ++ka)
#pragma unroll
          for (int kb = 0; kb < 3; ++kb) {
            const float rs = A[ka].w + B[kb].w;
            bits |= (d2_sph(A[ka], B[kb]) < rs * rs ? 1u : 0u) << (3 * ka + kb);
          }
        const uint32_t m = (SA.z >= 1 ? 0x007u : 0u) & ((1u << SB.z) - 1u);   // row mask for kb < nb
        uint32_t valid = 0;
#pragma unroll
        for (int ka = 0; ka < 3; ++ka)
          if (ka < SA.z) valid |= m << (3 * ka);
        bits = nobp ? valid : (bits & valid);
        if (COUNT) cnt.v[MRV_CNT_RR_BROAD] += (uint64_t)SA.z * SB.z;
      }
    }
    if (__any_sync(FULL, bits != 0u)) {
      int total;
      const int excl = scan_bits(w.lane, bits, total);
      if (nn + total > ncap<QUERY>(p)) {
        __syncwarp();
        merge<QUERY>(res, flush_narrow<QUERY, COUNT, PP, DIRECT, QUERY == Q_FFC && LEAN>(p, sv, w, nn, stop_on_hit ? res : MRV_NO_CONFLICT, cnt));
        nn = 0;
        __syncwarp();
        if (QUERY == Q_MOTVAL && stop_on_hit && mv_done(p, w, res)) return true;
      }
      if (total <= ncap<QUERY>(p)) {
        int pos = nn + excl;
        MRV_CHECK(nn + total <= ncap<QUERY>(p));
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1u;
          const int ka = b / 3, kb = b - 3 * ka;
          w.nq[pos++] = make_uint2(s | ((uint32_t)(ga0 + ka) << 5), (uint32_t)(gb0 + kb) | (rank << 16));
        }
        nn += total;
      } else {
        // more survivors in one round than the queue holds (only with very dense
        // contact or DIAG_NO_BROADPHASE): append lane by lane, flushing as it fills
        for (int src = 0; src < 32; ++src) {
          uint32_t bl = __shfl_sync(FULL, bits, src);
          const uint32_t sl = __shfl_sync(FULL, s, src), rl = __shfl_sync(FULL, rank, src);
          const int al = __shfl_sync(FULL, ga0, src), bl0 = __shfl_sync(FULL, gb0, src);
          while (bl) {
            if (nn == ncap<QUERY>(p)) {
              __syncwarp();
              merge<QUERY>(res, flush_narrow<QUERY, COUNT, PP, DIRECT, QUERY == Q_FFC && LEAN>(p, sv, w, nn, stop_on_hit ? res : MRV_NO_CONFLICT, cnt));
              nn = 0;
              __syncwarp();
              if (QUERY == Q_MOTVAL && stop_on_hit && mv_done(p, w, res)) return true;
            }
            const int b = __ffs(bl) - 1;
            bl &= bl - 1u;
            const int ka = b / 3, kb = b - 3 * ka;
            if (w.lane == 0) w.nq[nn] = make_uint2(sl | ((uint32_t)(al + ka) << 5), (uint32_t)(bl0 + kb) | (rl << 16));
            ++nn;
          }
        }
        __syncwarp();
      }
    }
  }
  return false;
}

// Tiled level 1 (FFC's lean instance and MotVal's spread packing, on scenes with
// ds.l1tile: 4 robots x 3 supergroups, supergroup 3r + k, W = 8).  Lane (robot r, state s) -- the lane whose FK produced those
// bounds -- tests its robot's 3 supergroups against robot r + 1's (all 9 pairs) and robot
// r + 2's (6 pairs: (0,0) (1,1) (2,2) (0,1) (0,2) (1,2), own index first; the lanes of
// robots 2 and 3 see the two diagonal robot pairs transposed, so together they cover all
// 9).  The four lanes of a state cover the 54 supergroup pairs of the 6 robot pairs with 15
// unrolled tests each and no segment records; the scene's per-role mask drops the
// statically pruned pairs and the (k, k) pairs tested twice.  The segment walk's predicate
// with the exact sign of d2 - rs^2 instead of d2 < fl(rs^2): survivors can differ only for
// bounds within an ulp of touching, far inside their 1e-5 m padding, so the sphere level --
// which decides every result -- sees the same candidates that can collide (outputs
// bit-identical, tested); queued in another order, which the narrow phase's min-reduction
// does not see.  Queue entry: s | a << 5 | b << 10 (the two supergroups).
template <int QUERY, bool COUNT, bool LEAN = false>
__device__ uint32_t rr_stage_tile(const KParams& p, const SV& sv, Warp& w, bool stop_on_hit, Counters& cnt) {
  constexpr int W = 8;
  const int s = w.lane & (W - 1), r = w.lane >> 3;
  const int x = (r + 1) & 3, y = (r + 2) & 3;
  uint32_t bits = 0;
  if ((w.amask >> s) & 1u) {
    const float4* own = w.sbc + 3 * r * W + s;
    const float4* X = w.sbc + 3 * x * W + s;
    const float4* Y = w.sbc + 3 * y * W + s;
    float4 A[3], B[3], C[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      A[k] = own[k * W];
      B[k] = X[k * W];
      C[k] = Y[k * W];
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const float rs = A[a].w + B[b].w;
        // (sign of d2 - rs^2 with one rounding: the exact strict test, inside the bounds'
      // 1e-5 m padding like the segment walk's rounded comparison)
      bits |= (__float_as_uint(fmaf(-rs, rs, d2_sph(A[a], B[b]))) >> 31) << (3 * a + b);
      }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      const int a = i < 3 ? i : i < 5 ? 0 : 1, b = i < 3 ? i : i == 3 ? 1 : 2;
      const float rs = A[a].w + C[b].w;
      bits |= (__float_as_uint(fmaf(-rs, rs, d2_sph(A[a], C[b]))) >> 31) << (9 + i);
    }
    const uint32_t m = (uint32_t)(p.sc.l1tile_masks >> (16 * r)) & 0x7FFFu;
    bits &= m;
    if (COUNT) cnt.v[MRV_CNT_RR_SUPER] += __popc(m);
  }
  // exclusive prefix of the per-lane counts (<= 15: four bit planes, one ballot each)
  const int nb = __popc(bits);
  const unsigned lt = (1u << w.lane) - 1u;
  int excl = 0, total = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const unsigned bal = __ballot_sync(FULL, (nb >> k) & 1);
    excl += __popc(bal & lt) << k;
    total += __popc(bal) << k;
  }
  uint32_t res = QUERY == Q_MOTVAL ? 0u : MRV_NO_CONFLICT;
  if (total == 0) return res;
  // bit -> (own supergroup, partner supergroup) nibbles: a | b << 2
  constexpr uint64_t kCode = 0x0ull | (0x4ull << 4) | (0x8ull << 8) | (0x1ull << 12) | (0x5ull << 16) |
                             (0x9ull << 20) | (0x2ull << 24) | (0x6ull << 28) | (0xAull << 32) |   // r+1: a = b / 3
                             (0x0ull << 36) | (0x5ull << 40) | (0xAull << 44) | (0x4ull << 48) |
                             (0x8ull << 52) | (0x9ull << 56);                                       // r+2: kTileDiag
  const uint32_t own0 = (uint32_t)(3 * r), px = (uint32_t)(3 * x), py = (uint32_t)(3 * y);
  int nn = 0;
  const int cap = qcap<QUERY>(p);
  for (int c = 0; c < 3; ++c) {   // one pass when the survivors fit the queue (the usual case),
                                  // else three passes of 5 bit positions (<= 160 entries each)
    uint32_t cb = bits;
    int pos = excl, tot = total;
    if (total > cap) {
      cb = bits & (0x1Fu << (5 * c));
      pos = scan_bits(w.lane, cb, tot);
      if (tot == 0) continue;
    }
    MRV_CHECK(pos + __popc(cb) <= cap);
    while (cb) {
      const int b = __ffs(cb) - 1;
      cb &= cb - 1u;
      const uint32_t code = (uint32_t)(kCode >> (4 * b)) & 15u;
      const uint32_t ga = own0 + (code & 3u), gb = (b < 9 ? px : py) + (code >> 2);
      w.queue[pos++] = (uint32_t)s | (ga << 5) | (gb << 10);
    }
    __syncwarp();
    const bool stop = flush_l1<QUERY, COUNT, LEAN, false, true>(p, sv, w, tot, nn, res, stop_on_hit, cnt);
    __syncwarp();
    if (stop) return res;   // (MotVal: every open state has a hit)
    if (total <= cap) break;
  }
  if (nn) {
    __syncwarp();
    merge<QUERY>(res, flush_narrow<QUERY, COUNT, false, true, QUERY == Q_FFC && LEAN>(p, sv, w, nn, stop_on_hit ? res : MRV_NO_CONFLICT, cnt));
    __syncwarp();
  }
  return res;
}

template <int QUERY, bool COUNT, bool LEAN = false, bool PP = false, bool T8 = false>
__device__ uint32_t rr_stage(const KParams& p, const SV& sv, Warp& w, bool stop_on_hit, Counters& cnt) {
  // the tiled level 1: the compile-time W = 8 instances (T8; the runtime-W ones keep their
  // code size -- cfg4's FFC measured 1.5 % slower with the tile compiled in), without a
  // focus robot (whose pairs are a subset) or MRV_DIAG_NO_BROADPHASE (segments without the
  // reach pruning: the reference of the tests)
  if (T8 && !PP && p.sc.l1tile && p.W == 8 && p.focus < 0 && !(p.flags & MRV_DIAG_NO_BROADPHASE))
    return rr_stage_tile<QUERY, COUNT, LEAN>(p, sv, w, stop_on_hit, cnt);
  const bool nobp = (p.flags & MRV_DIAG_NO_BROADPHASE) != 0;
  const uint32_t P = (uint32_t)p.sc.n_pairs;
  const int s = w.lane & (p.W - 1), gi = w.lane >> p.lgW, G = 32 >> p.lgW;
  const bool act = (w.amask >> s) & 1u;
  const float4* sbs = w.sbc + s;
  const int nseg = p.sc.n_rr_segs;
  uint32_t res = QUERY == Q_MOTVAL ? 0u : MRV_NO_CONFLICT;
  int qn = 0, nn = 0;
  for (int b0 = 0; b0 < nseg; b0 += G) {
    const int sg = b0 + gi;
    uint32_t bits = 0;
    if (act && sg < nseg) {
      const uint4* rec = sv.rr_segs + 2 * sg;
      const uint4 h = rec[0];
      // (no key-based skip here: a batch's conflict is rarely known before its levels 1
      // and 2 end, and the narrow phase prunes by key -- the checks cost cfg5 1.8 %, cfg4 3.7 %)
      {
        const uint4 h2 = rec[1];
        const uint32_t cidx[6] = {h.z, h.w, h2.x, h2.y, h2.z, h2.w};
        const int n = (h.x >> 16) & 15;
        uint32_t m = (1u << n) - 1u;
        if (p.focus >= 0 && !(PP && p.pp_nseg > 0)) {   // PP-ST-RRT variant: only pairs (focus, partner)
          const int i = sv.super[h.x & 0xFFFFu].x;
          uint32_t allow = 0;
#pragma unroll
          for (int k = 0; k < kRRSegLen; ++k) {
            const int j = sv.super[cidx[k]].x;
            const bool ok = (i == p.focus && ((p.partners >> j) & 1ull)) || (j == p.focus && ((p.partners >> i) & 1ull));
            allow |= (ok ? 1u : 0u) << k;
          }
          m &= allow;
        }
        if (!PP || m) {   // (PP: a segment of partner-partner pairs is skipped whole)
          const float4 A = sbs[(h.x & 0xFFFFu) << p.lgW];
#pragma unroll
          for (int k = 0; k < kRRSegLen; ++k) {
            const float4 B = sbs[cidx[k] << p.lgW];
            const float rs = A.w + B.w;
            bits |= (d2_sph(A, B) < rs * rs ? 1u : 0u) << k;
          }
        }
        bits = nobp ? m : (bits & m);
        if (COUNT) cnt.v[MRV_CNT_RR_SUPER] += __popc(m);
      }
    }
    if (__any_sync(FULL, bits != 0u)) {
      int total;
      const int excl = scan_bits(w.lane, bits, total);
      if (qn + total > qcap<QUERY>(p)) {   // total <= 32 * kRRSegLen <= qcap
        __syncwarp();
        const bool stop = flush_l1<QUERY, COUNT, LEAN, PP>(p, sv, w, qn, nn, res, stop_on_hit, cnt);
        qn = 0;
        __syncwarp();
        if (stop) return res;
      }
      enqueue_bits(w, bits, s, sg, qn, excl, total);
    }
  }
  if (qn) {
    __syncwarp();
    const bool stop = flush_l1<QUERY, COUNT, LEAN, PP>(p, sv, w, qn, nn, res, stop_on_hit, cnt);
    __syncwarp();
    if (stop) return res;
  }
  if (nn) {
    __syncwarp();
    merge<QUERY>(res, flush_narrow<QUERY, COUNT, PP>(p, sv, w, nn, stop_on_hit ? res : MRV_NO_CONFLICT, cnt));
    __syncwarp();
  }
  return res;
}

// ------------------------------------------------------------------ MotVal: FK fused with CC(S_i, E)
// Fast path (p.fuse_env, decided by the launcher): every robot is a fast-DH chain with
// the same dof, n_robots * W <= 32 (one FK lane per (robot, state)), combined order, no
// self-collision or focus robot, per-motion T.  The FK lanes run the obstacle broad phase
// as each link's group bound comes out of the chain walk (it is in registers already):
// grid-cell lookup, one candidate test per trip, survivors compacted into w.queue; a
// queue that could overflow is flushed to the narrow phase on the spot, so an obstacle
// hit ends the batch before the remaining links are computed.  Same predicates, same
// survivors as fk_stage + env_grid_pass; no per-group bounds are stored.  Returns nonzero
// on a hit (spread packing: the states with a hit; a lane whose motion has a hit stops
// its broad phase, and the walk ends once every motion in the batch has one).
template <bool COUNT, bool LEAN = false, bool PP = false>
__device__ uint32_t fk_env_fused(const KParams& p, const SV& sv, Warp& w, bool stop_on_hit, Counters& cnt) {
  // PP: lanes = the focus robot's states only (the batch holds its waypoints alone); its
  // group bounds are also stored (level 2 reads them), the partners' rows are in flight
  const int total = PP ? p.W : p.sc.n_robots << p.lgW;
  const bool on = w.lane < total;
  const int r = PP ? p.focus : on ? w.lane >> p.lgW : 0, s = w.lane & (p.W - 1);
  const bool act0 = on && ((w.amask >> s) & 1u);
  bool act = act0;
  const int Tl = p.spread ? w.mT : w.T;
  int t = p.spread ? w.mt : w.t_of(s, p.lgW);
  if (t >= Tl) t = Tl - 1;
  const Interp ip = interp_setup<!LEAN>(t, Tl, p.K);
  const int4 ra = sv.robot[3 * r];
  const int lb = ra.z, dof = ra.y;   // the same dof for every robot (launcher)
  const int W = p.W;
  float M[12];
  {   // base * link 0's fixed DH part (sv.dhbase; link 0's record is the identity step)
    const float4 b0 = sv.dhbase[3 * r], b1 = sv.dhbase[3 * r + 1], b2 = sv.dhbase[3 * r + 2];
    M[0] = b0.x; M[1] = b0.y; M[2] = b0.z; M[3] = b0.w;
    M[4] = b1.x; M[5] = b1.y; M[6] = b1.z; M[7] = b1.w;
    M[8] = b2.x; M[9] = b2.y; M[10] = b2.z; M[11] = b2.w;
  }
  const float* wr = (p.spread ? w.mwp : w.wp_smem) + (PP ? 0 : r) * p.K * p.S;
  const float* w0p = wr + ip.seg * p.S;    // the two knots' joint values, advanced per joint
  const float* w1p = wr + ip.seg1 * p.S;
  float* fp = w.frames + sv.link_off[lb];
  const float4* rec = sv.dhrec + 3 * lb;
  const float4 g0 = sv.grid[0];
  const float gox = -g0.x * g0.w, goy = -g0.y * g0.w, goz = -g0.z * g0.w;   // cell = floor(c / h - origin / h)
  const int4 gn = *reinterpret_cast<const int4*>(sv.grid + 1);
  const bool nobp = (p.flags & MRV_DIAG_NO_BROADPHASE) != 0;
  float cx = 0.0f, cy = 0.0f, cz = 0.0f, cr = -1e30f;   // Ritter accumulator (FrameSink::group_at)
  int qn = 0;
  uint32_t any = 0;
  for (int j = 0; j < dof; ++j, fp += 9 * W, rec += 3, ++w0p, ++w1p) {
    const float4 P = rec[0], GB = rec[1];
    const int4 ID = *reinterpret_cast<const int4*>(rec + 2);
    const float q = fmaf(ip.u, *w1p - *w0p, *w0p);
    float sn, cs;
    fast_sincos(q, sn, cs);
    const float ta = P.x, ca = P.y, sa = P.z, td = P.w;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const float m0 = M[4 * i], m1 = M[4 * i + 1], m2 = M[4 * i + 2], m3 = M[4 * i + 3];
      const float a1 = fmaf(m1, ca, m2 * sa);          // A = M * Tz(d) Tx(a) Rx(alpha)
      const float a2 = fmaf(m2, ca, -(m1 * sa));
      M[4 * i + 3] = fmaf(m0, ta, fmaf(m2, td, m3));
      M[4 * i + 0] = fmaf(cs, m0, sn * a1);             // M = A * Rz(q)
      M[4 * i + 1] = fmaf(cs, a1, -sn * m0);
      M[4 * i + 2] = a2;
    }
    // (the group bound's centre is on the link's x axis: column 0 and the translation)
    const float bx = fmaf(M[0], GB.x, M[3]), by = fmaf(M[4], GB.x, M[7]), bz = fmaf(M[8], GB.x, M[11]);
    if (on) {
      reinterpret_cast<float4*>(fp)[s] = make_float4(M[0], M[4], M[8], M[3]);
      reinterpret_cast<float4*>(fp + 4 * W)[s] = make_float4(M[1], M[5], M[9], M[7]);
      fp[8 * W + s] = M[11];
      if (PP) w.bc[ID.x * W + s] = make_float4(bx, by, bz, GB.w);
    }
    {   // supergroup bound (same merge as FrameSink::group_at)
      if (ID.y & 0x40000000) {
        cx = bx; cy = by; cz = bz; cr = GB.w;
      } else {
        const float dx = bx - cx, dy = by - cy, dz = bz - cz;
        const float d = sqrt_approx(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
        const bool contains = cr + d <= GB.w;
        const bool grow = d + GB.w > cr;
        const float nr = 0.5f * (cr + d + GB.w);
        const float f = (nr - cr) * rcp_approx(d);
        const float gx = fmaf(f, dx, cx), gy = fmaf(f, dy, cy), gz = fmaf(f, dz, cz);
        cx = contains ? bx : grow ? gx : cx;
        cy = contains ? by : grow ? gy : cy;
        cz = contains ? bz : grow ? gz : cz;
        cr = contains ? GB.w : grow ? nr : cr;
      }
      if (ID.y < 0 && on) w.sbc[(ID.y & 0x3FFFFFFF) * W + s] = make_float4(cx, cy, cz, fmaf(cr, 1.0f + 1e-6f, 1e-5f));
    }
    // (no __syncwarp here: every flush_env below is preceded by one, which orders these
    // frame stores before the flush's loads)
    // obstacle broad phase of this link's group (env_grid_pass, in registers)
    int beg = 0, n = 0;
    if (act && nobp) {   // diagnostic: no grid -- every obstacle is a candidate
      n = p.sc.n_osph + p.sc.n_box;
    } else if (act) {
      // (fp32 cell arithmetic: a centre rounded across a cell face stays within eps of the
      // cell it lands in, which the lists cover -- scene.cpp)
      const int ix = (int)floorf(fmaf(bx, g0.w, gox)), iy = (int)floorf(fmaf(by, g0.w, goy)),
                iz = (int)floorf(fmaf(bz, g0.w, goz));
      if ((unsigned)ix < (unsigned)gn.x && (unsigned)iy < (unsigned)gn.y && (unsigned)iz < (unsigned)gn.z) {
        const int c = (iz * gn.y + iy) * gn.x + ix;
        beg = sv.cell_start[c];
        n = (int)sv.cell_start[c + 1] - beg;
      }
    }
    for (int i = 0; __any_sync(FULL, i < n); ++i) {   // one candidate per trip (measured best)
      bool tt = false;
      if (i < n) {
        const uint32_t o = nobp ? (uint32_t)i : sv.cell_list[beg + i];
        const float4 lo = sv.obs[2 * o], hi = sv.obs[2 * o + 1];
        const float rs = GB.w + lo.w;
        tt = nobp || d2_obs(bx, by, bz, lo, hi) < rs * rs;
        if (COUNT) cnt.v[MRV_CNT_ENV_BROAD] += 1;
      }
      const unsigned bal = __ballot_sync(FULL, tt);
      if (bal) {
        if (qn + 32 > p.qcap) {
          __syncwarp();
          any |= flush_env<COUNT>(p, sv, w, qn, cnt);
          qn = 0;
          __syncwarp();
          if (stop_on_hit && any) {
            if (!p.spread) return any;
            const uint32_t dead = dead_states(w, any);
            if ((w.amask & ~dead) == 0) return any;
            if ((dead >> s) & 1u) {   // (this lane's motion is invalid: no further candidates)
              act = false;
              n = 0;
            }
          }
        }
        if (tt) w.queue[qn + __popc(bal & ((1u << w.lane) - 1u))] = (uint32_t)s | ((uint32_t)ID.x << 5) | ((uint32_t)(beg + i) << 16);
        qn += __popc(bal);
      }
    }
  }
  if (COUNT && act0) {
    cnt.v[MRV_CNT_SUPER_BOUNDS] += sv.robot[3 * r + 2].y;
    cnt.v[MRV_CNT_ROBOT_STATES] += 1;
    cnt.v[MRV_CNT_JOINTS] += dof;
    if (PP || r == 0) cnt.v[MRV_CNT_STATES] += 1;
  }
  if (qn) {
    __syncwarp();
    any |= flush_env<COUNT>(p, sv, w, qn, cnt);
    __syncwarp();
  }
  return any;
}

// ------------------------------------------------------------------ batches of one motion
__device__ __forceinline__ void set_batch(Warp& w, int c, int W, int lgW) {
  w.c = c;
  if (w.tb == 0 && w.te == w.T) {
    if (w.rake) {   // lane k < W active iff its rake timestep c + k nb is inside T (no division)
      w.amask = __ballot_sync(FULL, w.lane < W && c + w.lane * w.nb < w.T);
    } else {
      const int n_act = max(0, min(W, w.T - (c << lgW)));
      w.amask = n_act >= 32 ? FULL : ((1u << n_act) - 1u);
    }
  } else {  // time window: each lane < W tests its own timestep
    const int t = w.t_of(w.lane, lgW);
    w.amask = __ballot_sync(FULL, w.lane < W && t >= w.tb && t < w.te);
  }
}

template <int QUERY, bool COUNT, bool LEAN = false, bool PP = false, bool T8 = false>
__device__ void process_item(const KParams& p, const SV& sv, Warp& w, int64_t m, int slice, float* wp_smem,
                             Counters& cnt) {
  bool bad_T = false;
  if (p.Trob) {   // horizon = the longest robot path (t_max = max |p_i|)
    w.Tr = p.Trob + m * p.sc.n_robots;
    int T = 1, Tlo = 1;
    for (int r = w.lane; r < p.sc.n_robots; r += 32) {
      T = max(T, w.Tr[r]);
      Tlo = min(Tlo, w.Tr[r]);
    }
    w.T = __reduce_max_sync(FULL, T);
    bad_T = __reduce_min_sync(FULL, Tlo) < 1;
  } else if (LEAN) {   // the lean instance runs fixed-T batches only (validated by the launcher)
    w.Tr = nullptr;
    w.T = p.Tfix;
  } else {
    w.Tr = nullptr;
    w.T = p.Tm ? p.Tm[m] : p.Tfix;
    bad_T = w.T < 1;
  }
  w.t0 = PP ? p.pp_t0[m] : 0;
  // device-resident T cannot be validated before the launch (mrv.h): a T < 1, or an FFC
  // horizon whose keys t * P overflow uint32, leaves the motion's result at valid / no
  // conflict and raises a bit in the scene's status word
  const bool bad_range = QUERY == Q_FFC && !LEAN && !bad_T &&
                         (uint64_t)(uint32_t)w.T * (uint32_t)p.sc.n_pairs >= 0xFFFFFFFFull;
  const bool bad_start = PP && w.t0 < 0;   // (a negative start would index before the table)
  if (bad_T || bad_range || bad_start) {
    if (w.lane == 0) {
      atomicOr(p.dev_status, bad_T ? (uint32_t)MRV_DEVERR_TIMESTEPS
                             : bad_range ? (uint32_t)MRV_DEVERR_RANGE : (uint32_t)MRV_DEVERR_START);
      if (QUERY == Q_MOTVAL) p.out_valid[m] = 1;
      else p.out_key[m] = MRV_NO_CONFLICT;
      if (p.effort) p.effort[m] = 0;
    }
    return;
  }
  // stage the motion's waypoint block (coalesced, vectorised when aligned)
  const float* src = p.wp + m * (int64_t)p.nKS;
  if (p.wp_in_smem) {
    if (((reinterpret_cast<uintptr_t>(src) & 15u) == 0) && ((p.nKS & 3) == 0)) {
      const float4* s4 = reinterpret_cast<const float4*>(src);
      float4* d4 = reinterpret_cast<float4*>(wp_smem);
      bool big = false;
      for (int i = w.lane; i < (p.nKS >> 2); i += 32) {
        const float4 v = __ldg(s4 + i);
        d4[i] = v;
        big |= fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))) > 3.0f;
      }
      // (only the lean FFC walk reads w.wrap: its range-reduction-free copy)
      w.wrap = (QUERY == Q_FFC && LEAN) ? __any_sync(FULL, big) : true;
    } else {
      for (int i = w.lane; i < p.nKS; i += 32) wp_smem[i] = __ldg(src + i);
      w.wrap = true;
    }
    w.wp = wp_smem;
  } else {
    w.wp = src;
    w.wrap = true;
  }
  __syncwarp();
  const bool noexit = (p.flags & MRV_DIAG_NO_EARLY_EXIT) != 0;
  w.rake = QUERY == Q_MOTVAL && !(p.flags & MRV_PACK_LINEAR);
  w.nb = (w.T + p.W - 1) >> p.lgW;
  w.te = p.t_end > 0 ? min(w.T, p.t_end) : w.T;
  w.tb = min(max(p.t_begin, 0), w.te);
  uint32_t evaluated = 0;
  if (QUERY == Q_MOTVAL) {
    const bool env = (p.flags & (MRV_CHECK_ENV | MRV_CHECK_SELF)) != 0;   // CC(S_i, E) incl. self
    const bool hier = env && (p.flags & MRV_ORDER_HIERARCHICAL);
    bool invalid = false;
    for (int pass = hier ? 0 : 1; pass < 2; ++pass) {
      const bool do_env = env && (pass == 0 || !hier);
      const bool do_rr = pass == 1;
      for (int c = slice; c < w.nb; c += p.n_slices) {
        if (!noexit) {
          if (invalid) break;
          if (p.n_slices > 1) {
            int v = 1;
            if (w.lane == 0) v = *reinterpret_cast<volatile const uint8_t*>(p.out_valid + m);
            if (__shfl_sync(FULL, v, 0) == 0) {
              invalid = true;
              break;
            }
          }
        }
        set_batch(w, c, p.W, p.lgW);
        if (w.amask == 0) continue;   // outside the time window
        bool hit = false;
        if (p.fuse_env) {   // FK with the obstacle broad + narrow phase in its lanes
          if (PP) pp_request_rows<COUNT>(p, sv, w, cnt);   // (partners' rows in flight during the walk)
          hit = fk_env_fused<COUNT, LEAN, PP>(p, sv, w, !noexit, cnt);
          if (PP) asm volatile("cp.async.wait_all;" ::: "memory");
          __syncwarp();
        } else {
          fk_stage<QUERY, COUNT, LEAN, PP>(p, sv, w, cnt);
          __syncwarp();
          if (do_env) hit = env_stage<COUNT>(p, sv, w, !noexit, cnt);
        }
        ++evaluated;
        if (do_rr && !(hit && !noexit)) hit |= rr_stage<Q_MOTVAL, COUNT, false, PP, T8>(p, sv, w, !noexit, cnt) != 0;
        if (hit) invalid = true;
        __syncwarp();
      }
      if (invalid && !noexit) break;
    }
    if (w.lane == 0) {
      if (p.n_slices == 1) p.out_valid[m] = invalid ? 0 : 1;
      else if (invalid) p.out_valid[m] = 0;
    }
  } else {
    const uint32_t P = (uint32_t)p.sc.n_pairs;
    uint32_t kmin = MRV_NO_CONFLICT;
    if (P > 0) {
      const int c0 = w.tb >> p.lgW, c1 = (w.te + p.W - 1) >> p.lgW;   // linear batches covering [tb, te)
      for (int c = c0 + slice; c < c1; c += p.n_slices) {
        if (!noexit) {
          if (kmin != MRV_NO_CONFLICT) break;
          if (p.n_slices > 1) {
            uint32_t g = 0;
            if (w.lane == 0) g = *reinterpret_cast<volatile const uint32_t*>(p.out_key + m);
            g = __shfl_sync(FULL, g, 0);
            if (g != MRV_NO_CONFLICT && (uint32_t)(c << p.lgW) > g / P) break;
          }
        }
        set_batch(w, c, p.W, p.lgW);
        fk_stage<QUERY, COUNT, LEAN>(p, sv, w, cnt);
        __syncwarp();
        ++evaluated;
        const uint32_t kb = rr_stage<Q_FFC, COUNT, LEAN, false, T8>(p, sv, w, !noexit, cnt);
        kmin = min(kmin, kb);
        if (p.n_slices > 1 && kb != MRV_NO_CONFLICT && w.lane == 0) atomicMin(p.out_key + m, kb);
        __syncwarp();
      }
    }
    if (p.n_slices == 1 && w.lane == 0) p.out_key[m] = kmin;
  }
  if (p.effort && w.lane == 0) {
    if (p.n_slices == 1) p.effort[m] = evaluated;
    else atomicAdd(p.effort + m, evaluated);
  }
}

// ------------------------------------------------------------------ MotVal spread packing
// The production MotVal launch (fixed or per-motion T, whole horizon, default flags, the
// fused FK + obstacle path at W = 8).  Alg. 1's answer is "valid iff no state of the motion
// collides"; its batch size and batch order decide only how much is
// evaluated before the first hit.  Here a warp keeps up to W motions in flight (slots)
// and fills its W state lanes from them every batch: while motions remain to be grabbed
// each gets one lane, and as the supply runs dry the survivors share the lanes (a lone
// motion gets all W, as in the one-motion batch).  Each motion visits its timesteps in
// the order t_b = (T/2 + b * step) mod T, step ~ 0.618 T coprime with T: a bijection on
// [0, T) that spreads successive states over the path as the rake does (PAPER.md:246-
// 248) at one state per batch, starting in the middle (the start state of a planner's
// motion is a validated tree node).  DESIGN.md reading c.28; MRV_PACK_SEQUENTIAL runs
// Alg. 1's own batch loop instead (process_item).

// A motion's spread step: the integer nearest 0.618 T made coprime with T (per-motion T;
// the launcher computes the fixed-T one).  T <= kStepTab: a compile-time table.
constexpr uint32_t kStepTab = 4096;
struct StepTable {
  uint16_t v[kStepTab + 1];
};
constexpr StepTable make_step_table() {
  StepTable t{};
  for (uint32_t T = 1; T <= kStepTab; ++T) {
    uint32_t s = (T * 618034u + 500000u) / 1000000u;
    if (s < 1) s = 1;
    for (;; ++s) {
      uint32_t a = s, b = T;
      while (b) {
        const uint32_t r = a % b;
        a = b;
        b = r;
      }
      if (a == 1u) break;
    }
    t.v[T] = (uint16_t)(s % T);
  }
  return t;
}
__device__ const StepTable kSpreadSteps = make_step_table();

__device__ __noinline__ uint32_t spread_step(uint32_t T) {
  uint32_t s = max(1u, __float2uint_rn(0.6180340f * (float)T));
  for (;; ++s) {
    uint32_t a = s, b = T;
    while (b) {
      const uint32_t r = a % b;
      a = b;
      b = r;
    }
    if (a == 1u) break;
  }
  return s % T;
}

template <bool COUNT, bool LEAN, bool T8 = false>
__device__ void run_spread(const KParams& p, const SV& sv, Warp& w, float* wp_smem, Counters& cnt) {
  const int W = p.W;
  const unsigned long long M = (unsigned long long)p.M;
  const unsigned long long tail_guard = (unsigned long long)p.grab * gridDim.x * (blockDim.x >> 5) * 2ull;
  const bool vec = ((reinterpret_cast<uintptr_t>(p.wp) & 15u) == 0) && ((p.nKS & 3) == 0);
  const int nv = vec ? p.nKS >> 2 : p.nKS;   // copy units (float4 or float) per motion block
  const float inv_nv = 1.0f / (float)nv;
  const bool slot_lane = w.lane < W;
  const unsigned lt = (1u << w.lane) - 1u;
  // slot state, held by lane g < W: its motion, next timestep, states left, T and step
  long long sm = 0;
  uint32_t st = 0, left = 0, own = 0, sT = (uint32_t)p.Tfix, sstep = p.sp_step;
  bool live = false;
  unsigned long long nx = 0, end = 0;   // grabbed items not yet started (warp-uniform)
  bool dry = false;
  w.T = p.Tfix;
  w.Tr = nullptr;
  w.t0 = 0;
  w.tb = 0;
  w.te = p.Tfix;
  w.rake = false;
  w.wrap = true;
  w.wp = wp_smem;
  w.c = 0;
  w.nb = 1;
  for (;;) {
    // 1. refill empty slots from the warp's grabbed range (guided grabbing as in the
    //    one-motion loop), staging each new motion's waypoint block into its slot
    unsigned need = __ballot_sync(FULL, w.lane < p.sp_slots && !live);
    while (need && !dry) {
      if (nx >= end) {
        const unsigned long long g = nx + tail_guard < M ? (unsigned long long)p.grab : 1ull;
        unsigned long long it0 = 0;
        if (w.lane == 0) it0 = atomicAdd(p.work, g);
        it0 = __shfl_sync(FULL, it0, 0);
        if (it0 >= M) {
          dry = true;
          break;
        }
        nx = it0;
        end = min(it0 + g, M);
      }
      const int k = (int)min((unsigned long long)__popc(need), end - nx);
      const bool mine = ((need >> w.lane) & 1u) && __popc(need & lt) < k;
      if (mine) {
        sm = (long long)nx + __popc(need & lt);
        live = true;
        if (!LEAN && p.Tm) {   // per-motion T (device memory): T < 1 is reported, the motion left valid
          const int Tm = p.Tm[sm];
          if (Tm < 1) {
            atomicOr(p.dev_status, (uint32_t)MRV_DEVERR_TIMESTEPS);
            p.out_valid[sm] = 1;
            live = false;
          } else {
            sT = (uint32_t)Tm;
            sstep = sT <= kStepTab ? (uint32_t)kSpreadSteps.v[sT] : spread_step(sT);
          }
        }
        st = sT >> 1;
        left = sT;
      }
      const unsigned newm = __ballot_sync(FULL, mine);
      for (int i = w.lane; i < k * nv; i += 32) {
        const int q = (int)(((float)i + 0.5f) * inv_nv), e = i - q * nv;   // i / nv, i % nv
        unsigned mm = newm;
        for (int j = 0; j < q; ++j) mm &= mm - 1u;
        const int g = __ffs(mm) - 1;                                       // the q-th new slot
        MRV_CHECK(q < k && g >= 0 && g < W && e >= 0 && e < nv && nx + q < M);
        const size_t src = (size_t)(nx + q) * nv + e;
        if (vec) reinterpret_cast<float4*>(wp_smem)[g * nv + e] = __ldg(reinterpret_cast<const float4*>(p.wp) + src);
        else wp_smem[g * nv + e] = __ldg(p.wp + src);
      }
      need &= ~newm;
      nx += k;
    }
    const unsigned livem = __ballot_sync(FULL, slot_lane && live);
    if (!livem) break;
    __syncwarp();
    // 2. the W state lanes over the live motions in slot order: W / L each, the first
    //    W % L one more; owner and index-within-motion maps, 4 bits per lane
    const int s = w.lane & (W - 1);
    int g = s, k = 0;
    if (livem == (1u << W) - 1u) {   // every slot live (the steady state): one lane each
      own = 1u << w.lane;
    } else {
      const int L = __popc(livem), base = W / L, extra = W - base * L;
      uint32_t omap = 0, kmap = 0;
      if (slot_lane && live) {
        const int rk = __popc(livem & lt);
        const int n = base + (rk < extra ? 1 : 0), off = rk * base + min(rk, extra);
        own = ((1u << n) - 1u) << off;
        const uint32_t nib = (uint32_t)(((1ull << (4 * n)) - 1ull) << (4 * off));
        omap = ((uint32_t)w.lane * 0x11111111u) & nib;
        kmap = (uint32_t)((0x76543210ull << (4 * off)) & nib);
      }
      omap = __reduce_or_sync(FULL, omap);
      kmap = __reduce_or_sync(FULL, kmap);
      g = (omap >> (4 * s)) & 15;
      k = (kmap >> (4 * s)) & 15;
    }
    MRV_CHECK(g >= 0 && g < W && ((livem >> g) & 1u) && k >= 0 && k < W);
    const uint32_t gst = __shfl_sync(FULL, st, g), gleft = __shfl_sync(FULL, left, g);
    const uint32_t gT = __shfl_sync(FULL, sT, g), gstep = __shfl_sync(FULL, sstep, g);
    w.gmask = __shfl_sync(FULL, own, g);
    uint32_t t = gst;
    for (int i = 0; i < k; ++i) {
      t += gstep;
      t = t >= gT ? t - gT : t;
    }
    w.mt = (int)t;
    w.mT = (int)gT;
    w.mwp = wp_smem + g * p.nKS;
    w.amask = __ballot_sync(FULL, slot_lane && (uint32_t)k < gleft);
    // 3. the batch, Alg. 1's combined order: FK + CC(S_i, E), then CC(S_i, S_j) for the
    //    states whose motion is still open
    uint32_t hits = 0;
    if (p.fuse_env) {
      hits = fk_env_fused<COUNT, LEAN>(p, sv, w, true, cnt);
    } else {   // (teams the fused walk does not cover: more than 4 robots, general chains, bodies)
      fk_stage<Q_MOTVAL, COUNT, LEAN>(p, sv, w, cnt);
      __syncwarp();
      if (p.flags & MRV_CHECK_ENV) hits = env_stage<COUNT>(p, sv, w, true, cnt);
    }
    __syncwarp();
    if (hits) w.amask &= ~dead_states(w, hits);
    if (w.amask) hits |= rr_stage<Q_MOTVAL, COUNT, false, false, T8>(p, sv, w, true, cnt);
    __syncwarp();
    // 4. a hit ends the motion (invalid); else it advances by its lanes, valid after T states
    if (slot_lane && live) {
      if (hits & own) {
        p.out_valid[sm] = 0;
        live = false;
      } else {
        const uint32_t n = (uint32_t)__popc(own);
        if (left <= n) {
          p.out_valid[sm] = 1;
          live = false;
        } else {
          left -= n;
          for (uint32_t i = 0; i < n; ++i) {
            st += sstep;
            st = st >= sT ? st - sT : st;
          }
        }
      }
    }
  }
}

// ------------------------------------------------------------------ scene staging (1-D TMA bulk copy)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void stage_scene(uint8_t* dst, const uint8_t* src, uint32_t bytes, uint64_t* bar) {
  const uint32_t b = smem_u32(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    constexpr uint32_t kChunk = 32768;
    for (uint32_t off = 0; off < bytes; off += kChunk) {
      const uint32_t n = min(kChunk, bytes - off);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(dst + off)),
          "l"(src + off), "r"(n), "r"(b)
          : "memory");
    }
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(b),
      "r"(0)
      : "memory");
  __syncthreads();
}

// GTAIL: the tail tables (obstacles, grid, self / unpruned segments) are read from the blob
// in global memory rather than from the staged smem copy -- a separate instance so that
// the staged case keeps shared-space (LDS) addressing for every table
// TILE (LGW = 3): the tiled level 1 compiled in -- every W = 8 instance except FFC's general
// one on scenes without it (cfg4-class teams: the larger code measured 1.5 % slower there)
template <int QUERY, bool COUNT, int LGW, bool FIXED = false, bool GTAIL = false, bool PP = false,
          bool TILE = (QUERY == Q_MOTVAL || FIXED)>
// (launch bounds: the lean FFC instance may run kMaxWarpsFfc warps with compact frames; the other
// FFC instances keep kFfcWarpsFull -- the tighter register budget cost the general one 6 %)
__global__ void __launch_bounds__((QUERY == Q_FFC ? (FIXED ? kMaxWarpsFfc : kFfcWarpsFull) : kMaxWarpsPerCta) * 32, 1) mrv_query_kernel(const __grid_constant__ KParams p0) {
  // LGW > 0: the batch width is a compile-time constant (W = 8 specialisation)
  KParams p = p0;
  if (!COUNT) p.counters = nullptr;   // (folds the per-access counting of the PP accessors away)
  if (LGW > 0) {
    p.lgW = LGW;
    p.W = 1 << LGW;
    p.wi = LGW - 2;
  }
  if (FIXED) {   // the lean instances: the launcher guarantees these values (launch_query)
    p.sc.group_lg = 3;
    if (!PP) {
      p.focus = -1;
      p.partners = 0;
      p.pp_table = nullptr;
    }
    p.flags = QUERY == Q_MOTVAL ? (uint32_t)MRV_CHECK_ENV : 0u;
    p.t_begin = 0;
    p.t_end = 0;
    p.n_slices = 1;
    p.Trob = nullptr;
    p.Tm = nullptr;
    p.effort = nullptr;
    p.wp_in_smem = 1;
    if (QUERY == Q_MOTVAL) {
      p.fuse_env = 1;
      p.spread = PP ? 0 : 1;
      p.qcap = PP ? kQueueCap : kSpreadQCap;
      p.ncap = PP ? kNarrowCap : kSpreadNCap;
    }
  }
  if (QUERY != Q_MOTVAL || PP) p.spread = 0;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar;
  stage_scene(smem, p.blob, p.stage_bytes, &bar);
  // the tail tables: the staged copy, unless this is the global-tail instance (the launcher
  // stages the whole blob for every other instance that reads the tail)
  const uint8_t* tail = GTAIL ? p.blob : smem;
  SV sv = make_sv_q<FIXED>(smem, tail, p.sc, p.wi);
  if (!FIXED && (p.flags & MRV_DIAG_NO_BROADPHASE)) {
    // diagnostic: the robot-robot segments without the static reach pruning (every
    // supergroup pair of every robot pair), from the tail
    sv.rr_segs = reinterpret_cast<const uint4*>(tail + p.sc.off_rr_segs_all);
    p.sc.n_rr_segs = p.sc.n_rr_segs_all;
  }
  if (PP && p.pp_nseg > 0) {   // the (focus, partner) segments, after every warp's scratch
    uint32_t* segs = reinterpret_cast<uint32_t*>(smem + p.stage_bytes + (blockDim.x >> 5) * p.warp_bytes);
    for (int i = threadIdx.x; i < p.pp_nseg * 8; i += blockDim.x) segs[i] = __ldg(p.pp_segs + i);
    __syncthreads();
    sv.rr_segs = reinterpret_cast<const uint4*>(segs);
    p.sc.n_rr_segs = p.pp_nseg;
  }
  const int warp = threadIdx.x >> 5;
  uint8_t* ws = smem + p.stage_bytes + warp * p.warp_bytes;
  Warp w;
  w.lane = threadIdx.x & 31;
  w.frames = reinterpret_cast<float*>(ws + p.off_frames);
  w.bc = (QUERY == Q_MOTVAL && (!p.fuse_env || PP)) ? reinterpret_cast<float4*>(ws + p.off_bc) : nullptr;
  if (PP) {   // only the focus robot's frames / group bounds live in smem: bases shifted so that
              // the usual link_off / group indices address them
    w.frames -= p.pp_fbase;
    w.bc -= (size_t)p.pp_gbase << p.lgW;
  }
  w.sbc = reinterpret_cast<float4*>(ws + p.off_sbc);
  w.nq = reinterpret_cast<uint2*>(ws + p.off_nq);
  w.nsc = reinterpret_cast<float4*>(ws + p.off_nsc);
  w.queue = reinterpret_cast<uint32_t*>(ws + p.off_queue);
  float* wp_smem = reinterpret_cast<float*>(ws + p.off_wp);
  w.wp_smem = wp_smem;
  Counters cnt;
  if (COUNT)
#pragma unroll
    for (int i = 0; i < MRV_NUM_COUNTERS; ++i) cnt.v[i] = 0;
  const unsigned long long n_items = (unsigned long long)p.M * (unsigned long long)p.n_slices;
  const unsigned long long tail_guard = (unsigned long long)p.grab * gridDim.x * (blockDim.x >> 5) * 2ull;
  unsigned long long seen = 0;
  if (QUERY == Q_MOTVAL && !PP && p.spread) {
    run_spread<COUNT, FIXED, LGW == 3 && TILE>(p, sv, w, wp_smem, cnt);
  } else {
    for (;;) {
      unsigned long long it0 = 0;
      // guided: chunks of p.grab items while plenty remain, single items near the end
      // (a chunk of long FFC motions grabbed last would otherwise leave a long tail)
      const unsigned long long g = seen + tail_guard < n_items ? (unsigned long long)p.grab : 1ull;
      if (w.lane == 0) it0 = atomicAdd(p.work, g);
      it0 = __shfl_sync(FULL, it0, 0);
      if (it0 >= n_items) break;
      seen = it0;
      const unsigned long long it1 = min(it0 + g, n_items);
      for (unsigned long long it = it0; it < it1; ++it) {
        const int64_t m = (int64_t)(it / (unsigned long long)p.n_slices);
        const int slice = (int)(it % (unsigned long long)p.n_slices);
        process_item<QUERY, COUNT, FIXED, PP, LGW == 3 && TILE>(p, sv, w, m, slice, wp_smem, cnt);
      }
    }
  }
  if (COUNT) {
#pragma unroll
    for (int i = 0; i < MRV_NUM_COUNTERS; ++i) {
      unsigned long long v = cnt.v[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
      if (w.lane == 0 && v) atomicAdd(p.counters + i, v);
    }
  }
}

// ------------------------------------------------------------------ K3: SpheresFK export
struct OutSink {
  const SV* sv;
  float* out;   // [total_spheres][3] of this query
  __device__ __forceinline__ void operator()(int link, const float* M) {
    const int4 L = sv->link[link];
    for (int g = L.z; g < L.z + L.w; ++g) {
      const int4 G = sv->group[g];
      for (int k = G.y; k < G.y + G.z; ++k) {
        const float4 sp = sv->sphere[k];
        float x, y, z;
        xform(M, sp.x, sp.y, sp.z, x, y, z);
        float* o = out + 3 * (size_t)sv->sphere_index[k];
        o[0] = x; o[1] = y; o[2] = z;
      }
    }
  }
};

__global__ void mrv_fk_kernel(const DevScene sc, const uint8_t* blob, const float* wp, const int32_t* Tm, int32_t Tfix,
                              const int32_t* Trob, int64_t M, int32_t K, int32_t S, int64_t nq, const int64_t* motion,
                              const int32_t* tq, float* out) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= nq * sc.n_robots) return;
  const int64_t q = x / sc.n_robots;
  const int r = (int)(x % sc.n_robots);
  const SV sv = make_sv(blob, blob, sc, 0);
  float* oq = out + (size_t)q * sc.n_spheres * 3;
  const int64_t m = motion[q];
  const int t = tq[q];
  int T = 0;
  if (m >= 0 && m < M) {
    if (Trob) {
      T = 1;
      for (int rr = 0; rr < sc.n_robots; ++rr) T = max(T, Trob[m * sc.n_robots + rr]);
    } else {
      T = Tm ? Tm[m] : Tfix;
    }
  }
  if (m < 0 || m >= M || t < 0 || t >= T) {
    const int4 rb = sv.robot[3 * r + 1];
    for (int k = rb.z; k < rb.z + rb.w; ++k) {
      float* o = oq + 3 * (size_t)sv.sphere_index[k];
      o[0] = o[1] = o[2] = __int_as_float(0x7fc00000);
    }
    return;
  }
  const int Tr = Trob ? Trob[m * sc.n_robots + r] : T;   // stay at goal after the robot's own path
  const Interp ip = interp_setup(min(t, Tr - 1), Tr, K);
  OutSink sink{&sv, oq};
  robot_fk(sv, r, ip, wp + (size_t)m * sc.n_robots * K * S + (size_t)r * K * S, S, sink);
}

// ------------------------------------------------------------------ K4: PP-ST-RRT partner table
// Row t: supergroup bounds [n_super] | link frames [n_links][3] ({c0, tx}, {c1, ty}, {tz}) |
// group bounds [n_groups] of the partner robots at absolute timestep t (robot_fk + the FK
// sink's bound arithmetic, so the rows hold what fk_stage would have written).
struct TableSink {
  const SV* sv;
  float4* row;
  int nsup;
  FrameSink fs;   // W = 1, s = 0: bc -> the row's group bounds, sbc -> its supergroup bounds
  __device__ __forceinline__ void operator()(int link, const float* M) {
    float4* f = row + nsup + 3 * link;
    f[0] = make_float4(M[0], M[4], M[8], M[3]);
    f[1] = make_float4(M[1], M[5], M[9], M[7]);
    f[2] = make_float4(M[11], 0.0f, 0.0f, 0.0f);
    const int4 L = sv->link[link];
    for (int g = L.z; g < L.z + L.w; ++g) fs.group(M, sv->gbound[g], g, sv->group_super[g]);
  }
};

__global__ void mrv_pp_table_kernel(const DevScene sc, const uint8_t* blob, const float* wp, const int32_t* Tm,
                                    int32_t Tfix, const int32_t* Trob, int32_t K, int32_t S,
                                    unsigned long long partners, int32_t H, int32_t rec, float4* table,
                                    uint32_t* dev_status) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= (int64_t)H * sc.n_robots) return;
  const int t = (int)(x / sc.n_robots), r = (int)(x % sc.n_robots);
  if (!((partners >> r) & 1ull)) return;
  const SV sv = make_sv(blob, blob, sc, 0);
  int T = Trob ? Trob[r] : (Tm ? Tm[0] : Tfix);
  if (T < 1) {
    atomicOr(dev_status, (uint32_t)MRV_DEVERR_TIMESTEPS);
    T = 1;
  }
  const Interp ip = interp_setup(min(t, T - 1), T, K);   // stay at the goal after T_r
  TableSink sink;
  sink.sv = &sv;
  sink.row = table + (size_t)t * rec;
  sink.nsup = sc.n_super;
  sink.fs.sv = &sv;
  sink.fs.frames = nullptr;
  sink.fs.bc = sink.row + sc.n_super + 3 * sc.n_links;
  sink.fs.sbc = sink.row;
  sink.fs.W = 1;
  sink.fs.s = 0;
  sink.fs.reset();
  robot_fk(sv, r, ip, wp + (size_t)r * K * S, S, sink);
}

}  // namespace mrv

// ==================================================================== C ABI launchers
using namespace mrv;

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// only_robot >= 0: the batch holds that robot alone (PP-ST-RRT candidates)
#ifndef PP_DEFAULT_LGW
#define PP_DEFAULT_LGW 5   // W = 32: the focus robot's FK fills every lane
#endif

mrv_status validate_batch(const mrv_scene* s, const mrv_motion_batch* b, int only_robot = -1) {
  if (!s || !b) return MRV_EINVAL;
  if (b->n_motions < 0 || b->n_waypoints < 1) return MRV_EINVAL;
  if (b->n_waypoints > MRV_MAX_KNOTS) return MRV_EUNSUPPORTED;   // interp_setup's quotient bound
  int max_dof = 0;
  for (int r = 0; r < s->n_robots; ++r) {
    const int4* rec = reinterpret_cast<const int4*>(s->h_blob.data() + s->ds.off_robot) + 3 * r;
    if (only_robot < 0 || r == only_robot) max_dof = std::max(max_dof, rec->y);
  }
  if (b->dof_stride < max_dof) return MRV_EINVAL;
  if (b->n_motions > 0 && !b->waypoints) return MRV_EINVAL;
  if (!b->robot_timesteps && !b->n_timesteps && b->fixed_timesteps < 1) return MRV_EINVAL;
  return MRV_OK;
}

int pick_lgW(const mrv_scene* s, const mrv_launch_opts* o, bool pp = false) {
  if (o && o->states_per_batch) {
    switch (o->states_per_batch) {
      case 4: return 2;
      case 8: return 3;
      case 16: return 4;
      case 32: return 5;
      default: return -1;
    }
  }
  if (pp) return PP_DEFAULT_LGW;      // PP: one FK robot
  return s->n_robots <= 2 ? 4 : 3;   // W = 16 for 1-2 robots (fills the FK lanes), else W = 8
}

struct PPArgs {   // mrv_pp_motval_batch
  const float4* table;
  const int32_t* t0;
  int32_t H, focus;
  uint64_t partners;
};

int32_t pp_rec_f4(const mrv_scene* s) { return s->ds.n_super + 3 * s->ds.n_links + s->ds.n_groups; }

template <int QUERY>
mrv_status launch_query(const mrv_scene* s, const mrv_motion_batch* b, uint32_t flags, void* out, void* stream,
                        const mrv_launch_opts* o, bool dry_run = false, const PPArgs* pp = nullptr) {
  if (pp && (!s || pp->focus < 0 || pp->focus >= s->n_robots)) return MRV_EINVAL;
  mrv_status st = validate_batch(s, b, pp ? pp->focus : -1);
  if (st != MRV_OK) return st;
  if (pp) {
    if (QUERY != Q_MOTVAL || b->robot_timesteps || (flags & MRV_FOCUS)) return MRV_EINVAL;
    if (b->n_motions > 0 && (!pp->table || !pp->t0 || (reinterpret_cast<uintptr_t>(pp->table) & 15u))) return MRV_EINVAL;
    if (pp->H < 1) return MRV_EINVAL;
  }
  if (b->n_motions > 0 && !out) return MRV_EINVAL;
  if (QUERY == Q_FFC && !b->robot_timesteps && !b->n_timesteps && s->n_pairs > 0 &&
      (uint64_t)b->fixed_timesteps * (uint64_t)s->n_pairs >= 0xFFFFFFFFull)
    return MRV_ERANGE;
  if (b->n_motions == 0) return MRV_OK;
  int lgW = pick_lgW(s, o, pp != nullptr);
  if (lgW < 0) return MRV_EINVAL;
  if (o && o->n_slices < 0) return MRV_EINVAL;
  int max_wpc = QUERY == Q_FFC ? kFfcWarpsFull : kMaxWarpsPerCta;   // (FFC: kMaxWarpsFfc with compact frames)
  const int req_wpc = o ? o->warps_per_cta : 0;
  if (req_wpc < 0 || req_wpc > kMaxWarpsFfc) return MRV_EINVAL;
  if (req_wpc > (QUERY == Q_FFC ? kMaxWarpsFfc : kMaxWarpsPerCta)) return MRV_EUNSUPPORTED;
  DeviceGuard guard(s->device);
  cudaStream_t strm = static_cast<cudaStream_t>(stream);

  KParams p;
  std::memset(&p, 0, sizeof p);
  p.sc = s->ds;
  p.blob = static_cast<const uint8_t*>(s->d_blob);
  p.wp = b->waypoints;
  p.Tm = b->robot_timesteps ? nullptr : b->n_timesteps;
  p.Trob = b->robot_timesteps;
  p.M = b->n_motions;
  p.Tfix = b->fixed_timesteps;
  p.K = b->n_waypoints;
  p.S = b->dof_stride;
  const int64_t nKS = (int64_t)(pp ? 1 : s->n_robots) * b->n_waypoints * b->dof_stride;
  if (nKS > 0x7FFFFFFF) return MRV_ERANGE;
  p.nKS = (int32_t)nKS;
  p.flags = flags;
  p.out_valid = QUERY == Q_MOTVAL ? static_cast<uint8_t*>(out) : nullptr;
  p.out_key = QUERY == Q_FFC ? static_cast<uint32_t*>(out) : nullptr;
  p.counters = o ? reinterpret_cast<unsigned long long*>(o->counters) : nullptr;
  p.effort = o ? o->batches_evaluated : nullptr;
  p.dev_status = s->d_status;
  p.t_begin = o ? o->t_begin : 0;
  p.t_end = o ? o->t_end : 0;
  if (p.t_begin < 0) return MRV_EINVAL;
  p.focus = -1;
  p.partners = 0;
  if (flags & MRV_FOCUS) {
    if (!o || o->focus_robot < 0 || o->focus_robot >= s->n_robots) return MRV_EINVAL;
    p.focus = o->focus_robot;
    p.partners = o->partner_mask & ~(1ull << o->focus_robot);
    if (s->n_robots < 64) p.partners &= (1ull << s->n_robots) - 1ull;
  }
  if (pp) {
    p.focus = pp->focus;
    p.partners = pp->partners & ~(1ull << pp->focus);
    if (s->n_robots < 64) p.partners &= (1ull << s->n_robots) - 1ull;
    p.pp_table = pp->table;
    p.pp_t0 = pp->t0;
    p.pp_H = pp->H;
    p.pp_rec = pp_rec_f4(s);
    // level-1 segments of the (focus supergroup, partner supergroup) pairs only: each focus
    // supergroup against the partners' supergroups, kRRSegLen per segment (else the scene's
    // segments with a per-test filter)
    const int4* rec = reinterpret_cast<const int4*>(s->h_blob.data() + s->ds.off_robot);
    std::vector<uint32_t> part;
    for (int j = 0; j < s->n_robots; ++j)
      if ((p.partners >> j) & 1ull)
        for (int g = rec[3 * j + 2].x; g < rec[3 * j + 2].x + rec[3 * j + 2].y; ++g) part.push_back((uint32_t)g);
    const int fa0 = rec[3 * pp->focus + 2].x, nfa = rec[3 * pp->focus + 2].y;
    const int per = ((int)part.size() + kRRSegLen - 1) / kRRSegLen;
    if (nfa * per <= kPPSegs && !part.empty()) {
      std::lock_guard<std::mutex> lk(s->cfg_mu);
      for (const auto& e : s->pp_seg_cache)
        if (e.focus == pp->focus && e.partners == p.partners) {
          p.pp_segs = static_cast<const uint32_t*>(e.d);
          p.pp_nseg = e.n;
        }
      if (!p.pp_segs) {   // built once per (focus, partner set), kept until mrv_destroy_scene
        std::vector<uint32_t> tab;
        for (int a = fa0; a < fa0 + nfa; ++a)
          for (size_t c0 = 0; c0 < part.size(); c0 += kRRSegLen) {
            const size_t c1 = std::min(part.size(), c0 + (size_t)kRRSegLen);
            uint32_t rec8[8] = {(uint32_t)a | ((uint32_t)(c1 - c0) << 16), 0u, 0u, 0u, 0u, 0u, 0u, 0u};
            for (size_t c = c0; c < c1; ++c) rec8[2 + (c - c0)] = part[c];   // (word 1: rank_min, unused)
            tab.insert(tab.end(), rec8, rec8 + 8);
          }
        void* d = nullptr;
        if (cudaMalloc(&d, tab.size() * 4) != cudaSuccess ||
            cudaMemcpy(d, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
          cudaGetLastError();
          if (d) cudaFree(d);
          return MRV_ENOMEM;
        }
        s->pp_seg_cache.push_back({pp->focus, p.partners, d, (int)(tab.size() / 8)});
        p.pp_segs = static_cast<const uint32_t*>(d);
        p.pp_nseg = (int)(tab.size() / 8);
      }
    }
  }
  p.wp_in_smem = nKS <= kWpCapFloats;
  p.fuse_env = 0;
  if (QUERY == Q_MOTVAL && (flags & MRV_CHECK_ENV) && !(flags & (MRV_CHECK_SELF | MRV_ORDER_HIERARCHICAL | MRV_FOCUS)) &&
      p.focus < 0 &&
      !b->robot_timesteps && p.wp_in_smem && s->ds.n_cells > 0 && s->fuse_env_ok && s->n_robots * (1 << lgW) <= 32)
    p.fuse_env = 1;
  if (pp && (flags & MRV_CHECK_ENV) && !(flags & (MRV_CHECK_SELF | MRV_ORDER_HIERARCHICAL)) && p.wp_in_smem &&
      s->ds.n_cells > 0) {   // PP: the focus robot's walk with its obstacle broad phase (a fast-DH chain)
    const int4* rec = reinterpret_cast<const int4*>(s->h_blob.data() + s->ds.off_robot) + 3 * pp->focus;
    if (rec[2].z) p.fuse_env = 1;
  }
  // MotVal spread packing (run_spread): the fused path at W = 8, fixed T, whole horizon,
  // early exit, no effort output, no caller-chosen W / slices / packing; p.spread is
  // cleared again below if the launch needs several warps per motion
  // (non-fused teams too: default flags or robot-robot only, no self pairs or focus robot)
  const bool spread_path = p.fuse_env || (!(flags & (MRV_CHECK_SELF | MRV_ORDER_HIERARCHICAL | MRV_FOCUS)) &&
                                          p.focus < 0 && p.wp_in_smem);
  const bool spread_ok = QUERY == Q_MOTVAL && !pp && spread_path && lgW == 3 && !p.Trob && !p.effort &&
                         p.t_begin == 0 && p.t_end <= 0 &&
                         !(flags & (MRV_PACK_LINEAR | MRV_PACK_SEQUENTIAL | MRV_DIAG_NO_EARLY_EXIT)) &&
                         !(o && (o->states_per_batch || o->n_slices > 1)) &&
                         (int64_t)p.nKS * 8 <= (int64_t)kWpCapFloats;
  if (spread_ok) {
    p.spread = 1;
    const uint32_t T = (uint32_t)std::max(1, p.Tfix);   // (per-motion T: each motion's step on the device)
    uint32_t stp = std::max<uint32_t>(1u, (uint32_t)std::llround(0.6180339887498949 * (double)T));
    auto gcd = [](uint32_t a, uint32_t c) { while (c) { const uint32_t r = a % c; a = c; c = r; } return a; };
    while (gcd(stp, T) != 1u) ++stp;
    p.sp_step = stp % T;
  }

  // queue capacities: MotVal's broad-phase queue holds a self-collision round (32 x kSegLen)
  // only with MRV_CHECK_SELF; spread packing trims both queues so that 16 warps' scratch
  // (with its 8 waypoint slots) fits next to the staged prefix
  p.qcap = QUERY == Q_FFC ? kQCap<Q_FFC> : (flags & MRV_CHECK_SELF) ? kQueueCap : p.spread ? kSpreadQCap : kQueueCap;
  p.ncap = QUERY == Q_FFC ? kNCap<Q_FFC> : p.spread ? kSpreadNCap : kNarrowCap;
  const bool count = p.counters != nullptr;
  // The lean W = 8 instance: fixed-offset prefix, 8-sphere groups and the production
  // options (no focus robot, default flags, whole horizon, fixed T with (T - 1)(K - 1) < 2^32, one warp
  // per motion -- enough motions that the slice heuristic below picks 1, no effort
  // output); it folds those launch parameters to constants.
  const uint32_t lean_flags = QUERY == Q_MOTVAL ? (uint32_t)MRV_CHECK_ENV : 0u;
  const bool fixed = s->ds.fixed_layout && s->ds.group_lg == 3 && p.focus < 0 && flags == lean_flags &&
                     p.t_begin == 0 && p.t_end <= 0 && !p.Trob && !p.Tm && !p.effort && p.wp_in_smem &&
                     (uint64_t)(p.Tfix - 1) * (uint64_t)(p.K - 1) < 0x100000000ull &&
                     !(o && o->n_slices > 1) &&
                     b->n_motions >= 2 * (int64_t)s->sm_count * std::max(kMaxWarpsPerCta, kFfcWarpsFull) &&
                     (QUERY == Q_FFC || (p.fuse_env && p.spread));
  // (the lean FFC instance at W = 8 on ds.l1tile bit-2 scenes stores compact link frames:
  // 6 instead of 9 words per link and state, so up to kMaxWarpsFfc warps fit)
  bool cframes = false;
  // per-warp scratch layout; a smaller W if one warp does not fit next to the staged
  // prefix (the tables every query reads)
  const uint32_t prefix = (uint32_t)s->ds.rr_prefix_bytes;
  for (;; --lgW) {
    if (lgW < 2) return MRV_EUNSUPPORTED;
    const int W = 1 << lgW, wi = lgW - 2;
    cframes = QUERY == Q_FFC && fixed && !count && !pp && lgW == 3 && (s->ds.l1tile & 4);
    uint32_t off = 0;
    p.off_wp = off;
    off = align16(off + (p.wp_in_smem ? (uint32_t)nKS * 4u * (p.spread ? 8u : 1u) : 0u));
    p.off_frames = off;
    if (pp) {   // the focus robot's links and groups only (partners stream from the table)
      const int4* rec = reinterpret_cast<const int4*>(s->h_blob.data() + s->ds.off_robot) + 3 * pp->focus;
      const int32_t* lo_tab = reinterpret_cast<const int32_t*>(s->h_blob.data() + s->ds.off_link_off);
      const int lo_stride = s->ds.fixed_layout ? FixedLayout::kLinks : s->ds.n_links;
      p.pp_fbase = lo_tab[(size_t)wi * lo_stride + rec[0].z];
      p.pp_gbase = rec[1].x;
      off = align16(off + (uint32_t)rec[0].w * kFrameWords * W * 4u);
      p.off_bc = off;
      off = align16(off + (uint32_t)rec[1].y * W * 16u);
    } else {
      off = align16(off + (cframes ? (uint32_t)s->ds.n_links * 6u * W * 4u : (uint32_t)s->ds.frame_words[wi] * 4u));
      p.off_bc = off;
      if (QUERY == Q_MOTVAL && !(p.fuse_env && s->n_robots * W <= 32)) off = align16(off + (uint32_t)s->ds.n_groups * W * 16u);
    }
    p.off_sbc = off;
    off = align16(off + (uint32_t)s->ds.n_super * W * 16u);
    p.off_queue = off;
    off = align16(off + (uint32_t)p.qcap * 4u);
    p.off_nq = off;
    off = align16(off + (uint32_t)p.ncap * 8u);
    p.off_nsc = off;
    off = align16(off + 32u * 16u);
    p.warp_bytes = off;
    if ((pp ? s->ds.blob_bytes + (uint32_t)p.pp_nseg * 32u : prefix) + (size_t)off * std::max(1, req_wpc) + 1024 <=
        (size_t)s->max_smem_optin) {
      p.lgW = lgW;
      p.W = W;
      p.wi = wi;
      break;
    }
    if (o && o->states_per_batch) return MRV_EUNSUPPORTED;
  }
  if (cframes) max_wpc = kMaxWarpsFfc;
  if (req_wpc > max_wpc) return MRV_EUNSUPPORTED;

  // Kernel instance and staged tables.  FFC reads only the prefix (the whole blob under
  // MRV_DIAG_NO_BROADPHASE, whose unpruned segments sit in the tail).  MotVal also reads the
  // tail (obstacles, grid, self segments): staged with the prefix, unless that costs
  // resident warps (scenes with many obstacles) -- then the global-tail instance reads it
  // from global memory (L1/L2-cached).  Warps per CTA: the count that keeps the most warps
  // resident per SM (every CTA holds its own copy of the staged tables, so larger CTAs
  // amortise them), or the caller's.  Cached per scene so repeated small calls (ARC-style
  // FFC loops) skip the occupancy queries.
  struct Cand { const void* fn; uint32_t stage; };
  Cand cands[2];
  int n_cands = 0;
  const bool nobp = (flags & MRV_DIAG_NO_BROADPHASE) != 0;
  // the lean PP instance (W = 32): the production pp5 options, as the lean MotVal one
  const bool pp_fixed = QUERY == Q_MOTVAL && pp && s->ds.fixed_layout && s->ds.group_lg == 3 && flags == (uint32_t)MRV_CHECK_ENV &&
                          p.t_begin == 0 && p.t_end <= 0 && !p.Tm && !p.Trob && !p.effort && p.wp_in_smem &&
                          p.fuse_env && (uint64_t)(p.Tfix - 1) * (uint64_t)(p.K - 1) < 0x100000000ull &&
                          !(o && o->n_slices > 1) &&
                          b->n_motions >= 2 * (int64_t)s->sm_count * std::max(kMaxWarpsPerCta, kFfcWarpsFull);
  if (QUERY == Q_MOTVAL && pp) {   // (the tail must be staged: no global-tail PP instance)
    cands[n_cands++] = {count ? (const void*)mrv_query_kernel<Q_MOTVAL, true, 0, false, false, true>
                        : p.lgW == 5 ? (pp_fixed ? (const void*)mrv_query_kernel<Q_MOTVAL, false, 5, true, false, true>
                                                 : (const void*)mrv_query_kernel<Q_MOTVAL, false, 5, false, false, true>)
                                     : (const void*)mrv_query_kernel<Q_MOTVAL, false, 0, false, false, true>,
                        s->ds.blob_bytes};
  } else if (QUERY == Q_MOTVAL) {
    // (the staged copy stops before the tables MotVal never reads from it: the SpheresFK
    // sphere index and, without MRV_DIAG_NO_BROADPHASE, the unpruned segments)
    const uint32_t motval_stage = nobp ? s->ds.blob_bytes : align16((uint32_t)s->ds.off_sphere_index);
    cands[n_cands++] = {count ? (const void*)mrv_query_kernel<Q_MOTVAL, true, 0>
                        : p.lgW == 3 ? (fixed ? (const void*)mrv_query_kernel<Q_MOTVAL, false, 3, true>
                                              : (const void*)mrv_query_kernel<Q_MOTVAL, false, 3>)
                                     : (const void*)mrv_query_kernel<Q_MOTVAL, false, 0>,
                        motval_stage};
    cands[n_cands++] = {count ? (const void*)mrv_query_kernel<Q_MOTVAL, true, 0, false, true>
                        : p.lgW == 3 ? (fixed ? (const void*)mrv_query_kernel<Q_MOTVAL, false, 3, true, true>
                                              : (const void*)mrv_query_kernel<Q_MOTVAL, false, 3, false, true>)
                                     : (const void*)mrv_query_kernel<Q_MOTVAL, false, 0, false, true>,
                        prefix};
  } else {
    cands[n_cands++] = {count ? (const void*)mrv_query_kernel<Q_FFC, true, 0>
                        : p.lgW == 3 ? (fixed ? (const void*)mrv_query_kernel<Q_FFC, false, 3, true>
                                              : s->ds.l1tile ? (const void*)mrv_query_kernel<Q_FFC, false, 3, false, false, false, true>
                                                             : (const void*)mrv_query_kernel<Q_FFC, false, 3>)
                                     : (const void*)mrv_query_kernel<Q_FFC, false, 0>,
                        nobp ? s->ds.blob_bytes : prefix};
  }
  const void* fn = nullptr;
  int wpc = 0, occ = 0;
  size_t smem = 0;
  bool cached = false;
  const uint32_t extra = (uint32_t)p.pp_nseg * 32u;   // PP segments after the warps' scratch
  {
    std::lock_guard<std::mutex> lk(s->cfg_mu);
    for (const auto& c : s->cfg_cache)
      if (c.key == cands[0].fn && c.warp_bytes == p.warp_bytes && c.req_wpc == req_wpc &&
          c.stage_key == cands[0].stage + extra) {
        fn = c.fn;
        wpc = c.wpc;
        occ = c.occ;
        smem = c.smem;
        p.stage_bytes = c.stage_bytes;
        cached = true;
        break;
      }
  }
  if (!cached) {
    int best_warps = 0;
    for (int ci = 0; ci < n_cands; ++ci) {
      if (cudaFuncSetAttribute(cands[ci].fn, cudaFuncAttributeMaxDynamicSharedMemorySize, s->max_smem_optin - 1024) !=
          cudaSuccess) {
        cudaGetLastError();
        return MRV_ECUDA;
      }
      for (int cand = req_wpc ? req_wpc : max_wpc; cand >= (req_wpc ? req_wpc : 1); --cand) {
        const size_t sm_c = cands[ci].stage + (size_t)cand * p.warp_bytes + extra;
        if (sm_c + 1024 > (size_t)s->max_smem_optin) continue;
        int oc = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc, cands[ci].fn, cand * 32, sm_c) != cudaSuccess) {
          cudaGetLastError();
          return MRV_ECUDA;
        }
        if (oc * cand > best_warps) {   // strictly more: the staged-tail candidate wins ties
          best_warps = oc * cand;
          fn = cands[ci].fn;
          wpc = cand;
          occ = oc;
          smem = sm_c;
          p.stage_bytes = cands[ci].stage;
        }
      }
    }
    if (occ >= 1) {
      std::lock_guard<std::mutex> lk(s->cfg_mu);
      s->cfg_cache.push_back({cands[0].fn, cands[0].stage + extra, fn, p.warp_bytes, p.stage_bytes, req_wpc, wpc, occ, smem});
      if (std::getenv("MRV_LAUNCH_LOG"))   // diagnostic: the configuration each new launch shape gets
        std::fprintf(stderr, "mrv launch: %s W=%d fixed=%d spread=%d instance=%d/%d warp_bytes=%u stage=%u "
                     "(prefix %u, blob %u) wpc=%d occ=%d smem=%zu\n", QUERY == Q_MOTVAL ? "motval" : "ffc", p.W,
                     (int)(fixed || pp_fixed), p.spread, fn == cands[0].fn ? 0 : 1, n_cands, p.warp_bytes, p.stage_bytes, prefix,
                     (uint32_t)s->ds.blob_bytes, wpc, occ, smem);
    }
  }
  if (occ < 1) return req_wpc ? MRV_EUNSUPPORTED : MRV_ECUDA;
  const int blocks = s->sm_count * occ;
  const int64_t total_warps = (int64_t)blocks * wpc;
  // batches per motion; per-motion T lives on the device: MotVal assumes up to 16 batches
  // (extra slices of a shorter motion find no batch; an invalid flag stops the others),
  // FFC keeps one warp per motion (measured: its slices past the conflict cost more than
  // the parallelism returns at cfg2's size)
  const int nb_hint = (b->n_timesteps || b->robot_timesteps) ? (QUERY == Q_MOTVAL ? 16 : 1)
                                                             : std::max(1, (b->fixed_timesteps + p.W - 1) / p.W);
  int ns = o && o->n_slices ? o->n_slices : 1;
  if (!(o && o->n_slices) && b->n_motions < 2 * total_warps)
    ns = (int)std::min<int64_t>(nb_hint, (2 * total_warps + b->n_motions - 1) / b->n_motions);
  p.n_slices = std::max(1, ns);
  if (p.n_slices > 1) p.spread = 0;
  // spread packing's slots: one per 4 motions a warp has to process, at most W (so that a
  // small batch is not taken up by the first warps' slots; measured: cfg3 MotVal 0.58 ->
  // 0.17 ms against one slot per 16 motions, cfg5 unchanged at 2^20 motions and 17-30 %
  // slower at 2^16-2^17; MRV_SPREAD_SLOTS overrides, for experiments)
  p.sp_slots = (int)std::min<int64_t>(p.W, std::max<int64_t>(1, b->n_motions / (4 * total_warps)));
  if (const char* e = std::getenv("MRV_SPREAD_SLOTS")) p.sp_slots = std::max(1, std::min(p.W, std::atoi(e)));
  const int64_t n_items = b->n_motions * p.n_slices;
  p.grab = (int)std::max<int64_t>(1, std::min<int64_t>(8, n_items / (total_warps * 16)));
  if (dry_run) return MRV_OK;   // every check that can fail synchronously has run

  const uint32_t slot = s->ring_next.fetch_add(1) % MRV_MAX_INFLIGHT;
  p.work = s->d_ring + slot;
  if (cudaMemsetAsync(p.work, 0, sizeof(unsigned long long), strm) != cudaSuccess) return MRV_ECUDA;
  if (p.n_slices > 1) {
    if (QUERY == Q_MOTVAL) {
      if (cudaMemsetAsync(out, 1, (size_t)b->n_motions, strm) != cudaSuccess) return MRV_ECUDA;
    } else {
      if (cudaMemsetAsync(out, 0xFF, (size_t)b->n_motions * 4, strm) != cudaSuccess) return MRV_ECUDA;
    }
    if (p.effort && cudaMemsetAsync(p.effort, 0, (size_t)b->n_motions * 4, strm) != cudaSuccess) return MRV_ECUDA;
  }
  void* args[] = {&p};
  if (cudaLaunchKernel(fn, dim3(blocks), dim3(wpc * 32), args, smem, strm) != cudaSuccess) {
    cudaGetLastError();
    return MRV_ECUDA;
  }
  return MRV_OK;
}

}  // namespace

extern "C" {

mrv_status mrv_motval_batch_ex(const mrv_scene* s, const mrv_motion_batch* b, uint32_t flags, uint8_t* out_valid,
                               void* cuda_stream, const mrv_launch_opts* opts) {
  return launch_query<Q_MOTVAL>(s, b, flags, out_valid, cuda_stream, opts);
}

mrv_status mrv_motval_batch(const mrv_scene* s, const mrv_motion_batch* b, uint32_t flags, uint8_t* out_valid,
                            void* cuda_stream) {
  return launch_query<Q_MOTVAL>(s, b, flags, out_valid, cuda_stream, nullptr);
}

mrv_status mrv_ffc_batch_ex(const mrv_scene* s, const mrv_motion_batch* b, uint32_t flags, uint32_t* out_key,
                            void* cuda_stream, const mrv_launch_opts* opts) {
  return launch_query<Q_FFC>(s, b, flags, out_key, cuda_stream, opts);
}

mrv_status mrv_ffc_batch(const mrv_scene* s, const mrv_motion_batch* b, uint32_t flags, uint32_t* out_key,
                         void* cuda_stream) {
  return launch_query<Q_FFC>(s, b, flags, out_key, cuda_stream, nullptr);
}

mrv_status mrv_run_host_batch(const mrv_scene* s, const mrv_motion_batch* hb, uint32_t motval_flags, uint8_t* out_valid,
                              uint32_t ffc_flags, uint32_t* out_key, int64_t chunk_motions, void* cuda_stream) {
  mrv_status st = validate_batch(s, hb);
  if (st != MRV_OK) return st;
  if (hb->robot_timesteps || chunk_motions < 0) return MRV_EINVAL;
  if (hb->n_motions == 0 || (!out_valid && !out_key)) return MRV_OK;
  // the per-motion T array is in host memory here, so it is range-checked up front
  if (hb->n_timesteps) {
    int32_t t_lo = INT32_MAX, t_hi = 0;
    for (int64_t m = 0; m < hb->n_motions; ++m) {
      t_lo = std::min(t_lo, hb->n_timesteps[m]);
      t_hi = std::max(t_hi, hb->n_timesteps[m]);
    }
    if (t_lo < 1) return MRV_EINVAL;
    if (out_key && s->n_pairs > 0 && (uint64_t)t_hi * (uint64_t)s->n_pairs >= 0xFFFFFFFFull) return MRV_ERANGE;
  }
  const int64_t chunk = chunk_motions ? chunk_motions : 1048576;
  // outputs: device memory (the kernels write them), or page-locked host memory (the
  // kernels write a device staging copy that each chunk sends back as soon as its kernel
  // is done, overlapped with the later chunks)
  bool host_v = false, host_k = false;
  for (int q = 0; q < 2; ++q) {
    const void* ptr = q == 0 ? static_cast<const void*>(out_valid) : static_cast<const void*>(out_key);
    if (!ptr) continue;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
      cudaGetLastError();
      return MRV_EINVAL;
    }
    if (at.type == cudaMemoryTypeUnregistered) return MRV_EINVAL;   // pageable host memory
    const bool host = at.type == cudaMemoryTypeHost;
    (q == 0 ? host_v : host_k) = host;
  }
  {   // dry runs of both queries on the first chunk's shape: every synchronous error
      // (flags, launch configuration, FFC range) before anything is enqueued
    mrv_motion_batch probe = *hb;
    probe.n_motions = std::min<int64_t>(std::max<int64_t>(1, chunk / 32), hb->n_motions);
    probe.waypoints = reinterpret_cast<const float*>(16);   // not dereferenced by a dry run
    probe.n_timesteps = hb->n_timesteps ? reinterpret_cast<const int32_t*>(16) : nullptr;
    if (out_valid && (st = launch_query<Q_MOTVAL>(s, &probe, motval_flags, out_valid, cuda_stream, nullptr, true)) != MRV_OK)
      return st;
    if (out_key && (st = launch_query<Q_FFC>(s, &probe, ffc_flags, out_key, cuda_stream, nullptr, true)) != MRV_OK)
      return st;
  }
  const size_t row = (size_t)s->n_robots * hb->n_waypoints * hb->dof_stride * sizeof(float);
  const int64_t cm = std::min<int64_t>(chunk, hb->n_motions);
  const size_t wp_bytes = ((size_t)cm * row + 255) & ~(size_t)255;
  const size_t t_bytes = hb->n_timesteps ? (((size_t)cm * sizeof(int32_t) + 255) & ~(size_t)255) : 0;
  const size_t v_bytes = host_v ? (((size_t)cm + 255) & ~(size_t)255) : 0;   // output staging (host outputs)
  const size_t need = wp_bytes + t_bytes + v_bytes + (host_k ? (size_t)cm * sizeof(uint32_t) : 0);
  DeviceGuard guard(s->device);
  std::lock_guard<std::mutex> lk(s->host_mu);
  if (!s->copy_stream) {
    cudaStream_t cs;
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return MRV_ECUDA;
    s->copy_stream = cs;
    for (int b = 0; b < 2; ++b) {
      cudaEvent_t e0, e1, e2;
      if (cudaEventCreateWithFlags(&e0, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&e1, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&e2, cudaEventDisableTiming) != cudaSuccess)
        return MRV_ECUDA;
      s->ev_copied[b] = e0;
      s->ev_free[b] = e1;
      s->ev_free2[b] = e2;
      cudaEventRecord(e1, cs);   // staging b starts free
      cudaEventRecord(e2, cs);
    }
    for (int b = 0; b < 4; ++b) {
      cudaStream_t ps;
      if (cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking) != cudaSuccess) return MRV_ECUDA;
      s->comp_stream[b] = ps;
    }
    for (int b = 0; b < 5; ++b) {
      cudaEvent_t e;
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return MRV_ECUDA;
      s->ev_join[b] = e;
    }
  }
  if (s->stage_bytes < need) {
    cudaStreamSynchronize(static_cast<cudaStream_t>(s->copy_stream));
    for (int b = 0; b < 2; ++b) {
      if (s->d_stage[b]) cudaEventSynchronize(static_cast<cudaEvent_t>(s->ev_free[b]));
      if (s->d_stage[b]) cudaEventSynchronize(static_cast<cudaEvent_t>(s->ev_free2[b]));
      if (s->d_stage[b]) cudaFree(s->d_stage[b]);
      s->d_stage[b] = nullptr;
    }
    s->stage_bytes = 0;
    for (int b = 0; b < 2; ++b)
      if (cudaMalloc(&s->d_stage[b], need) != cudaSuccess) {
        cudaGetLastError();
        return MRV_ENOMEM;
      }
    s->stage_bytes = need;
  }
  cudaStream_t cs = static_cast<cudaStream_t>(s->copy_stream);
  cudaStream_t caller = static_cast<cudaStream_t>(cuda_stream);
  cudaStream_t ps[4];
  for (int b = 0; b < 4; ++b) ps[b] = static_cast<cudaStream_t>(s->comp_stream[b]);
  cudaEvent_t* ej = reinterpret_cast<cudaEvent_t*>(s->ev_join);
  // fork: everything already enqueued on the caller's stream happens first
  if (cudaEventRecord(ej[4], caller) != cudaSuccess || cudaStreamWaitEvent(cs, ej[4], 0) != cudaSuccess) return MRV_ECUDA;
  for (int b = 0; b < 4; ++b)
    if (cudaStreamWaitEvent(ps[b], ej[4], 0) != cudaSuccess) return MRV_ECUDA;
  const uint8_t* hwp = reinterpret_cast<const uint8_t*>(hb->waypoints);
  // chunk sizes grow geometrically (x4) up to `chunk`: the only copy
  // nothing overlaps (the first) is short, each later copy hides behind the previous
  // chunk's kernels (compute per motion is ~5x its copy), and there are few launches
  // (the first chunk: chunk / 32, or an eighth of a smaller batch, but at least 8192 motions:
  // below that the launches cost more than the exposed copy)
  int64_t next = std::max<int64_t>(1, std::min<int64_t>(chunk / 32, std::max<int64_t>(hb->n_motions / 8, 8192)));
  // chunks alternate between two streams per query (MotVal: 0 / 1, FFC: 2 / 3 with both
  // queries), so a chunk's kernels start on the SMs the previous chunk's tail frees, and
  // the two queries' kernels overlap as in the bench step
  const bool both = out_valid && out_key;
  for (int64_t c0 = 0, i = 0, n = 0; c0 < hb->n_motions; c0 += n, ++i) {
    const int b = (int)(i & 1);
    cudaStream_t strm = ps[b];
    n = std::min<int64_t>(next, hb->n_motions - c0);
    next = std::min<int64_t>(chunk, next * 4);
    uint8_t* stage = static_cast<uint8_t*>(s->d_stage[b]);
    if (cudaStreamWaitEvent(cs, static_cast<cudaEvent_t>(s->ev_free[b]), 0) != cudaSuccess ||
        cudaStreamWaitEvent(cs, static_cast<cudaEvent_t>(s->ev_free2[b]), 0) != cudaSuccess)
      { st = MRV_ECUDA; break; }
    if (cudaMemcpyAsync(stage, hwp + (size_t)c0 * row, (size_t)n * row, cudaMemcpyHostToDevice, cs) != cudaSuccess)
      { st = MRV_ECUDA; break; }
    int32_t* dT = nullptr;
    if (hb->n_timesteps) {
      dT = reinterpret_cast<int32_t*>(stage + wp_bytes);
      if (cudaMemcpyAsync(dT, hb->n_timesteps + c0, (size_t)n * sizeof(int32_t), cudaMemcpyHostToDevice, cs) !=
          cudaSuccess)
        { st = MRV_ECUDA; break; }
    }
    if (cudaEventRecord(static_cast<cudaEvent_t>(s->ev_copied[b]), cs) != cudaSuccess) { st = MRV_ECUDA; break; }
    mrv_motion_batch sub = *hb;
    sub.n_motions = n;
    sub.waypoints = reinterpret_cast<const float*>(stage);
    sub.n_timesteps = dT;
    // the kernels' outputs: the caller's device arrays, or this staging slot's (host outputs)
    uint8_t* ov = host_v ? stage + wp_bytes + t_bytes : out_valid + c0;
    uint32_t* ok = host_k ? reinterpret_cast<uint32_t*>(stage + wp_bytes + t_bytes + v_bytes) : out_key + c0;
    auto motval = [&](cudaStream_t q) -> mrv_status {
      mrv_status r = launch_query<Q_MOTVAL>(s, &sub, motval_flags, ov, q, nullptr);
      if (r == MRV_OK && host_v && cudaMemcpyAsync(out_valid + c0, ov, (size_t)n, cudaMemcpyDeviceToHost, q) != cudaSuccess)
        r = MRV_ECUDA;
      return r;
    };
    auto ffc = [&](cudaStream_t q) -> mrv_status {
      mrv_status r = launch_query<Q_FFC>(s, &sub, ffc_flags, ok, q, nullptr);
      if (r == MRV_OK && host_k &&
          cudaMemcpyAsync(out_key + c0, ok, (size_t)n * sizeof(uint32_t), cudaMemcpyDeviceToHost, q) != cudaSuccess)
        r = MRV_ECUDA;
      return r;
    };
    // (ev_free / ev_free2 follow the result copies too: the slot's output staging is reused)
    if (both) {
      if (cudaStreamWaitEvent(ps[b], static_cast<cudaEvent_t>(s->ev_copied[b]), 0) != cudaSuccess ||
          cudaStreamWaitEvent(ps[2 + b], static_cast<cudaEvent_t>(s->ev_copied[b]), 0) != cudaSuccess)
        { st = MRV_ECUDA; break; }
      if ((st = motval(ps[b])) != MRV_OK) break;
      if (cudaEventRecord(static_cast<cudaEvent_t>(s->ev_free2[b]), ps[b]) != cudaSuccess) { st = MRV_ECUDA; break; }
      if ((st = ffc(ps[2 + b])) != MRV_OK) break;
      if (cudaEventRecord(static_cast<cudaEvent_t>(s->ev_free[b]), ps[2 + b]) != cudaSuccess) { st = MRV_ECUDA; break; }
    } else {
      if (cudaStreamWaitEvent(strm, static_cast<cudaEvent_t>(s->ev_copied[b]), 0) != cudaSuccess) { st = MRV_ECUDA; break; }
      if (out_valid && (st = motval(strm)) != MRV_OK) break;
      if (out_key && (st = ffc(strm)) != MRV_OK) break;
      if (cudaEventRecord(static_cast<cudaEvent_t>(s->ev_free[b]), strm) != cudaSuccess) { st = MRV_ECUDA; break; }
    }
  }
  // join: the caller's stream waits for both compute streams -- also after an error in
  // the loop, so that nothing enqueued so far outlives the caller's buffers unordered
  for (int b = 0; b < 4; ++b)
    if (cudaEventRecord(ej[b], ps[b]) != cudaSuccess || cudaStreamWaitEvent(caller, ej[b], 0) != cudaSuccess)
      return MRV_ECUDA;
  if (cudaEventRecord(ej[4], cs) != cudaSuccess || cudaStreamWaitEvent(caller, ej[4], 0) != cudaSuccess)
    return MRV_ECUDA;   // (the copies too: after an error a copy may have no kernel waiting on it)
  return st;
}

mrv_status mrv_pp_table_bytes(const mrv_scene* s, int32_t horizon, uint64_t* bytes) {
  if (!s || !bytes || horizon < 1) return MRV_EINVAL;
  *bytes = (uint64_t)horizon * (uint64_t)pp_rec_f4(s) * 16u;
  return MRV_OK;
}

mrv_status mrv_pp_build_table(const mrv_scene* s, const mrv_motion_batch* paths, uint64_t partner_mask,
                              int32_t horizon, void* table, void* cuda_stream) {
  mrv_status st = validate_batch(s, paths);
  if (st != MRV_OK) return st;
  if (paths->n_motions != 1 || !paths->waypoints || horizon < 1 || !table ||
      (reinterpret_cast<uintptr_t>(table) & 15u))
    return MRV_EINVAL;
  DeviceGuard guard(s->device);
  const int64_t threads = (int64_t)horizon * s->n_robots;
  const int bs = 128;
  const int64_t grid = (threads + bs - 1) / bs;
  if (grid > 0x7FFFFFFF) return MRV_ERANGE;
  mrv_pp_table_kernel<<<(unsigned)grid, bs, 0, static_cast<cudaStream_t>(cuda_stream)>>>(
      s->ds, static_cast<const uint8_t*>(s->d_blob), paths->waypoints,
      paths->robot_timesteps ? nullptr : paths->n_timesteps, paths->fixed_timesteps, paths->robot_timesteps,
      paths->n_waypoints, paths->dof_stride, (unsigned long long)partner_mask, horizon, pp_rec_f4(s),
      static_cast<float4*>(table), s->d_status);
  if (cudaGetLastError() != cudaSuccess) return MRV_ECUDA;
  return MRV_OK;
}

mrv_status mrv_pp_motval_batch(const mrv_scene* s, const mrv_motion_batch* focus_batch, const int32_t* t_start,
                               int32_t focus_robot, uint64_t partner_mask, const void* table, int32_t horizon,
                               uint32_t flags, uint8_t* out_valid, void* cuda_stream, const mrv_launch_opts* opts) {
  const PPArgs pp{static_cast<const float4*>(table), t_start, horizon, focus_robot, partner_mask};
  return launch_query<Q_MOTVAL>(s, focus_batch, flags, out_valid, cuda_stream, opts, false, &pp);
}

mrv_status mrv_device_status(const mrv_scene* s, void* cuda_stream, int32_t clear, uint32_t* bits) {
  if (!s || !bits) return MRV_EINVAL;
  DeviceGuard guard(s->device);
  cudaStream_t strm = static_cast<cudaStream_t>(cuda_stream);
  uint32_t v = 0;
  if (cudaMemcpyAsync(&v, s->d_status, sizeof v, cudaMemcpyDeviceToHost, strm) != cudaSuccess) {
    cudaGetLastError();
    return MRV_ECUDA;
  }
  if (clear && cudaMemsetAsync(s->d_status, 0, sizeof(uint32_t), strm) != cudaSuccess) {
    cudaGetLastError();
    return MRV_ECUDA;
  }
  if (cudaStreamSynchronize(strm) != cudaSuccess) {
    cudaGetLastError();
    return MRV_ECUDA;
  }
  *bits = v;
  return MRV_OK;
}

mrv_status mrv_fk_states(const mrv_scene* s, const mrv_motion_batch* b, int64_t n_queries, const int64_t* motion,
                         const int32_t* t, float* out_xyz, void* cuda_stream) {
  mrv_status st = validate_batch(s, b);
  if (st != MRV_OK) return st;
  if (n_queries < 0) return MRV_EINVAL;
  if (n_queries == 0) return MRV_OK;
  if (!motion || !t || !out_xyz) return MRV_EINVAL;
  DeviceGuard guard(s->device);
  const int64_t threads = n_queries * s->n_robots;
  const int bs = 128;
  const int64_t grid = (threads + bs - 1) / bs;
  if (grid > 0x7FFFFFFF) return MRV_ERANGE;
  mrv_fk_kernel<<<(unsigned)grid, bs, 0, static_cast<cudaStream_t>(cuda_stream)>>>(
      s->ds, static_cast<const uint8_t*>(s->d_blob), b->waypoints, b->robot_timesteps ? nullptr : b->n_timesteps,
      b->fixed_timesteps, b->robot_timesteps, b->n_motions,
      b->n_waypoints, b->dof_stride, n_queries, motion, t, out_xyz);
  if (cudaGetLastError() != cudaSuccess) return MRV_ECUDA;
  return MRV_OK;
}

}  // extern "C"
