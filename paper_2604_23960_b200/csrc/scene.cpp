// scene.cpp -- host side of libmrv: argument validation, scene precompute and
// upload, status/decode helpers.
//
// Precompute (once per scene; the scene is immutable afterwards):
//   * robots -> links (FK frames: chain joints, or the single body frame)
//   * links -> collision groups of <= 32 spheres, each with a local bounding
//     sphere inflated by kBoundEps (+ a relative term) so that the fp32 broad
//     phase never culls a pair the fp32 narrow phase would report
//   * static per-group obstacle lists for fixed-base revolute chains: an obstacle
//     farther from the base than the group's reach ball can never be touched.
//     This replaces the paper's per-robot cached obstacle transforms
//     (PAPER.md:278-280): everything is tested in the world frame.
//   * the robot-robot work list: (group a, group b, pair rank) in lexicographic
//     pair order (Alg. 1/2 pair loops), minus group
//     pairs of two fixed-base chains whose reach balls can never meet.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "../../include/mrv.h"
#include "mrv_internal.h"
#include "scene_impl.h"

using namespace mrv;

namespace {

bool finite_all(const float* p, int n) {
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

// rotation block of a row-major 3x4 is orthonormal to 1e-4
bool orthonormal(const float* m) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double d = 0.0;
      for (int k = 0; k < 3; ++k) d += (double)m[4 * k + i] * (double)m[4 * k + j];
      if (std::fabs(d - (i == j ? 1.0 : 0.0)) > 1e-4) return false;
    }
  return true;
}

// rotation block orthonormal to 1e-3 with determinant +1
bool proper_rotation(const float* m) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double d = 0.0;
      for (int k = 0; k < 3; ++k) d += (double)m[4 * k + i] * (double)m[4 * k + j];
      if (std::fabs(d - (i == j ? 1.0 : 0.0)) > 1e-3) return false;
    }
  const double det = (double)m[0] * ((double)m[5] * m[10] - (double)m[6] * m[9]) -
                     (double)m[1] * ((double)m[4] * m[10] - (double)m[6] * m[8]) +
                     (double)m[2] * ((double)m[4] * m[9] - (double)m[5] * m[8]);
  return det > 0.0;
}

double tnorm(const float* m) {
  return std::sqrt((double)m[3] * m[3] + (double)m[7] * m[7] + (double)m[11] * m[11]);
}

// place v at byte offset `at` (fixed layout; blob padded with zeros up to it)
template <class T>
uint32_t put_at(std::vector<uint8_t>& blob, const std::vector<T>& v, uint32_t at) {
  if (blob.size() < at) blob.resize(at, 0);
  blob.resize(std::max<size_t>(blob.size(), at + align16((uint32_t)(v.size() * sizeof(T)))), 0);
  if (!v.empty()) std::memcpy(blob.data() + at, v.data(), v.size() * sizeof(T));
  return at;
}

template <class T>
uint32_t put(std::vector<uint8_t>& blob, const std::vector<T>& v) {
  uint32_t off = align16((uint32_t)blob.size());
  blob.resize(off + align16((uint32_t)(v.size() * sizeof(T))), 0);
  if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
  return off;
}

struct F4 { float x, y, z, w; };
struct I4 { int32_t x, y, z, w; };
struct U2 { uint32_t x, y; };

}  // namespace

extern "C" {

const char* mrv_status_string(mrv_status st) {
  switch (st) {
    case MRV_OK: return "MRV_OK";
    case MRV_EINVAL: return "MRV_EINVAL";
    case MRV_ENOMEM: return "MRV_ENOMEM";
    case MRV_ECUDA: return "MRV_ECUDA";
    case MRV_ERANGE: return "MRV_ERANGE";
    case MRV_EUNSUPPORTED: return "MRV_EUNSUPPORTED";
  }
  return "MRV_<unknown>";
}

int32_t mrv_abi_version(void) { return MRV_ABI_VERSION; }

mrv_status mrv_create_scene(const mrv_robot_desc* robots, int32_t n_robots, const mrv_env_desc* env,
                            int32_t cuda_device, mrv_scene** out) {
  if (!robots || !out || n_robots < 1) return MRV_EINVAL;
  if (n_robots > MRV_MAX_ROBOTS) return MRV_EUNSUPPORTED;
  // ---------------------------------------------------------------- validation
  for (int r = 0; r < n_robots; ++r) {
    const mrv_robot_desc& d = robots[r];
    if (d.kind == MRV_CHAIN) {
      if (d.dof < 1) return MRV_EINVAL;
      if (d.dof > MRV_MAX_DOF) return MRV_EUNSUPPORTED;
      if (!d.joint_origin || !d.joint_type) return MRV_EINVAL;
      if (!finite_all(d.joint_origin, 12 * d.dof)) return MRV_EINVAL;
      for (int j = 0; j < d.dof; ++j)
        if (d.joint_type[j] != 0 && d.joint_type[j] != 1) return MRV_EINVAL;
      if (d.base && !finite_all(d.base, 12)) return MRV_EINVAL;
      // rigid transforms only (the kernels store frames as 2 rotation columns + translation)
      if (d.base && !proper_rotation(d.base)) return MRV_EINVAL;
      for (int j = 0; j < d.dof; ++j)
        if (!proper_rotation(d.joint_origin + 12 * j)) return MRV_EINVAL;
    } else if (d.kind == MRV_SE2) {
      if (d.dof != 3) return MRV_EINVAL;
    } else if (d.kind == MRV_SE3) {
      if (d.dof != 7) return MRV_EINVAL;
    } else {
      return MRV_EINVAL;
    }
    if (d.n_spheres < 1 || !d.sphere || !d.sphere_link) return MRV_EINVAL;
    if (d.n_self_pairs < 0 || (d.n_self_pairs > 0 && !d.self_pairs)) return MRV_EINVAL;
    if (d.n_self_pairs > 0 && d.kind != MRV_CHAIN) return MRV_EINVAL;
    for (int k = 0; k < d.n_self_pairs; ++k) {
      const int a = d.self_pairs[2 * k], b = d.self_pairs[2 * k + 1];
      if (a < 0 || b < 0 || a >= d.dof || b >= d.dof || a == b) return MRV_EINVAL;
    }
    if (!finite_all(d.sphere, 4 * d.n_spheres)) return MRV_EINVAL;
    const int n_links = d.kind == MRV_CHAIN ? d.dof : 1;
    for (int k = 0; k < d.n_spheres; ++k) {
      if (!(d.sphere[4 * k + 3] > 0.0f)) return MRV_EINVAL;
      if (d.sphere_link[k] < 0 || d.sphere_link[k] >= n_links) return MRV_EINVAL;
    }
  }
  int n_osph = 0, n_box = 0;
  const float* osph = nullptr;
  const float* box = nullptr;
  if (env) {
    if (env->n_spheres < 0 || env->n_boxes < 0) return MRV_EINVAL;
    n_osph = env->n_spheres;
    n_box = env->n_boxes;
    osph = env->spheres;
    box = env->boxes;
    if ((n_osph > 0 && !osph) || (n_box > 0 && !box)) return MRV_EINVAL;
    if (n_osph > 0 && !finite_all(osph, 4 * n_osph)) return MRV_EINVAL;
    if (n_box > 0 && !finite_all(box, 6 * n_box)) return MRV_EINVAL;
    for (int o = 0; o < n_osph; ++o)
      if (!(osph[4 * o + 3] > 0.0f)) return MRV_EINVAL;
    for (int o = 0; o < n_box; ++o)
      for (int k = 0; k < 3; ++k)
        if (!(box[6 * o + k] < box[6 * o + 3 + k])) return MRV_EINVAL;
    if (n_osph > 65535 || n_box > 65535 || n_osph + n_box > 65535) return MRV_EUNSUPPORTED;   // u16 obstacle ids (grid)
  }

  // ---------------------------------------------------------------- device check
  int prev_dev = 0;
  if (cudaGetDevice(&prev_dev) != cudaSuccess) return MRV_ECUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cuda_device) != cudaSuccess) {
    cudaGetLastError();
    return MRV_ECUDA;
  }
  if (prop.major != 10) return MRV_ECUDA;  // built for sm_100a only: no fallback

  // ---------------------------------------------------------------- links / groups
  std::vector<I4> robA, robB, linkI, groupI;
  std::vector<F4> robBase, linkO, gbound, gcap, sph, osphv, boxv;
  bool use_caps = false;
  std::vector<int32_t> sphere_index;
  std::vector<double> group_reach;    // reach radius of the group's bounding ball around its base (inf if unbounded)
  std::vector<F4> robot_base_pos;     // world position of each robot's base (chains)
  int scene_sphere_base = 0;
  // relative term of the inflation: fp32 rounding grows with coordinate magnitude
  double extent = 1.0;
  for (int o = 0; o < n_osph; ++o)
    for (int k = 0; k < 3; ++k) extent = std::max(extent, (double)std::fabs(osph[4 * o + k]));
  for (int o = 0; o < n_box; ++o)
    for (int k = 0; k < 6; ++k) extent = std::max(extent, (double)std::fabs(box[6 * o + k]));
  const double eps = (double)kBoundEps + 2e-6 * extent;

  for (int r = 0; r < n_robots; ++r) {
    const mrv_robot_desc& d = robots[r];
    const int n_links = d.kind == MRV_CHAIN ? d.dof : 1;
    const int link_begin = (int)linkI.size(), group_begin = (int)groupI.size(), sphere_begin = (int)sph.size();
    float base[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
    if (d.kind == MRV_CHAIN && d.base) std::memcpy(base, d.base, sizeof base);
    for (int i = 0; i < 3; ++i) robBase.push_back({base[4 * i], base[4 * i + 1], base[4 * i + 2], base[4 * i + 3]});
    robot_base_pos.push_back({base[3], base[7], base[11], 0.0f});
    bool bounded = d.kind == MRV_CHAIN && orthonormal(base);
    double rho = 0.0;
    for (int j = 0; j < n_links; ++j) {
      const int link = (int)linkI.size();
      float O[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
      int jt = 0;
      if (d.kind == MRV_CHAIN) {
        std::memcpy(O, d.joint_origin + 12 * j, sizeof O);
        jt = d.joint_type[j];
        if (!orthonormal(O) || jt == 1) bounded = false;
        rho += tnorm(O);
      }
      for (int i = 0; i < 3; ++i) linkO.push_back({O[4 * i], O[4 * i + 1], O[4 * i + 2], O[4 * i + 3]});
      // fast path flag: O is in distal-DH form Tz(d) Tx(a) Rx(alpha) =
      // [[1,0,0,a],[0,c,-s,0],[0,s,c,d]] (exact zeros/ones), so M*O needs 18 instead of 36 FMAs
      const int dh_form = (O[0] == 1.0f && O[1] == 0.0f && O[2] == 0.0f && O[4] == 0.0f && O[7] == 0.0f &&
                           O[8] == 0.0f && O[5] == O[10] && O[6] == -O[9]) ? 1 : 0;
      std::vector<int> ks;
      for (int k = 0; k < d.n_spheres; ++k)
        if (d.sphere_link[k] == j) ks.push_back(k);
      const int g_begin = (int)groupI.size();
      for (size_t c0 = 0; c0 < ks.size(); c0 += kMaxGroupSpheres) {
        const size_t c1 = std::min(ks.size(), c0 + (size_t)kMaxGroupSpheres);
        double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
        for (size_t c = c0; c < c1; ++c) {
          const float* s = d.sphere + 4 * ks[c];
          for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], (double)s[a] - s[3]);
            hi[a] = std::max(hi[a], (double)s[a] + s[3]);
          }
        }
        double cen[3] = {0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2])};
        const float cf[3] = {(float)cen[0], (float)cen[1], (float)cen[2]};
        double R = 0.0;
        for (size_t c = c0; c < c1; ++c) {
          const float* s = d.sphere + 4 * ks[c];
          double dx = s[0] - (double)cf[0], dy = s[1] - (double)cf[1], dz = s[2] - (double)cf[2];
          R = std::max(R, std::sqrt(dx * dx + dy * dy + dz * dz) + s[3]);
        }
        const double Rinf = R + eps;
        float Rf = (float)Rinf;
        if ((double)Rf < Rinf) Rf = std::nextafter(Rf, INFINITY);
        const int g = (int)groupI.size();
        groupI.push_back({link, (int)sph.size(), (int)(c1 - c0), r});
        gbound.push_back({cf[0], cf[1], cf[2], Rf});
        // capsule around the group's spheres: the segment between its two farthest-apart
        // centres, radius = max (distance to the segment + r), inflated like the bound
        // (fp64); kept only if tighter than the bound sphere (the narrow phase's prefilter)
        {
          size_t ia = c0, ib = c0;
          double dmax = -1.0;
          for (size_t c = c0; c < c1; ++c)
            for (size_t e = c; e < c1; ++e) {
              const float *u = d.sphere + 4 * ks[c], *v = d.sphere + 4 * ks[e];
              const double dx = (double)u[0] - v[0], dy = (double)u[1] - v[1], dz = (double)u[2] - v[2];
              const double dd = dx * dx + dy * dy + dz * dz;
              if (dd > dmax) { dmax = dd; ia = c; ib = e; }
            }
          const float *p0 = d.sphere + 4 * ks[ia], *p1 = d.sphere + 4 * ks[ib];
          const double ux = (double)p1[0] - p0[0], uy = (double)p1[1] - p0[1], uz = (double)p1[2] - p0[2];
          const double uu = ux * ux + uy * uy + uz * uz;
          double rc = 0.0;
          for (size_t c = c0; c < c1; ++c) {
            const float* q = d.sphere + 4 * ks[c];
            const double wx = (double)q[0] - p0[0], wy = (double)q[1] - p0[1], wz = (double)q[2] - p0[2];
            const double t = uu > 0.0 ? std::min(1.0, std::max(0.0, (wx * ux + wy * uy + wz * uz) / uu)) : 0.0;
            const double ex = wx - t * ux, ey = wy - t * uy, ez = wz - t * uz;
            rc = std::max(rc, std::sqrt(ex * ex + ey * ey + ez * ez) + q[3]);
          }
          const double rci = rc + eps;
          float rcf = (float)rci;
          if ((double)rcf < rci) rcf = std::nextafter(rcf, INFINITY);
          if (rcf < 0.9f * Rf) {
            gcap.push_back({p0[0], p0[1], p0[2], rcf});
            gcap.push_back({p1[0], p1[1], p1[2], 1.0f});
            use_caps = true;
          } else {
            gcap.push_back({cf[0], cf[1], cf[2], Rf});
            gcap.push_back({cf[0], cf[1], cf[2], 0.0f});
          }
        }
        const double cn = std::sqrt((double)cf[0] * cf[0] + (double)cf[1] * cf[1] + (double)cf[2] * cf[2]);
        group_reach.push_back(bounded ? rho + cn + Rinf : INFINITY);
        for (size_t c = c0; c < c1; ++c) {
          const float* s = d.sphere + 4 * ks[c];
          sph.push_back({s[0], s[1], s[2], s[3]});
          sphere_index.push_back(scene_sphere_base + ks[c]);
        }
        (void)g;
      }
      linkI.push_back({r, jt | (dh_form << 1), g_begin, (int)groupI.size() - g_begin});
    }
    robA.push_back({d.kind, d.dof, link_begin, n_links});
    robB.push_back({group_begin, (int)groupI.size() - group_begin, sphere_begin, (int)sph.size() - sphere_begin});
    scene_sphere_base += d.n_spheres;
  }
  const int n_links_total = (int)linkI.size(), n_groups = (int)groupI.size();
  if (n_groups > 65535) return MRV_EUNSUPPORTED;
  if (n_osph + n_box > 0 && n_groups > 2047) return MRV_EUNSUPPORTED;   // env queue entries carry an 11-bit group
  // fast-DH robots (every joint a revolute DH-form joint carrying exactly one collision
  // group, consecutive): the chain walk of the kernels (robot_fk_dh, fk_env_fused)
  std::vector<int> fast_dh(n_robots, 0);
  for (int r = 0; r < n_robots; ++r) {
    bool fast = robA[r].x == MRV_CHAIN;
    for (int l = robA[r].z; fast && l < robA[r].z + robA[r].w; ++l)
      fast = (linkI[l].y & 1) == 0 && (linkI[l].y & 2) != 0 && linkI[l].w == 1 &&
             linkI[l].z == linkI[robA[r].z].z + (l - robA[r].z);   // one group per link, consecutive
    fast_dh[r] = fast ? 1 : 0;
  }
  // their group bounds are centred on the link's x axis (DH links run along x): the walk
  // places them with 3 FMAs (column 0 and the translation) instead of 9; the same enclosure
  // rule (max distance + radius, inflated, fp64) -- a sphere off the axis only grows R
  for (int r = 0; r < n_robots; ++r) {
    if (!fast_dh[r]) continue;
    for (int g = robB[r].x; g < robB[r].x + robB[r].y; ++g) {
      double lo = 1e300, hi = -1e300;
      for (int k = groupI[g].y; k < groupI[g].y + groupI[g].z; ++k) {
        lo = std::min(lo, (double)sph[k].x - sph[k].w);
        hi = std::max(hi, (double)sph[k].x + sph[k].w);
      }
      const float cx = (float)(0.5 * (lo + hi));
      double R = 0.0;
      for (int k = groupI[g].y; k < groupI[g].y + groupI[g].z; ++k) {
        const double dx = sph[k].x - (double)cx, dy = sph[k].y, dz = sph[k].z;
        R = std::max(R, std::sqrt(dx * dx + dy * dy + dz * dz) + sph[k].w);
      }
      const double Rinf = R + eps;
      float Rf = (float)Rinf;
      if ((double)Rf < Rinf) Rf = std::nextafter(Rf, INFINITY);
      gbound[g] = {cx, 0.0f, 0.0f, Rf};
    }
  }

  // ---------------------------------------------------------------- obstacles + uniform grid
  // Obstacles in one table, 2 x float4 each: {lo, r}, {hi, 0}.  A sphere obstacle is
  // the degenerate box lo = hi = centre with rounding radius r, a box has r = 0; the
  // clamped distance e_k = max(lo_k - c_k, 0, c_k - hi_k) then gives |c - o| for a
  // sphere bit for bit (reading c.2), so one predicate serves both kinds:
  // sum e_k^2 < (R + r)^2.  Index o < n_osph: sphere obstacle o; else box o - n_osph.
  std::vector<F4> obsv;
  for (int o = 0; o < n_osph; ++o) {
    obsv.push_back({osph[4 * o], osph[4 * o + 1], osph[4 * o + 2], osph[4 * o + 3]});
    obsv.push_back({osph[4 * o], osph[4 * o + 1], osph[4 * o + 2], 0.0f});
  }
  for (int o = 0; o < n_box; ++o) {
    obsv.push_back({box[6 * o], box[6 * o + 1], box[6 * o + 2], 0.0f});
    obsv.push_back({box[6 * o + 3], box[6 * o + 4], box[6 * o + 5], 0.0f});
  }
  const int n_obs = n_osph + n_box;
  // Broad phase of CC(S_i, E) (MotVal): a group's world bound (c, R) can only touch
  // obstacles within R <= Rmax of c, so a uniform grid over the obstacles' AABBs grown by
  // Rmax lists, per cell, every obstacle within Rmax + eps of any point of the cell
  // (fp64, conservative); the kernel tests the bound against its centre's cell list only.
  // A centre outside the grid is farther than Rmax from every obstacle.  The cell size is
  // the one with the fewest list entries per cell within a smem budget.
  std::vector<uint16_t> cell_start, cell_list;
  float grid_hdr[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // origin xyz, 1/h, nx, ny, nz (as int bits), 0
  if (n_obs > 0 && n_groups > 0) {
    double Rmax = 0.0;
    for (const F4& gb : gbound) Rmax = std::max(Rmax, (double)gb.w);
    const double grow = Rmax + eps;
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int o = 0; o < n_obs; ++o) {
      const F4 a = obsv[2 * o], b = obsv[2 * o + 1];
      const double ol[3] = {a.x, a.y, a.z}, oh[3] = {b.x, b.y, b.z};
      for (int k = 0; k < 3; ++k) {
        lo[k] = std::min(lo[k], ol[k] - (double)a.w - grow);
        hi[k] = std::max(hi[k], oh[k] + (double)a.w + grow);
      }
    }
    // distance from the cell box [clo, chi] to obstacle o (box minus rounding radius)
    auto cell_obs_dist = [&](const double* clo, const double* chi, int o) {
      double s2 = 0.0;
      const double ol[3] = {obsv[2 * o].x, obsv[2 * o].y, obsv[2 * o].z};
      const double oh[3] = {obsv[2 * o + 1].x, obsv[2 * o + 1].y, obsv[2 * o + 1].z};
      for (int k = 0; k < 3; ++k) {
        const double e = std::max({ol[k] - chi[k], 0.0, clo[k] - oh[k]});
        s2 += e * e;
      }
      return std::sqrt(s2) - (double)obsv[2 * o].w;
    };
    const double span = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]});
    // bytes of cell offsets + lists: small enough to share smem with the per-warp scratch,
    // unless the obstacle table alone is large (then MotVal reads the tail tables from
    // global memory anyway, and a finer grid pays)
    const size_t kBudget = n_obs > 512 ? ((size_t)1 << 20) : 12288;
    double best_cost = 1e300;
    for (int steps = 1; steps <= 64; ++steps) {
      const double h = span / steps;
      int n[3];
      for (int k = 0; k < 3; ++k) n[k] = std::max(1, (int)std::ceil((hi[k] - lo[k]) / h));
      const long cells = (long)n[0] * n[1] * n[2];
      if (cells > 16384) break;
      std::vector<uint16_t> st(cells + 1, 0), li;
      bool ok = true;
      for (long c = 0; c < cells && ok; ++c) {
        const int ix = (int)(c % n[0]), iy = (int)((c / n[0]) % n[1]), iz = (int)(c / ((long)n[0] * n[1]));
        const double clo[3] = {lo[0] + ix * h, lo[1] + iy * h, lo[2] + iz * h};
        const double chi[3] = {clo[0] + h, clo[1] + h, clo[2] + h};
        for (int o = 0; o < n_obs; ++o)
          if (cell_obs_dist(clo, chi, o) < grow) li.push_back((uint16_t)o);
        if (li.size() > 65535) ok = false;
        st[c + 1] = (uint16_t)li.size();
      }
      if (!ok) break;
      const size_t bytes = (st.size() + li.size()) * sizeof(uint16_t);
      if (bytes > kBudget && !cell_start.empty()) break;
      const double cost = (double)li.size() / (double)cells;   // mean candidates per lookup
      if (cost < best_cost || cell_start.empty()) {
        best_cost = cost;
        cell_start = st;
        cell_list = li;
        grid_hdr[0] = (float)lo[0];
        grid_hdr[1] = (float)lo[1];
        grid_hdr[2] = (float)lo[2];
        grid_hdr[3] = (float)(1.0 / h);
        std::memcpy(&grid_hdr[4], n, sizeof n);
      }
    }
    // the kernel computes the cell in fp32: a centre that rounds across a cell boundary
    // is still within eps (>= 1e-4 m) of the cell it lands in, which the lists cover
  }
  std::vector<F4> grid_rec(2);
  std::memcpy(grid_rec.data(), grid_hdr, sizeof grid_hdr);
  const std::vector<uint32_t> no_ranks;
  // (self-collision segments below use the generic segment record)
  struct Seg { uint32_t hdr, rank_min, pad0, pad1; uint16_t idx[kSegLen]; float rs2[kSegLen]; };
  static_assert(sizeof(Seg) == 64, "segment record is 4 x uint4");
  // rs2[k] = (R_a + R_k)^2 of the two (inflated) group bounds, rounded up
  auto add_segs = [&](std::vector<Seg>& out, int a, const std::vector<int>& cand) {
    for (size_t c0 = 0; c0 < cand.size(); c0 += kSegLen) {
      Seg sg;
      std::memset(&sg, 0, sizeof sg);
      const size_t c1 = std::min(cand.size(), c0 + (size_t)kSegLen);
      sg.hdr = (uint32_t)a | ((uint32_t)(c1 - c0) << 16);
      sg.rank_min = 0xFFFFFFFFu;
      for (size_t c = c0; c < c1; ++c) {
        sg.idx[c - c0] = (uint16_t)cand[c];
        const double Ra = gbound[a].w, Rb = gbound[cand[c]].w;
        const double r2 = (Ra + Rb) * (Ra + Rb);
        float f = (float)r2;
        if ((double)f < r2) f = std::nextafter(f, INFINITY);
        sg.rs2[c - c0] = f;
      }
      out.push_back(sg);
    }
  };

  // ---------------------------------------------------------------- self-collision work list
  // per group a of link la: the groups of the links paired with la
  std::vector<Seg> self_segs;
  int n_self = 0;
  for (int r = 0; r < n_robots; ++r) {
    const mrv_robot_desc& d = robots[r];
    if (d.n_self_pairs == 0) continue;
    std::vector<std::vector<int>> partner(d.dof);
    for (int k = 0; k < d.n_self_pairs; ++k) {
      int a = d.self_pairs[2 * k], b = d.self_pairs[2 * k + 1];
      if (a > b) std::swap(a, b);
      if (std::find(partner[a].begin(), partner[a].end(), b) == partner[a].end()) partner[a].push_back(b);
    }
    for (int la = 0; la < d.dof; ++la) {
      std::sort(partner[la].begin(), partner[la].end());
      const I4 LA = linkI[robA[r].z + la];
      for (int ga = LA.z; ga < LA.z + LA.w; ++ga) {
        std::vector<int> cand;
        for (int lb : partner[la]) {
          const I4 LB = linkI[robA[r].z + lb];
          for (int gb = LB.z; gb < LB.z + LB.w; ++gb) cand.push_back(gb);
        }
        n_self += (int)cand.size();
        add_segs(self_segs, ga, cand);
      }
    }
  }

  // ---------------------------------------------------------------- robot-robot work list
  // Two-level: each robot's groups are partitioned into supergroups of <= 3
  // consecutive groups (7-link arms: links {0,1,2}, {3,4}, {5,6}); a supergroup's
  // per-state bound is derived from its members' bounds in the kernel.  The first
  // level tests supergroup a of robot i against supergroups b of robots j > i (in
  // lexicographic pair order, Alg. 1/2 pair loops);
  // survivors expand to their <= 9 group pairs.  Supergroup pairs of two fixed-base
  // chains whose member reach balls can never meet are dropped.
  std::vector<I4> superI, robC;
  for (int r = 0; r < n_robots; ++r) {
    const int g0 = robB[r].x, ng = robB[r].y;
    const int nsg = ng == 0 ? 0 : (ng + kSuperMax - 1) / kSuperMax;
    robC.push_back({(int)superI.size(), nsg, 0, 0});
    int g = g0;
    for (int k = 0; k < nsg; ++k) {
      const int cnt = ng / nsg + (k < ng % nsg ? 1 : 0);
      superI.push_back({r, g, cnt, 0});
      g += cnt;
    }
  }
  for (int r = 0; r < n_robots; ++r) robC[r].z = fast_dh[r];   // (see the dhrec table below)
  struct RRPair { int a, b; uint32_t rank; };
  std::vector<RRPair> rr_list;
  int n_rr = 0;
  for (int i = 0; i < n_robots; ++i)
    for (int sa = robC[i].x; sa < robC[i].x + robC[i].y; ++sa)
      for (int j = i + 1; j < n_robots; ++j) {
        const uint32_t rank = (uint32_t)(i * n_robots - i * (i + 1) / 2 + (j - i - 1));
        const double bx = (double)robot_base_pos[i].x - robot_base_pos[j].x;
        const double by = (double)robot_base_pos[i].y - robot_base_pos[j].y;
        const double bz = (double)robot_base_pos[i].z - robot_base_pos[j].z;
        const double bd = std::sqrt(bx * bx + by * by + bz * bz);
        for (int sb = robC[j].x; sb < robC[j].x + robC[j].y; ++sb) {
          bool any = false;
          for (int ga = superI[sa].y; ga < superI[sa].y + superI[sa].z; ++ga)
            for (int gb = superI[sb].y; gb < superI[sb].y + superI[sb].z; ++gb)
              if (!(std::isfinite(group_reach[ga]) && std::isfinite(group_reach[gb]) &&
                    bd >= group_reach[ga] + group_reach[gb] + eps)) {
                any = true;
                ++n_rr;
              }
          if (any) rr_list.push_back({sa, sb, rank});
        }
      }
  // The test is symmetric, so each pair is owned by whichever supergroup has fewer
  // pairs so far (balanced out-degrees -> short, evenly filled segments); the kernel
  // recovers the robot order (i < j) for the rank.  Segments hold <= kRRSegLen pairs
  // (the kernel's unrolled tests per lane).
  std::vector<int> owner(rr_list.size()), deg(superI.size(), 0);
  for (size_t e = 0; e < rr_list.size(); ++e) {
    owner[e] = deg[rr_list[e].a] <= deg[rr_list[e].b] ? rr_list[e].a : rr_list[e].b;
    ++deg[owner[e]];
  }
  for (bool changed = true; changed;) {   // flip u->v while deg(u) > deg(v) + 1 (sum of deg^2 drops)
    changed = false;
    for (size_t e = 0; e < rr_list.size(); ++e) {
      const int u = owner[e], v = u == rr_list[e].a ? rr_list[e].b : rr_list[e].a;
      if (deg[u] > deg[v] + 1) {
        owner[e] = v;
        --deg[u];
        ++deg[v];
        changed = true;
      }
    }
  }
  std::vector<std::vector<std::pair<int, uint32_t>>> owned(superI.size());
  for (size_t e = 0; e < rr_list.size(); ++e) {
    const RRPair& q = rr_list[e];
    owned[owner[e]].push_back({owner[e] == q.a ? q.b : q.a, q.rank});
  }
  const int rr_len = kRRSegLen;
  // rr segment record (2 x uint4): {a | n << 16, rank_min, c0, c1}, {c2, c3, c4, 0}
  // (rank_min: the smallest pair rank of the segment; kept in the record, no longer read)
  struct RRSeg { uint32_t hdr, rank_min, c[6]; };
  static_assert(sizeof(RRSeg) == 32 && kRRSegLen <= 6, "rr segment record is 2 x uint4");
  std::vector<RRSeg> rr_segs;
  for (size_t x = 0; x < owned.size(); ++x)
    for (size_t c0 = 0; c0 < owned[x].size(); c0 += kRRSegLen) {
      const size_t c1 = std::min(owned[x].size(), c0 + (size_t)kRRSegLen);
      RRSeg sg;
      std::memset(&sg, 0, sizeof sg);
      sg.hdr = (uint32_t)x | ((uint32_t)(c1 - c0) << 16);
      sg.rank_min = 0xFFFFFFFFu;
      for (size_t c = c0; c < c1; ++c) {
        sg.c[c - c0] = (uint32_t)owned[x][c].first;
        sg.rank_min = std::min(sg.rank_min, owned[x][c].second);
      }
      rr_segs.push_back(sg);
    }

  // MRV_DIAG_NO_BROADPHASE: the same record over every supergroup pair of every robot pair
  // (no static reach pruning, owner = the lower robot's supergroup), so the diagnostic's
  // on/off bit-identity covers the pruning too
  std::vector<RRSeg> rr_segs_all;
  for (int i = 0; i < n_robots; ++i)
    for (int sa = robC[i].x; sa < robC[i].x + robC[i].y; ++sa) {
      std::vector<std::pair<int, uint32_t>> cand;
      for (int j = i + 1; j < n_robots; ++j)
        for (int sb = robC[j].x; sb < robC[j].x + robC[j].y; ++sb)
          cand.push_back({sb, (uint32_t)(i * n_robots - i * (i + 1) / 2 + (j - i - 1))});
      for (size_t c0 = 0; c0 < cand.size(); c0 += kRRSegLen) {
        const size_t c1 = std::min(cand.size(), c0 + (size_t)kRRSegLen);
        RRSeg sg;
        std::memset(&sg, 0, sizeof sg);
        sg.hdr = (uint32_t)sa | ((uint32_t)(c1 - c0) << 16);
        sg.rank_min = 0xFFFFFFFFu;
        for (size_t c = c0; c < c1; ++c) {
          sg.c[c - c0] = (uint32_t)cand[c].first;
          sg.rank_min = std::min(sg.rank_min, cand[c].second);
        }
        rr_segs_all.push_back(sg);
      }
    }

  // ---------------------------------------------------------------- per-W frame offsets (bank staggered)
  typedef FixedLayout FL;
  const bool fixed = n_robots <= FL::kRobots && n_links_total <= FL::kLinks && n_groups <= FL::kGroups &&
                     (int)sph.size() <= FL::kSpheres && (int)rr_segs.size() <= FL::kRRSegs &&
                     (int)superI.size() <= FL::kSuper;
  const int lo_stride = fixed ? FL::kLinks : n_links_total;   // link_off row stride
  std::vector<int32_t> link_off(4 * (size_t)lo_stride);
  int32_t frame_words[4];
  for (int wi = 0; wi < 4; ++wi) {
    const int W = 4 << wi, G = 32 / W;
    int cur = 0;
    for (int r = 0; r < n_robots; ++r) {
      const int want = ((r % G) * W) % 32;
      while (cur % 32 != want) ++cur;
      for (int l = 0; l < robA[r].w; ++l) link_off[(size_t)wi * lo_stride + robA[r].z + l] = cur + l * kFrameWords * W;
      cur += robA[r].w * kFrameWords * W;
    }
    frame_words[wi] = (cur + 3) & ~3;
  }

  // ---------------------------------------------------------------- blob
  mrv_scene* s = new (std::nothrow) mrv_scene();
  if (!s) return MRV_ENOMEM;
  std::vector<uint8_t>& blob = s->h_blob;
  DevScene& ds = s->ds;
  std::memset(&ds, 0, sizeof ds);
  std::vector<I4> robot_rec;
  for (int r = 0; r < n_robots; ++r) {
    robot_rec.push_back(robA[r]);
    robot_rec.push_back(robB[r]);
    robot_rec.push_back(robC[r]);
  }
  ds.off_robot = fixed ? put_at(blob, robot_rec, FL::robot) : put(blob, robot_rec);
  ds.off_robot_base = fixed ? put_at(blob, robBase, FL::robot_base) : put(blob, robBase);
  ds.off_link = fixed ? put_at(blob, linkI, FL::link) : put(blob, linkI);
  ds.off_link_origin = fixed ? put_at(blob, linkO, FL::link_origin) : put(blob, linkO);
  ds.off_group = fixed ? put_at(blob, groupI, FL::group) : put(blob, groupI);
  ds.off_gbound = fixed ? put_at(blob, gbound, FL::gbound) : put(blob, gbound);
  ds.off_sphere = fixed ? put_at(blob, sph, FL::sphere) : put(blob, sph);
  ds.off_rr_segs = fixed ? put_at(blob, rr_segs, FL::rr_segs) : put(blob, rr_segs);
  ds.off_super = fixed ? put_at(blob, superI, FL::super) : put(blob, superI);
  // fast-DH records (per link, 3 x 16 B): {a, cos alpha, sin alpha, d}, the link's single
  // group bound, {group, group_super code, 0, 0}; robot C.z = 1 when every joint is a
  // revolute DH-form joint carrying exactly one collision group
  std::vector<F4> dhrec(3 * (size_t)n_links_total, F4{0, 0, 0, 0});
  for (int r = 0; r < n_robots; ++r) {
    if (!robC[r].z) continue;
    for (int l = robA[r].z; l < robA[r].z + robA[r].w; ++l) {
      const F4 o0 = linkO[3 * l], o1 = linkO[3 * l + 1], o2 = linkO[3 * l + 2];
      dhrec[3 * l] = {o0.w, o1.y, o2.y, o2.w};
      const int g = linkI[l].z;
      dhrec[3 * l + 1] = gbound[g];
      int32_t ids[4] = {g, 0, 0, 0};
      std::memcpy(&dhrec[3 * l + 2], ids, sizeof ids);
    }
  }
  std::vector<int32_t> group_super(n_groups, 0);
  for (size_t sg = 0; sg < superI.size(); ++sg)
    for (int g = superI[sg].y; g < superI[sg].y + superI[sg].z; ++g)
      group_super[g] = (int32_t)sg | (g == superI[sg].y + superI[sg].z - 1 ? (int32_t)0x80000000 : 0) |
                       (g == superI[sg].y ? 0x40000000 : 0);
  for (int l = 0; l < n_links_total; ++l) {
    int32_t ids[4];
    std::memcpy(ids, &dhrec[3 * l + 2], sizeof ids);
    if (robC[linkI[l].x].z) {
      ids[1] = group_super[ids[0]];
      std::memcpy(&dhrec[3 * l + 2], ids, sizeof ids);
    }
  }
  ds.off_group_super = fixed ? put_at(blob, group_super, FL::group_super) : put(blob, group_super);
  // the first joint's fixed part folded into the base (fp64, rounded once): fast-DH robots
  // walk their chain from base * Tz(d_0) Tx(a_0) Rx(alpha_0) and apply Rz(q_0) alone
  std::vector<F4> dhbase(3 * (size_t)n_robots, F4{0, 0, 0, 0});
  for (int r = 0; r < n_robots; ++r) {
    for (int i = 0; i < 3; ++i) dhbase[3 * r + i] = robBase[3 * r + i];
    if (!robC[r].z) continue;
    const F4 P = dhrec[3 * robA[r].z];   // {a, cos alpha, sin alpha, d} of link 0
    for (int i = 0; i < 3; ++i) {
      const F4 b = robBase[3 * r + i];
      const double m0 = b.x, m1 = b.y, m2 = b.z, m3 = b.w;
      dhbase[3 * r + i] = {(float)m0, (float)(m1 * P.y + m2 * P.z), (float)(m2 * P.y - m1 * P.z),
                           (float)(m0 * P.x + m2 * P.w + m3)};
    }
    // link 0's record becomes the identity DH step {a 0, cos 1, sin 0, d 0}: a walk that
    // applies it (fk_env_fused) computes exactly what the one that skips it does
    dhrec[3 * robA[r].z] = F4{0.0f, 1.0f, 0.0f, 0.0f};
  }
  ds.off_dhrec = fixed ? put_at(blob, dhrec, FL::dhrec) : put(blob, dhrec);
  ds.off_dhbase = fixed ? put_at(blob, dhbase, FL::dhbase) : put(blob, dhbase);
  ds.off_link_off = fixed ? put_at(blob, link_off, FL::link_off) : put(blob, link_off);
  ds.off_gcap = fixed ? put_at(blob, gcap, FL::gcap) : put(blob, gcap);
  // everything above is what FFC reads: it stages only this prefix into shared memory
  blob.resize(align16((uint32_t)blob.size()), 0);
  ds.rr_prefix_bytes = (int32_t)blob.size();
  ds.off_obs = put(blob, obsv);
  ds.off_grid = put(blob, grid_rec);
  ds.off_cell_start = put(blob, cell_start);
  ds.off_cell_list = put(blob, cell_list);
  ds.off_self_segs = put(blob, self_segs);
  ds.off_sphere_index = put(blob, sphere_index);   // SpheresFK export only (read from global memory)
  ds.off_rr_segs_all = put(blob, rr_segs_all);      // MRV_DIAG_NO_BROADPHASE only
  ds.n_rr_segs_all = (int32_t)rr_segs_all.size();
  blob.resize(align16((uint32_t)blob.size()), 0);
  ds.blob_bytes = (uint32_t)blob.size();
  ds.fixed_layout = fixed ? 1 : 0;
  ds.use_caps = use_caps ? 1 : 0;
  ds.n_robots = n_robots;
  ds.n_links = n_links_total;
  ds.n_groups = n_groups;
  ds.n_spheres = (int)sph.size();
  ds.n_osph = n_osph;
  ds.n_box = n_box;
  ds.n_cells = (int)(cell_start.empty() ? 0 : cell_start.size() - 1);
  ds.n_cell_entries = (int)cell_list.size();
  ds.n_rr_items = n_rr;
  ds.n_rr_segs = (int)rr_segs.size();
  ds.rr_seg_len = rr_len;
  ds.n_self_segs = (int)self_segs.size();
  ds.n_self_items = n_self;
  ds.group_lg = -1;
  if (!groupI.empty()) {
    const int gs = groupI[0].z;
    bool same = (gs & (gs - 1)) == 0;
    for (const I4& g : groupI) same = same && g.z == gs;
    if (same) ds.group_lg = __builtin_ctz((unsigned)gs);
  }
  ds.n_super = (int)superI.size();
  ds.n_pairs = n_robots * (n_robots - 1) / 2;
  // Tiled level 1 (the lean W = 8 FFC instance, kernels.cu rr_stage_tile): four robots of
  // three supergroups each, lane (robot r, state s) tests its supergroups against robot
  // r + 1's (9 pairs) and against robot r + 2's in the pattern kTileDiag (6 pairs; lanes of
  // robots 2 and 3 see the same diagonal robot pairs transposed, so the (k, k) pairs are
  // theirs twice and masked there).  Bit b of robot r's 15-bit mask: the pair is in the
  // statically pruned work list (rr_list).
  ds.l1tile = 0;
  ds.l1tile_masks = 0;
  if (n_robots == 4 && fixed) {
    bool ok = true;
    for (int r = 0; r < 4; ++r) ok = ok && robC[r].y == 3 && robC[r].x == 3 * r;
    if (ok) {
      auto listed = [&](int sa, int sb) {
        if (sa > sb) std::swap(sa, sb);
        for (const RRPair& q : rr_list)
          if (q.a == sa && q.b == sb) return true;
        return false;
      };
      static const int kDa[6] = {0, 1, 2, 0, 0, 1}, kDb[6] = {0, 1, 2, 1, 2, 2};
      for (int r = 0; r < 4; ++r) {
        const int x = (r + 1) & 3, y = (r + 2) & 3;
        uint64_t m = 0;
        for (int b = 0; b < 9; ++b)
          if (listed(3 * r + b / 3, 3 * x + b % 3)) m |= 1ull << b;
        for (int i = 0; i < 6; ++i)
          if (!(r >= 2 && kDa[i] == kDb[i]) && listed(3 * r + kDa[i], 3 * y + kDb[i])) m |= 1ull << (9 + i);
        ds.l1tile_masks |= m << (16 * r);
      }
      ds.l1tile = 1;
      // bit 1: every robot a fast-DH chain, group g = link g's only group, bounds on the
      // link's x axis -- level 2 places a group bound with 3 FMAs from the stored frame
      bool xaxis = true;
      for (int r = 0; r < 4; ++r) xaxis = xaxis && fast_dh[r];
      for (int g = 0; xaxis && g < n_groups; ++g) xaxis = groupI[g].x == g && gbound[g].y == 0.0f && gbound[g].z == 0.0f;
      if (xaxis) ds.l1tile |= 2;
      // bit 2: also every sphere centre and capsule endpoint on its link's x axis (DH links
      // modelled along x): the narrow phase and the capsule prefilter place them with 3 FMAs
      bool onx = xaxis;
      for (size_t k = 0; onx && k < sph.size(); ++k) onx = sph[k].y == 0.0f && sph[k].z == 0.0f;
      for (size_t k = 0; onx && k < gcap.size(); ++k) onx = gcap[k].y == 0.0f && gcap[k].z == 0.0f;
      if (onx) ds.l1tile |= 4;
    }
  }
  int max_links = 0;
  for (int r = 0; r < n_robots; ++r) max_links = std::max(max_links, robA[r].w);
  ds.max_link_per_robot = max_links;
  for (int wi = 0; wi < 4; ++wi) ds.frame_words[wi] = frame_words[wi];

  s->device = cuda_device;
  s->sm_count = prop.multiProcessorCount;
  s->max_smem_optin = (int)prop.sharedMemPerBlockOptin;
  s->n_robots = n_robots;
  s->n_pairs = ds.n_pairs;
  s->fuse_env_ok = n_robots > 0;
  for (int r = 0; r < n_robots; ++r) s->fuse_env_ok = s->fuse_env_ok && robC[r].z && robA[r].y == robA[0].y;
  s->total_spheres = ds.n_spheres;
  s->kinds.resize(n_robots);
  for (int r = 0; r < n_robots; ++r) s->kinds[r] = robots[r].kind;

  if (cudaSetDevice(cuda_device) != cudaSuccess) {
    delete s;
    return MRV_ECUDA;
  }
  mrv_status st = MRV_OK;
  if (cudaMalloc(&s->d_blob, ds.blob_bytes) != cudaSuccess ||
      cudaMalloc(&s->d_ring, sizeof(unsigned long long) * MRV_MAX_INFLIGHT) != cudaSuccess ||
      cudaMalloc(&s->d_status, sizeof(uint32_t)) != cudaSuccess) {
    st = MRV_ENOMEM;
  } else if (cudaMemcpy(s->d_blob, blob.data(), ds.blob_bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
             cudaMemset(s->d_ring, 0, sizeof(unsigned long long) * MRV_MAX_INFLIGHT) != cudaSuccess ||
             cudaMemset(s->d_status, 0, sizeof(uint32_t)) != cudaSuccess) {
    st = MRV_ECUDA;
  }
  cudaSetDevice(prev_dev);
  if (st != MRV_OK) {
    cudaGetLastError();
    mrv_destroy_scene(s);
    return st;
  }
  *out = s;
  return MRV_OK;
}

mrv_status mrv_destroy_scene(mrv_scene* s) {
  if (!s) return MRV_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(s->device);
  if (s->d_blob) cudaFree(s->d_blob);
  if (s->d_ring) cudaFree(s->d_ring);
  if (s->d_status) cudaFree(s->d_status);
  for (auto& e : s->pp_seg_cache) cudaFree(e.d);
  if (s->copy_stream) cudaStreamSynchronize(static_cast<cudaStream_t>(s->copy_stream));
  for (int b = 0; b < 2; ++b) {
    if (s->d_stage[b]) cudaFree(s->d_stage[b]);
    if (s->ev_copied[b]) cudaEventDestroy(static_cast<cudaEvent_t>(s->ev_copied[b]));
    if (s->ev_free[b]) cudaEventDestroy(static_cast<cudaEvent_t>(s->ev_free[b]));
    if (s->ev_free2[b]) cudaEventDestroy(static_cast<cudaEvent_t>(s->ev_free2[b]));
  }
  if (s->copy_stream) cudaStreamDestroy(static_cast<cudaStream_t>(s->copy_stream));
  for (int b = 0; b < 4; ++b)
    if (s->comp_stream[b]) {
      cudaStreamSynchronize(static_cast<cudaStream_t>(s->comp_stream[b]));
      cudaStreamDestroy(static_cast<cudaStream_t>(s->comp_stream[b]));
    }
  for (int b = 0; b < 5; ++b)
    if (s->ev_join[b]) cudaEventDestroy(static_cast<cudaEvent_t>(s->ev_join[b]));
  cudaSetDevice(prev);
  delete s;
  return MRV_OK;
}

mrv_status mrv_scene_info(const mrv_scene* s, int32_t* n_robots, int32_t* n_pairs, int32_t* total_spheres,
                          int32_t* total_frames) {
  if (!s) return MRV_EINVAL;
  if (n_robots) *n_robots = s->n_robots;
  if (n_pairs) *n_pairs = s->n_pairs;
  if (total_spheres) *total_spheres = s->total_spheres;
  if (total_frames) *total_frames = s->ds.n_links;
  return MRV_OK;
}

mrv_status mrv_decode_conflict(const mrv_scene* s, uint32_t key, int32_t* t, int32_t* i, int32_t* j) {
  if (!s || !t || !i || !j) return MRV_EINVAL;
  if (key == MRV_NO_CONFLICT) {
    *t = *i = *j = -1;
    return MRV_OK;
  }
  const uint32_t P = (uint32_t)s->n_pairs;
  if (P == 0) return MRV_EINVAL;
  const uint32_t tt = key / P;
  uint32_t p = key % P;
  const int n = s->n_robots;
  for (int a = 0; a < n; ++a) {
    const uint32_t row = (uint32_t)(n - 1 - a);
    if (p < row) {
      *t = (int32_t)tt;
      *i = a;
      *j = a + 1 + (int32_t)p;
      return MRV_OK;
    }
    p -= row;
  }
  return MRV_EINVAL;
}

}  // extern "C"
