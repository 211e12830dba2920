/* orc.h -- fp64 scalar CPU ORACLE for batched multi-robot MotVal / FFC.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code, header, table or constant with the CUDA path
 * (paper_2604_23960_b200/csrc, include/mrv.h) and neither includes the other.
 *
 * What it computes is the plain definition, not a
 * re-enactment of the paper's batching:
 *   - MotVal(P, E) is false iff some timestep has a robot-obstacle or
 *     robot-robot sphere overlap ("A collision of any kind at any timestep
 *     invalidates the motion"; Alg. 1).
 *   - FFC(P) is the lexicographically smallest (t, i, j) with a robot-robot
 *     overlap ("the *first* conflict"; Alg. 2's strict
 *     replacement "C.t > t_conflict", induces (t, i, j) order).
 * Inputs are the same fp32 arrays the GPU reads, promoted to double.
 * Readings of silent/ambiguous passages are listed in DESIGN.md §3 (c.1..c.25).
 *
 * Pins: tests/test_oracle_pins.py (closed forms, hand FK, DH-vs-chain, slerp,
 * brute-force Alg. 1/2 transcriptions, cross-query invariant, Cross scenario).
 */
#ifndef ORC_H
#define ORC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_CHAIN = 0, ORC_SE2 = 1, ORC_SE3 = 2 };
#define ORC_NONE 0xFFFFFFFFu

typedef struct {
  int32_t kind;               /* ORC_CHAIN / ORC_SE2 / ORC_SE3 */
  int32_t dof;                /* chain joints; SE2: 3; SE3: 7 */
  const float* joint_origin;  /* chain: [dof][12] row-major 3x4 */
  const int32_t* joint_type;  /* chain: [dof] 0 revolute about z, 1 prismatic along z */
  const float* base;          /* chain: [12] or NULL (identity) */
  int32_t n_spheres;
  const int32_t* sphere_link; /* [n_spheres] */
  const float* sphere;        /* [n_spheres][4] (ox, oy, oz, r) */
  int32_t n_self_pairs;       /* link pairs checked for self-collision */
  const int32_t* self_pairs;  /* [n_self_pairs][2] (link a, link b) */
} orc_robot;

/* `check_env` arguments below are a bit mask: ORC_ENV_OBSTACLES checks robot-obstacle
 * overlaps, ORC_ENV_SELF the robot's self-collision link pairs ("robot-obstacle
 * validation also checks the robot for self-collision"). */
enum { ORC_ENV_OBSTACLES = 1, ORC_ENV_SELF = 2 };

typedef struct {
  int32_t n_robots;
  const orc_robot* robots;
  int32_t n_obs_spheres;
  const float* obs_spheres;   /* [n][4] (x, y, z, R) */
  int32_t n_boxes;
  const float* boxes;         /* [n][6] (lo xyz, hi xyz) */
} orc_scene;

typedef struct {
  int64_t M;
  int32_t K;                  /* waypoints per robot */
  int32_t S;                  /* dof stride */
  const float* waypoints;     /* [M][n_robots][K][S] */
  const int32_t* n_timesteps; /* [M] or NULL */
  int32_t fixed_timesteps;
  const int32_t* robot_timesteps; /* [M][n_robots] or NULL: per-robot path lengths; the motion's
                                     horizon is their maximum (t_max = max |p_i|) and a
                                     robot stays at its last waypoint after its path ends */
} orc_motions;

/* Configuration of robot r of motion m at timestep t (reading c.4 / c.8). */
void orc_interp(const orc_scene* sc, const orc_motions* mo, int64_t m, int32_t r, int32_t t, double* q);

/* World sphere centres of one robot at configuration q, [n_spheres][3]
 * (SpheresFK; chain convention reading c.9). */
void orc_fk(const orc_robot* rb, const double* q, double* xyz);

/* All robots' centres at state (m, t), concatenated in scene order. */
void orc_centres_at(const orc_scene* sc, const orc_motions* mo, int64_t m, int32_t t, double* xyz);

/* Per-state tables for motion m over all t: env_hit/env_sep [T][n_robots],
 * pair_hit/pair_sep [T][P] (strict predicates, signed separations). */
void orc_state_tables(const orc_scene* sc, const orc_motions* mo, int64_t m, int32_t check_env,
                      int32_t* env_hit, double* env_sep, int32_t* pair_hit, double* pair_sep);

/* Composite configurations q [N][n_robots][S]: min signed separation over
 * obstacles (if check_env) and all pairs; strict hit flag. */
void orc_config_eval(const orc_scene* sc, const float* q, int64_t N, int32_t S, int32_t check_env,
                     int32_t n_threads, double* min_sep, uint8_t* hit);

/* Plain-definition MotVal with the band classification of SURVEY §8(c):
 * valid[m] strict verdict; cls[m] = 0 exact-comparable, 1 ambiguous motion;
 * def_hit[m] = 1 if some state has min sep <= -band. */
void orc_motval_batch(const orc_scene* sc, const orc_motions* mo, int32_t check_env, double band,
                      int32_t n_threads, uint8_t* valid, uint8_t* cls, uint8_t* def_hit);

/* As orc_motval_batch, plus per-motion state counts (either pointer may be NULL):
 * amb_states[m] = number of scanned states whose minimum signed separation (over the
 * obstacles, if check_env, and all robot pairs) lies strictly within (-band, +band)
 * (BASELINE.json north_star: "states whose oracle minimum signed sphere separation is
 * within 1e-4 m of zero ... are counted and reported"); scanned[m] = states classified.
 * full_scan = 0 stops at the first definite hit (as orc_motval_batch); 1 classifies all T. */
void orc_motval_batch_ex(const orc_scene* sc, const orc_motions* mo, int32_t check_env, double band,
                         int32_t full_scan, int32_t n_threads, uint8_t* valid, uint8_t* cls, uint8_t* def_hit,
                         int32_t* amb_states, int32_t* scanned);

/* Plain-definition FFC: key = t*P + rank(i,j) of the lexmin strict overlap
 * (ORC_NONE if none); k_lo = min key with sep < band; k_hi = min key with
 * sep <= -band; amb = 1 if a (t,pair) with key <= key (all if none) has
 * |sep| < band. */
void orc_ffc_batch(const orc_scene* sc, const orc_motions* mo, double band, int32_t n_threads,
                   uint32_t* key, uint32_t* k_lo, uint32_t* k_hi, uint8_t* amb);

/* As orc_ffc_batch, plus per-motion counts: amb_states[m] = scanned timesteps at which
 * some robot pair's signed separation lies within (-band, +band); scanned[m] = timesteps
 * classified (full_scan = 0: up to the first t with a definite-hit pair; 1: all T). */
void orc_ffc_batch_ex(const orc_scene* sc, const orc_motions* mo, double band, int32_t full_scan,
                      int32_t n_threads, uint32_t* key, uint32_t* k_lo, uint32_t* k_hi, uint8_t* amb,
                      int32_t* amb_states, int32_t* scanned);

/* Signed separation of pair (i<j) at state (m, t). */
double orc_pair_sep(const orc_scene* sc, const orc_motions* mo, int64_t m, int32_t t, int32_t i, int32_t j);

/* CPU baseline (the paper's "sphere-based" sequential
 * linear scan): t ascending, exit at the first strict hit.
 * Returns the number of states evaluated. */
int64_t orc_baseline_motval(const orc_scene* sc, const orc_motions* mo, int32_t check_env, int32_t n_threads,
                            uint8_t* valid);
int64_t orc_baseline_ffc(const orc_scene* sc, const orc_motions* mo, int32_t n_threads, uint32_t* key);

/* PP-ST-RRT's MotVal variant: "the outer loop ... is replaced with only
 * the current robot and the inner loop ... iterates over only higher priority robots", whose
 * paths are fixed ("treated as dynamic obstacles").  Candidate m is a motion
 * of robot `focus` alone: cand->waypoints [M][1][K][S] with its own T_m (n_timesteps or
 * fixed).  At its local timestep t the focus robot is at its interpolated configuration and
 * every robot r with bit r of partner_mask set at the configuration of the fixed path
 * paths (M = 1, [1][n_robots][Kp][S], per-robot lengths in robot_timesteps: stay at the goal)
 * at the absolute timestep min(t_start[m] + t, horizon - 1).  A state collides iff the focus
 * robot overlaps an obstacle (check_env bit 1) or one of its self pairs (bit 2) or any
 * partner.  Outputs and band classification as orc_motval_batch. */
void orc_pp_motval_batch(const orc_scene* sc, int32_t focus, uint64_t partner_mask, const orc_motions* cand,
                         const int32_t* t_start, const orc_motions* paths, int32_t horizon, int32_t check_env,
                         double band, int32_t n_threads, uint8_t* valid, uint8_t* cls, uint8_t* def_hit);

#ifdef __cplusplus
}
#endif
#endif
