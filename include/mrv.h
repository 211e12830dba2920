/* mrv.h -- C ABI of libmrv.so: batched multi-robot MotionValidation (MotVal) and
 * FindFirstConflict (FFC) on NVIDIA B200 (sm_100a).
 *
 * Paper: arxiv 2604.23960, "vector-accelerated multi-robot primitives".
 * Citations "PAPER.md:n" are lines of /root/reference/PAPER.md (the paper's
 * LaTeX), "SPEC.md:n" of the CPU-program spec, "§8(x)" of SURVEY.md.
 *
 * Conventions (all entry points):
 *   - Floating point is fp32, integers as declared; arrays are row-major and
 *     densely packed.
 *   - No C++ exception crosses the ABI; every call returns an mrv_status.
 *   - Argument validation is synchronous and happens BEFORE anything is
 *     enqueued: on MRV_EINVAL / MRV_ERANGE / MRV_EUNSUPPORTED nothing was
 *     launched and no output was touched.
 *   - Batch calls enqueue on `cuda_stream` (a cudaStream_t; NULL = legacy
 *     default stream) and return without synchronising.  Launch failures
 *     are MRV_ECUDA (cudaGetLastError); asynchronous device faults surface
 *     at the caller's next synchronisation.
 *   - Ownership: mrv_create_scene deep-copies every input array (host and
 *     device copies owned by the scene); the caller keeps ownership of its
 *     arrays.  Batch inputs/outputs are caller-owned DEVICE buffers on the
 *     scene's device and must stay alive until the enqueued work completes.
 *   - Thread safety: a scene is immutable after creation; concurrent calls
 *     on the same scene from several host threads / streams are safe (up to
 *     MRV_MAX_INFLIGHT calls in flight per scene at once).
 *   - The library never falls back to a CPU path: without a usable
 *     sm_100 device, mrv_create_scene returns MRV_ECUDA.
 */
#ifndef MRV_H
#define MRV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MRV_ABI_VERSION 5
#define MRV_NO_CONFLICT 0xFFFFFFFFu
#define MRV_MAX_INFLIGHT 256

typedef enum {
  MRV_OK = 0,
  MRV_EINVAL = 1,       /* bad argument (null pointer, radius <= 0, box lo >= hi, dof < 1, K < 1, T < 1, ...) */
  MRV_ENOMEM = 2,       /* host or device allocation failed */
  MRV_ECUDA = 3,        /* CUDA runtime error (no device, launch failure, wrong architecture) */
  MRV_ERANGE = 4,       /* a result does not fit its encoding (FFC: T * P >= 2^32 - 1) */
  MRV_EUNSUPPORTED = 5  /* valid request this build does not support (e.g. dof > MRV_MAX_DOF) */
} mrv_status;

typedef enum { MRV_CHAIN = 0, MRV_SE2 = 1, MRV_SE3 = 2 } mrv_robot_kind;

#define MRV_MAX_DOF 16        /* chain joints per robot */
#define MRV_MAX_KNOTS (1 << 20) /* waypoints per motion (K) */
#define MRV_MAX_ROBOTS 64
#define MRV_MAX_SPHERES_PER_FRAME 1024

/* A robot: a kinematic chain or a rigid body carrying collision spheres
 * ("sphere-based representation of a robot"; SpheresFK
 * "return[s] the positions of each sphere").
 *
 * Chain FK (reading c.9 in DESIGN.md): T_0 = base, T_j = T_{j-1} * O_j * J(q_j)
 * with J = Rz(q_j) (revolute) or Tz(q_j) (prismatic); the spheres of link j
 * are expressed in frame T_j.  SE2: q = (x, y, theta), c = (x + R(theta) o_xy,
 * o_z).  SE3: q = (x, y, z, qw, qx, qy, qz), c = p + R(q) o with
 * R from q using s = 2 / (q.q).  3x4 transforms are row-major [R | p]. */
typedef struct {
  int32_t kind;                 /* mrv_robot_kind */
  int32_t dof;                  /* chain: n_joints in [1, MRV_MAX_DOF]; SE2: 3; SE3: 7 */
  const float* joint_origin;    /* chain: HOST [dof][12] fixed transform O_j; ignored otherwise */
  const int32_t* joint_type;    /* chain: HOST [dof] 0 = revolute about local z, 1 = prismatic along local z */
  const float* base;            /* chain: HOST [12] world <- base, or NULL = identity; ignored otherwise */
  int32_t n_spheres;            /* >= 1 */
  const int32_t* sphere_link;   /* HOST [n_spheres] chain: link in [0, dof); SE2/SE3: 0 */
  const float* sphere;          /* HOST [n_spheres][4] (ox, oy, oz, r) in the link/body frame, r > 0 */
  int32_t n_self_pairs;         /* chain: link pairs checked for self-collision under MRV_CHECK_SELF (>= 0) */
  const int32_t* self_pairs;    /* HOST [n_self_pairs][2] distinct links in [0, dof) (NULL if n_self_pairs = 0);
                                   "robot-obstacle validation also checks the robot for self-collision",
                                   PAPER.md:240 */
} mrv_robot_desc;

/* Environment E: sphere and axis-aligned box obstacles
 * (BASELINE north_star; reading c.2).  Both counts may be 0. */
typedef struct {
  int32_t n_spheres;
  const float* spheres;         /* HOST [n_spheres][4] (x, y, z, R), R > 0 */
  int32_t n_boxes;
  const float* boxes;           /* HOST [n_boxes][6] (lo x, y, z, hi x, y, z), lo < hi per axis */
} mrv_env_desc;

/* A batch of M synchronized multi-robot motions P = {p_1..p_n}
 * (PAPER.md:288, :337).  Robot r of motion m follows the knots
 * waypoints[m][r][0..K-1] placed at timesteps t_k = k (T_m - 1)/(K - 1); the
 * motion is "discretiz[ed] into intermediate configurations",
 * one per timestep t = 0..T_m-1, by linear interpolation
 * (SE3 orientation: slerp).  Reading c.4: exact at knots. */
typedef struct {
  int64_t n_motions;            /* M >= 0 */
  int32_t n_waypoints;          /* K >= 1 (<= MRV_MAX_KNOTS, else MRV_EUNSUPPORTED), same for every motion and robot */
  int32_t dof_stride;           /* S >= max robot dof; robot r reads the first dof_r entries */
  const float* waypoints;       /* DEVICE [M][n_robots][K][S]; SE3 quaternions (qw,qx,qy,qz) pre-aligned
                                   so consecutive knots have dot >= 0; SE2 theta pre-unwrapped */
  const int32_t* n_timesteps;   /* DEVICE [M], each >= 1; or NULL to use fixed_timesteps for every motion.  A
                                   device T < 1 (or, for FFC, T * P >= 2^32 - 1) cannot be checked before the
                                   launch: the kernel leaves that motion's result at "valid" / MRV_NO_CONFLICT
                                   and sets a bit in the scene's device status word (mrv_device_status) */
  int32_t fixed_timesteps;      /* >= 1 when n_timesteps == NULL */
  const int32_t* robot_timesteps; /* DEVICE [M][n_robots] per-robot path lengths (each >= 1), or NULL.  When
                                     given, motion m spans t_max = max_r T_mr timesteps, robot r's
                                     knots sit at k (T_mr - 1)/(K - 1) and it stays at its last waypoint for
                                     t >= T_mr; n_timesteps / fixed_timesteps are then ignored.  Out-of-range
                                     values are reported as for n_timesteps */
} mrv_motion_batch;

/* flags */
enum {
  MRV_CHECK_ENV = 1u << 0,          /* MotVal: include robot-obstacle checks (Alg. 1 check_environment) */
  MRV_ORDER_HIERARCHICAL = 1u << 1, /* MotVal: all obstacle batches before any robot-robot batch */
  MRV_PACK_LINEAR = 1u << 2,        /* MotVal: linear instead of rake batches; FFC is always linear */
  MRV_DIAG_NO_EARLY_EXIT = 1u << 3, /* evaluate every state (diagnostic / roofline); results unchanged */
  MRV_DIAG_NO_BROADPHASE = 1u << 4, /* skip bounding-sphere culling (diagnostic); results unchanged */
  MRV_CHECK_SELF = 1u << 5,         /* MotVal: include each robot's self-collision link pairs, tested with the
                                       robot-obstacle checks; FFC ignores it */
  MRV_FOCUS = 1u << 6,              /* _ex only: apply opts->focus_robot / opts->partner_mask (PP-ST-RRT variant) */
  MRV_PACK_SEQUENTIAL = 1u << 7     /* MotVal: run Alg. 1's own batch loop (rake batches of W states, b = 0, 1, ...,
                                       PAPER.md:289-322) instead of the spread packing the default launch uses
                                       when it applies (see mrv_motval_batch); results unchanged */
};

/* Optional launch knobs and diagnostics for the _ex entry points.  Zero-initialise
 * for defaults.  None of them changes any result. */
typedef struct {
  int32_t states_per_batch;     /* W, states per warp batch: 0 = auto, else one of 4, 8, 16, 32 */
  int32_t n_slices;             /* warps cooperating on one motion's batches: 0 = auto, else >= 1 */
  uint64_t* counters;           /* DEVICE [MRV_NUM_COUNTERS] or NULL: work counters are atomically ADDED */
  uint32_t* batches_evaluated;  /* DEVICE [M] or NULL: batches evaluated per motion (effort) */
  int32_t t_begin;              /* time window [t_begin, t_end): only these timesteps are evaluated; splitting */
  int32_t t_end;                /*   one long horizon across devices (FFC: all_reduce(MIN) of the keys, MotVal:
                                     AND of the flags); t_end <= 0 means T.  0/0 = the whole motion */
  int32_t focus_robot;          /* with MRV_FOCUS: the PP-ST-RRT MotVal variant -- the outer */
  uint64_t partner_mask;        /*   robot loop is only `focus_robot` (its obstacle/self checks) and the inner
                                     loop only the robots j with bit j set (the higher-priority robots); every
                                     other robot is ignored.  FFC: only pairs (focus, partner) */
  int32_t warps_per_cta;        /* 0 = auto (the residency-maximising count), else 1..20 (diagnostic: the
                                     race stress test varies it; results unchanged).  MRV_EUNSUPPORTED above
                                     16 (MotVal) or 18 (FFC; 20 where its lean instance stores compact link
                                     frames), or if that many warps' shared memory does not fit one CTA */
} mrv_launch_opts;

/* Device status bits (mrv_device_status): conditions only the kernel can see, because
 * the values live in device memory. */
enum {
  MRV_DEVERR_TIMESTEPS = 1u << 0,   /* a per-motion / per-robot T < 1 */
  MRV_DEVERR_RANGE = 1u << 1,       /* FFC: a motion's T * P >= 2^32 - 1 (its key does not fit uint32) */
  MRV_DEVERR_START = 1u << 2        /* mrv_pp_motval_batch: a t_start < 0 (that candidate is left valid) */
};

enum {
  MRV_CNT_STATES = 0,           /* (motion, timestep) states whose FK was evaluated */
  MRV_CNT_ROBOT_STATES,         /* robot FK evaluations */
  MRV_CNT_JOINTS,               /* chain joint transforms composed */
  MRV_CNT_ENV_BROAD,            /* group-bound vs obstacle tests */
  MRV_CNT_ENV_NARROW,           /* sphere vs obstacle tests */
  MRV_CNT_RR_BROAD,             /* group-bound vs group-bound tests (second level) */
  MRV_CNT_RR_NARROW,            /* sphere vs sphere tests */
  MRV_CNT_SPHERE_XFORM,         /* sphere centres computed in the narrow phase */
  MRV_CNT_RR_SUPER,             /* supergroup-bound vs supergroup-bound tests (first level) */
  MRV_CNT_SUPER_BOUNDS,         /* supergroup bounds derived from member bounds */
  MRV_CNT_SELF_BROAD,           /* group-bound vs group-bound self-collision tests */
  MRV_CNT_RR_CAPSULE,           /* group-capsule vs group-capsule prefilter tests (before the sphere tests) */
  MRV_CNT_TABLE_BYTES,          /* bytes read from a PP-ST-RRT partner table (mrv_pp_motval_batch) */
  MRV_NUM_COUNTERS = 13
};

typedef struct mrv_scene mrv_scene;  /* opaque, immutable after create */

/* Create a scene on `cuda_device`: validates every robot and obstacle
 * (SPEC.md:24,52 radius > 0; SPEC.md:40,59 box lo < hi), folds the base into
 * the chain, precomputes per-frame bounding spheres (inflated by 1e-4 m so the
 * fp32 broad phase is conservative), a uniform obstacle grid (per cell, the
 * obstacles within the largest group bound of it) and the robot-robot pair lists, and
 * uploads one contiguous device table.  n_robots in [1, MRV_MAX_ROBOTS].
 * Errors: MRV_EINVAL (any invalid field; *out untouched), MRV_ENOMEM,
 * MRV_ECUDA (no device / not sm_100), MRV_EUNSUPPORTED (dof > MRV_MAX_DOF, more than 65535
 * obstacles in total, more than 65535 collision groups, or more than 2047 collision
 * groups when the scene has obstacles). */
mrv_status mrv_create_scene(const mrv_robot_desc* robots, int32_t n_robots, const mrv_env_desc* env,
                            int32_t cuda_device, mrv_scene** out);

/* Free a scene (NULL is a no-op).  The caller must ensure no enqueued work
 * still uses it. */
mrv_status mrv_destroy_scene(mrv_scene* s);

/* MotionValidation, Alg. 1: out_valid[m] = 1 iff no
 * timestep of motion m has a robot-robot sphere overlap or (with
 * MRV_CHECK_ENV) a robot-obstacle overlap or (with MRV_CHECK_SELF) an overlap of a
 * robot's self-collision link pair ("A collision of any kind at any
 * timestep invalidates the motion").  Overlap is strict:
 * |c_a - c_b|^2 < (r_a + r_b)^2; sphere-box: squared distance to the box < r^2
 * (reading c.1).  Evaluation is in rake-ordered warp batches with early
 * termination at the first hit; flags
 * MRV_ORDER_HIERARCHICAL / MRV_PACK_LINEAR change effort, never results.  Spread
 * packing (reading c.28): with default flags (or MRV_CHECK_ENV alone), a fixed
 * or per-motion T (not robot_timesteps), no time window, effort output or caller-chosen
 * W / slices, a team of 3-4 fast-DH robots and enough motions for one warp per motion, a
 * warp evaluates up to 8 motions at once (fewer when the batch has under 32 motions per
 * resident warp), one state each per batch, each motion's timesteps in the order
 * (T/2 + b * step) mod T (step ~ 0.618 T, coprime with T) -- fewer states evaluated
 * before the first hit, same results; MRV_PACK_SEQUENTIAL turns it off.
 * out_valid: DEVICE uint8 [M], fully written.  M = 0: MRV_OK, no launch. */
mrv_status mrv_motval_batch(const mrv_scene* s, const mrv_motion_batch* b, uint32_t flags, uint8_t* out_valid,
                            void* cuda_stream);
mrv_status mrv_motval_batch_ex(const mrv_scene* s, const mrv_motion_batch* b, uint32_t flags, uint8_t* out_valid,
                               void* cuda_stream, const mrv_launch_opts* opts);

/* FindFirstConflict, Alg. 2: out_key[m] = t * P + rank(i, j)
 * for the lexicographically smallest (t, i, j), i < j, at which robots i and j
 * have a strict sphere overlap (the "first conflict"; ties at
 * equal t go to the lexicographically first pair, as Alg. 2's strict
 * replacement "C.t > t_conflict", induces), or MRV_NO_CONFLICT.
 * P = n(n-1)/2, rank(i, j) = i n - i(i+1)/2 + (j - i - 1).  Obstacles are
 * ignored.  Linear batches, skipping batches that start
 * after a known conflict.  Errors: MRV_ERANGE if
 * fixed_timesteps * P >= 2^32 - 1 (per-motion T in device memory: the motion's
 * key is MRV_NO_CONFLICT and MRV_DEVERR_RANGE is raised in the device status word).
 * out_key: DEVICE uint32 [M], fully written. */
mrv_status mrv_ffc_batch(const mrv_scene* s, const mrv_motion_batch* b, uint32_t flags, uint32_t* out_key,
                         void* cuda_stream);
mrv_status mrv_ffc_batch_ex(const mrv_scene* s, const mrv_motion_batch* b, uint32_t flags, uint32_t* out_key,
                            void* cuda_stream, const mrv_launch_opts* opts);

/* Decode an FFC key into (t, i, j) (host-side arithmetic on the scene's n).
 * MRV_NO_CONFLICT -> MRV_OK with t = i = j = -1.  Key out of range -> MRV_EINVAL. */
mrv_status mrv_decode_conflict(const mrv_scene* s, uint32_t key, int32_t* t, int32_t* i, int32_t* j);

/* SpheresFK export for parity: world-frame centres of every
 * sphere of every robot (scene order, robots concatenated) at the states
 * (motion[q], t[q]).  motion, t: DEVICE [n_queries]; out_xyz: DEVICE float
 * [n_queries][total_spheres][3].  Uses the same interpolation and FK code as
 * the MotVal/FFC kernels.  Out-of-range motion/t entries produce NaN rows. */
mrv_status mrv_fk_states(const mrv_scene* s, const mrv_motion_batch* b, int64_t n_queries, const int64_t* motion,
                         const int32_t* t, float* out_xyz, void* cuda_stream);

/* Scene facts: n_robots, n_pairs P, total spheres, total frames. */
mrv_status mrv_scene_info(const mrv_scene* s, int32_t* n_robots, int32_t* n_pairs, int32_t* total_spheres,
                          int32_t* total_frames);

/* End-to-end call with HOST inputs: MotVal (out_valid != NULL, motval_flags) and/or FFC
 * (out_key != NULL, ffc_flags) over a batch whose `waypoints` and `n_timesteps` are
 * HOST arrays (page-locked memory lets the copies overlap; pageable memory works but
 * serialises).  The batch is cut into chunks that grow x4 from min(chunk_motions / 32,
 * max(M / 8, 8192)) up to `chunk_motions` (0 = 1048576) motions; chunk i+1's host-to-device copy runs on a
 * scene-owned copy stream while chunk i's kernels run, through two scene-owned device
 * staging buffers of `chunk_motions` motions each (allocated on first use, kept until
 * mrv_destroy_scene).  Each query's chunks alternate between two scene-owned compute
 * streams (four with both queries), so a chunk's kernels start on the SMs the previous
 * chunk's tail frees and the two queries' kernels overlap.
 * All of it is ordered after the work already on `cuda_stream`, which waits for it.  Results are identical to
 * mrv_motval_batch / mrv_ffc_batch on the same data; outputs are caller-owned [M] buffers
 * in DEVICE memory or in page-locked HOST memory (cudaHostAlloc / cudaHostRegister; the
 * kernels then write a staging copy that each chunk copies back as soon as its kernel is
 * done, overlapped with the later chunks; pageable host memory: MRV_EINVAL).  Returns
 * after enqueueing; work enqueued on `cuda_stream` afterwards sees the results (a host
 * output is complete once that stream reaches it), and the host arrays must stay valid
 * until then.  robot_timesteps must be
 * NULL.  The host T array is range-checked up front (MRV_EINVAL for T < 1, MRV_ERANGE for
 * FFC T * P >= 2^32 - 1), and both queries' launch configurations are validated before
 * the first copy is enqueued, so every synchronous error leaves nothing enqueued; a CUDA
 * error in the middle (MRV_ECUDA) still makes `cuda_stream` wait for what was enqueued.
 * Errors as the batch calls, plus MRV_ENOMEM (staging).  Two host-batch calls on
 * the same scene must not run concurrently (they share the staging buffers). */
mrv_status mrv_run_host_batch(const mrv_scene* s, const mrv_motion_batch* host_batch, uint32_t motval_flags,
                              uint8_t* out_valid, uint32_t ffc_flags, uint32_t* out_key, int64_t chunk_motions,
                              void* cuda_stream);

/* ---- PP-ST-RRT's MotVal variant with shared fixed partner paths ----
 * "PP-ST-RRT plans for one robot at a time, the outer loop ... is replaced with only the
 * current robot and the inner loop ... iterates over only higher priority robots"
 * (PAPER.md:404-405), whose already planned paths are "treated as dynamic obstacles"
 * (PAPER.md:403).  Every candidate motion of the current (focus) robot is checked against
 * the SAME fixed paths, so their per-timestep world geometry is computed once into a
 * partner table and streamed from HBM/L2 by every candidate instead of being recomputed.
 *
 * Partner table: `horizon` rows, one per absolute timestep t = 0..horizon-1; row t holds,
 * for every robot in `partner_mask`, its supergroup bounds, link frames and collision-group
 * bounds at t (rows are mrv_pp_table_bytes / horizon bytes; the layout is internal).  The
 * table is caller-owned DEVICE memory of mrv_pp_table_bytes(horizon) bytes, 16-B aligned. */
mrv_status mrv_pp_table_bytes(const mrv_scene* s, int32_t horizon, uint64_t* bytes);

/* Fill the partner table from the fixed paths: `paths` holds ONE motion (n_motions = 1,
 * DEVICE waypoints [1][n_robots][K][S]; per-robot path lengths in robot_timesteps (DEVICE
 * [1][n_robots]) or one T); robot r at absolute t is at its interpolated configuration at
 * min(t, T_r - 1) (stay at the goal).  Only the rows' entries of the robots in
 * `partner_mask` are written.  horizon >= 1.  Enqueued on cuda_stream. */
mrv_status mrv_pp_build_table(const mrv_scene* s, const mrv_motion_batch* paths, uint64_t partner_mask,
                              int32_t horizon, void* table, void* cuda_stream);

/* MotVal of M candidate motions of robot `focus_robot` against the partners' fixed paths:
 * out_valid[m] = 1 iff for every local timestep t < T_m of candidate m there is no overlap
 * of the focus robot with an obstacle (MRV_CHECK_ENV), with its own self-collision pairs
 * (MRV_CHECK_SELF) or with a robot j in partner_mask at the absolute timestep
 * min(t_start[m] + t, horizon - 1) (read from `table`, built for a superset of
 * partner_mask).  Robots outside {focus} + partner_mask are ignored.  The batch holds only
 * the focus robot: DEVICE waypoints [M][1][K][S] (S >= its dof), per-motion or fixed T,
 * robot_timesteps NULL; t_start: DEVICE int32 [M], each >= 0 (a negative one leaves that
 * candidate at valid and raises MRV_DEVERR_START).  Flags as mrv_motval_batch
 * (MRV_FOCUS implied); opts as the _ex calls (focus_robot / partner_mask ignored).  Same
 * rake-ordered early exit; results equal the oracle's orc_pp_motval_batch. */
mrv_status mrv_pp_motval_batch(const mrv_scene* s, const mrv_motion_batch* focus_batch, const int32_t* t_start,
                               int32_t focus_robot, uint64_t partner_mask, const void* table, int32_t horizon,
                               uint32_t flags, uint8_t* out_valid, void* cuda_stream, const mrv_launch_opts* opts);

/* The scene's device status word: the OR of the MRV_DEVERR_* bits raised by every batch
 * call on the scene since it was last cleared.  Synchronises `cuda_stream` (call it on
 * the stream the batches ran on, after them), writes the word to *bits and, if `clear`,
 * resets it to 0.  MRV_EINVAL on null arguments, MRV_ECUDA on a CUDA error. */
mrv_status mrv_device_status(const mrv_scene* s, void* cuda_stream, int32_t clear, uint32_t* bits);

/* Human-readable status name (static storage). */
const char* mrv_status_string(mrv_status st);

/* MRV_ABI_VERSION of the loaded library. */
int32_t mrv_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MRV_H */
