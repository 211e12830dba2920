/* mrv_example.c -- the C ABI of libmrv.so used from plain C (no Python, no torch).
 *
 * Two SE(3) bodies, each one sphere of radius 0.5 (PAPER.md:138's sphere representation),
 * no obstacles; three motions of K = 2 waypoints over T = 11 timesteps
 * (t_k = k (T-1)/(K-1), include/mrv.h):
 *   0: body 0 slides along x from 0 to 10 through body 1 parked at x = 5
 *      -> first strict overlap |c0 - c1| < 1 at t = 5 (t = 4, 6 are exactly 1 apart);
 *   1: body 1 parked at x = 20: never within reach -> valid, no conflict;
 *   2: as 0 but body 1 at y = 0.99: the centres come within 0.99 < 1 only at t = 5.
 * MotVal (Alg. 1) and FFC (Alg. 2, key t * P + rank(i, j), P = 1) on the device, the key
 * decoded with mrv_decode_conflict.  Exit status 0 iff every result is the expected one.
 *
 *   cc -std=c11 examples/mrv_example.c -Iinclude -I/usr/local/cuda/include \
 *      -Lpaper_2604_23960_b200 -lmrv -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,...
 */
#include <stdio.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "mrv.h"

#define M 3
#define K 2
#define S 7
#define T 11

static int check(mrv_status st, const char* what) {
  if (st != MRV_OK) {
    fprintf(stderr, "%s: %s\n", what, mrv_status_string(st));
    return 1;
  }
  return 0;
}

int main(void) {
  if (mrv_abi_version() != MRV_ABI_VERSION) {
    fprintf(stderr, "ABI %d, header %d\n", mrv_abi_version(), MRV_ABI_VERSION);
    return 1;
  }
  const int32_t link0[1] = {0};
  const float ball[4] = {0.0f, 0.0f, 0.0f, 0.5f};
  mrv_robot_desc robots[2];
  memset(robots, 0, sizeof robots);
  for (int r = 0; r < 2; ++r) {
    robots[r].kind = MRV_SE3;
    robots[r].dof = 7;
    robots[r].n_spheres = 1;
    robots[r].sphere_link = link0;
    robots[r].sphere = ball;
  }
  const mrv_env_desc env = {0, NULL, 0, NULL};
  mrv_scene* scene = NULL;
  if (check(mrv_create_scene(robots, 2, &env, 0, &scene), "mrv_create_scene")) return 1;

  /* waypoints [M][n = 2][K][S]: SE(3) poses (x, y, z, qw, qx, qy, qz) */
  float wp[M][2][K][S];
  memset(wp, 0, sizeof wp);
  const float body1[M][2] = {{5.0f, 0.0f}, {20.0f, 0.0f}, {5.0f, 0.99f}};
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < K; ++k) {
      wp[m][0][k][0] = 10.0f * (float)k;   /* body 0: x = 0 -> 10 */
      wp[m][0][k][3] = 1.0f;
      wp[m][1][k][0] = body1[m][0];        /* body 1: parked */
      wp[m][1][k][1] = body1[m][1];
      wp[m][1][k][3] = 1.0f;
    }
  float* d_wp = NULL;
  uint8_t* d_valid = NULL;
  uint32_t* d_key = NULL;
  if (cudaMalloc((void**)&d_wp, sizeof wp) != cudaSuccess || cudaMalloc((void**)&d_valid, M) != cudaSuccess ||
      cudaMalloc((void**)&d_key, M * sizeof(uint32_t)) != cudaSuccess ||
      cudaMemcpy(d_wp, wp, sizeof wp, cudaMemcpyHostToDevice) != cudaSuccess) {
    fprintf(stderr, "CUDA allocation / copy failed\n");
    return 1;
  }
  mrv_motion_batch batch;
  memset(&batch, 0, sizeof batch);
  batch.n_motions = M;
  batch.n_waypoints = K;
  batch.dof_stride = S;
  batch.waypoints = d_wp;
  batch.fixed_timesteps = T;
  if (check(mrv_motval_batch(scene, &batch, 0, d_valid, NULL), "mrv_motval_batch") ||
      check(mrv_ffc_batch(scene, &batch, 0, d_key, NULL), "mrv_ffc_batch"))
    return 1;
  uint8_t valid[M];
  uint32_t key[M];
  if (cudaMemcpy(valid, d_valid, M, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(key, d_key, sizeof key, cudaMemcpyDeviceToHost) != cudaSuccess) {
    fprintf(stderr, "CUDA copy failed\n");
    return 1;
  }
  const uint8_t want_valid[M] = {0, 1, 0};
  const int want_t[M] = {5, -1, 5};
  int bad = 0;
  for (int m = 0; m < M; ++m) {
    int32_t t, i, j;
    if (check(mrv_decode_conflict(scene, key[m], &t, &i, &j), "mrv_decode_conflict")) return 1;
    printf("motion %d: valid %d, first conflict t = %d between robots %d and %d\n", m, valid[m], t, i, j);
    bad |= valid[m] != want_valid[m] || t != want_t[m] || (t >= 0 && (i != 0 || j != 1));
  }
  uint32_t status = 0;
  if (check(mrv_device_status(scene, NULL, 1, &status), "mrv_device_status")) return 1;
  bad |= status != 0;
  mrv_destroy_scene(scene);
  cudaFree(d_wp);
  cudaFree(d_valid);
  cudaFree(d_key);
  printf(bad ? "example: MISMATCH\n" : "example: ok\n");
  return bad;
}
