// scene_impl.h -- the opaque mrv_scene (host side).  Not part of the ABI.
#pragma once
#include <atomic>
#include <cstdint>
#include <mutex>
#include <vector>

#include "mrv_internal.h"

struct mrv_scene {
  int device = 0;
  int sm_count = 0;
  int max_smem_optin = 0;
  int n_robots = 0, n_pairs = 0, total_spheres = 0;
  bool fuse_env_ok = false;   // every robot a fast-DH chain with the same dof (MotVal fk_env_fused)
  std::vector<int> kinds;
  mrv::DevScene ds{};
  std::vector<uint8_t> h_blob;
  void* d_blob = nullptr;
  unsigned long long* d_ring = nullptr;   // MRV_MAX_INFLIGHT work counters for persistent scheduling
  uint32_t* d_status = nullptr;           // device status word (MRV_DEVERR_* bits, mrv_device_status)
  mutable std::atomic<uint32_t> ring_next{0};
  // launch-configuration cache: (kernel, per-warp bytes) -> (warps per CTA, CTAs per SM, smem)
  struct LaunchCfg {
    const void* key;          // the first candidate instance (lookup key) and its staged bytes
    uint32_t stage_key;
    const void* fn;           // the chosen instance
    uint32_t warp_bytes, stage_bytes;
    int req_wpc;
    int wpc, occ;
    size_t smem;
  };
  mutable std::mutex cfg_mu;
  mutable std::vector<LaunchCfg> cfg_cache;
  // mrv_pp_motval_batch: device copies of the (focus, partner) level-1 segment tables
  struct PPSegs {
    int focus;
    uint64_t partners;
    void* d;
    int n;
  };
  mutable std::vector<PPSegs> pp_seg_cache;
  // mrv_run_host_batch: two device staging buffers, a copy stream and its events
  mutable std::mutex host_mu;
  mutable void* d_stage[2] = {nullptr, nullptr};
  mutable size_t stage_bytes = 0;
  mutable void* copy_stream = nullptr;      // cudaStream_t
  mutable void* ev_copied[2] = {nullptr, nullptr};
  mutable void* ev_free[2] = {nullptr, nullptr};
  mutable void* ev_free2[2] = {nullptr, nullptr};      // staging b released by the MotVal stream (both queries)
  // chunk i's kernels run on comp_stream[i & 1] (FFC, when both queries run: comp_stream[2 + (i & 1)]),
  // so each chunk's kernels fill the previous chunk's tail
  mutable void* comp_stream[4] = {nullptr, nullptr, nullptr, nullptr};
  mutable void* ev_join[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
};
