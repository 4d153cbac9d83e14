// nccl_stats.cpp — a compiled C caller of the path's one collective (test
// harness; built by tests/cpp/Makefile, run by tests/test_cpp_dropin.py on a
// GPU): K4 + ncclAllReduce through mlob_venv_allreduce_episode_stats with a
// real NCCL communicator (one rank per GPU; the gpurun box has one GPU, so a
// one-rank communicator), checked against MarketVecEnv::episode_stats
// (rollout.hpp:255-270) computed in env order on the host.
#include <cmath>
#include <cstdio>
#include <cstring>

#include <cuda_runtime.h>
#include <nccl.h>

#include "mlob.h"

#define CHECK(x)                                                          \
  do {                                                                    \
    const mlob_status s_ = (x);                                           \
    if (s_ != MLOB_OK) {                                                  \
      std::printf("FAIL %s: %d %s\n", #x, (int)s_, mlob_last_error());    \
      return 1;                                                           \
    }                                                                     \
  } while (0)

int main() {
  mlob_synth_config sc;
  mlob_default_synth_config(&sc);
  sc.n_messages = 30000;
  sc.state_sample_every = 80;  // = start_stride_steps * messages_per_step
  mlob_host_store* hs = nullptr;
  CHECK(mlob_host_store_synth(&sc, 4, &hs));
  mlob_store* st = nullptr;
  CHECK(mlob_store_upload(hs, 0, &st));
  mlob_env_config cfg;
  mlob_default_env_config(&cfg);
  cfg.steps_per_episode = 5;
  cfg.messages_per_step = 40;
  cfg.start_stride_steps = 2;
  cfg.n_specs = 2;
  mlob_default_agent_spec(&cfg.specs[0]);
  mlob_default_agent_spec(&cfg.specs[1]);
  cfg.specs[1].type = MLOB_EXECUTOR;
  cfg.specs[1].obs_space = MLOB_OBS_EXEC;
  cfg.specs[1].reward = MLOB_REWARD_EXEC;
  cfg.specs[1].params.task_size = 70;
  mlob_venv_desc d;
  std::memset(&d, 0, sizeof d);
  d.store = st;
  d.cfg = cfg;
  d.seed = 2;
  d.n_envs_local = d.n_envs_global = 300;
  d.flags = MLOB_VENV_AUTO_RESET;
  mlob_venv* v = nullptr;
  CHECK(mlob_venv_create(&d, &v));
  CHECK(mlob_venv_reset_all(v));
  for (uint64_t t = 0; t < 17; ++t) CHECK(mlob_venv_step_random(v, 0, t));  // 3 episodes per env

  ncclComm_t comm;
  int dev = 0;
  if (ncclCommInitAll(&comm, 1, &dev) != ncclSuccess) {
    std::printf("FAIL ncclCommInitAll\n");
    return 1;
  }
  mlob_episode_stats red[2], loc[2];
  CHECK(mlob_venv_allreduce_episode_stats(v, comm, red));
  CHECK(mlob_venv_allreduce_episode_stats(v, nullptr, loc));
  int fail = 0;
  for (int t = 0; t < 2; ++t) {
    mlob_episode_stats ref;
    CHECK(mlob_venv_episode_stats(v, t, &ref));
    const bool exact = red[t].pv_sum == ref.pv_sum && red[t].slippage_sum == ref.slippage_sum &&
                       red[t].inventory_sq_sum == ref.inventory_sq_sum && red[t].episodes == ref.episodes &&
                       std::memcmp(&red[t], &loc[t], sizeof red[t]) == 0;
    const double tol = 1e-12 * (std::fabs(ref.completion_sum) > 1.0 ? std::fabs(ref.completion_sum) : 1.0);
    const bool comp = std::fabs(red[t].completion_sum - ref.completion_sum) <= tol;
    std::printf("type %d: episodes %lld pv %.17g slip %.17g completion %.17g (ref %.17g) inv2 %.17g\n", t,
                (long long)red[t].episodes, red[t].pv_sum, red[t].slippage_sum, red[t].completion_sum,
                ref.completion_sum, red[t].inventory_sq_sum);
    if (!exact || !comp || ref.episodes < 600) ++fail;
  }
  ncclCommDestroy(comm);
  mlob_venv_destroy(v);
  mlob_store_free(st);
  mlob_host_store_free(hs);
  if (fail) {
    std::printf("FAIL\n");
    return 1;
  }
  std::printf("OK: ncclAllReduce of the K4 episode statistics == env-ordered episode_stats\n");
  return 0;
}
