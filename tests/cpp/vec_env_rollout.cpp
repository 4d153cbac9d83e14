// vec_env_rollout.cpp — the C++ drop-in exercised through the reference's own
// templates (test harness; built by tests/cpp/Makefile against the reference
// headers in /root/reference, run by tests/test_cpp_dropin.py on a GPU).
//
// The reference's ippo::collect_rollout and ippo::train_loop
// (marlob/ippo/rollout.hpp:41-145) are instantiated twice on the same store,
// config, seed and initial networks: once over the reference's CPU
// ippo::MarketVecEnv (rollout.hpp:151-336) and once over
// marlob::ippo::CudaMarketVecEnv (include/mlob/vec_env.hpp).  The policy, the
// sampling, GAE and the PPO update are the reference's host code in both
// runs, so every RolloutBatch field, every UpdateMetrics value, every
// network weight and the episode statistics must be bit-identical.
#include <cstdio>
#include <cstring>
#include <vector>

#include "marlob/data/synth.hpp"
#include "marlob/ippo/rollout.hpp"
#include "mlob/vec_env.hpp"

using namespace marlob;

static int g_fail = 0;

template <class T>
static void same(const char* what, const std::vector<T>& a, const std::vector<T>& b) {
  if (a.size() != b.size() || (!a.empty() && std::memcmp(a.data(), b.data(), a.size() * sizeof(T)) != 0)) {
    std::size_t i = 0;
    while (i < a.size() && i < b.size() && std::memcmp(&a[i], &b[i], sizeof(T)) == 0) ++i;
    std::printf("MISMATCH %s (size %zu vs %zu, first difference at %zu)\n", what, a.size(), b.size(), i);
    ++g_fail;
  }
}
static void same_d(const char* what, double a, double b) {
  if (std::memcmp(&a, &b, sizeof a) != 0) {
    std::printf("MISMATCH %s: %.17g vs %.17g\n", what, a, b);
    ++g_fail;
  }
}

static env::EnvConfig config() {
  env::EnvConfig c;
  env::AgentSpec mm;  // struct defaults: MarketMaker, FixedQuant, MMBasic, Spooner
  env::AgentSpec ex;
  ex.type = env::AgentType::Executor;
  ex.obs_space = agents::ObsSpaceId::Exec;
  ex.reward = env::RewardId::Exec;
  ex.params.task_size = 120;
  c.specs = {mm, ex};
  c.steps_per_episode = 8;
  c.messages_per_step = 50;
  c.start_stride_steps = 2;
  return c;
}

int main(int argc, char** argv) {
  const int n_envs = argc > 1 ? std::atoi(argv[1]) : 64;
  data::SynthConfig sc;
  sc.n_messages = 40000;
  sc.state_sample_every = 100;
  const data::MessageStore store = data::synth_generate(sc, 11);
  const env::EnvConfig cfg = config();
  const data::EpisodeIndex index =
      data::build_episode_index(store, cfg.steps_per_episode, cfg.messages_per_step, cfg.start_stride_steps);
  std::vector<std::size_t> pool;
  for (std::size_t e = 0; e < index.episode_count(); e += 3) pool.push_back(e);
  const std::uint64_t seed = 5;

  util::ThreadPool threads(4);
  ippo::MarketVecEnv cpu(&store, &index, cfg, pool, seed, n_envs, &threads);
  ippo::CudaMessageStore dstore(store, 0);
  ippo::CudaMarketVecEnv gpu(dstore, index, cfg, pool, seed, n_envs, 0);

  std::vector<ippo::PolicyNet> nets_c, nets_g;
  for (int t = 0; t < cpu.n_types(); ++t) {
    if (cpu.obs_dim(t) != gpu.obs_dim(t) || cpu.n_actions(t) != gpu.n_actions(t) ||
        cpu.n_streams(t) != gpu.n_streams(t)) {
      std::printf("MISMATCH shapes of type %d\n", t);
      return 1;
    }
    nets_c.push_back(ippo::make_policy_net(static_cast<int>(cpu.obs_dim(t)), 16, cpu.n_actions(t),
                                           make_key(seed, 0x6e657473ull, static_cast<std::uint64_t>(t))));
  }
  nets_g = nets_c;

  ippo::TrainLoopConfig lc;
  lc.updates = 3;
  lc.rollout_len = 12;  // rollouts straddle episode boundaries (8-step episodes)
  lc.seed = seed;

  // (1) collect_rollout, three consecutive rollouts with persistent hidden state
  {
    const int NT = cpu.n_types();
    std::vector<ippo::RolloutBatch> bc(NT), bg(NT);
    std::vector<std::vector<double>> hc(NT), hg(NT);
    for (int t = 0; t < NT; ++t) {
      hc[t].assign(cpu.n_streams(t) * 16, 0.0);
      hg[t].assign(gpu.n_streams(t) * 16, 0.0);
    }
    cpu.reset_all();
    gpu.reset_all();
    for (std::uint64_t u = 1; u <= 3; ++u) {
      ippo::collect_rollout(cpu, nets_c, hc, bc, lc, u);
      ippo::collect_rollout(gpu, nets_g, hg, bg, lc, u);
      for (int t = 0; t < NT; ++t) {
        same("obs", bc[t].obs, bg[t].obs);
        same("actions", bc[t].actions, bg[t].actions);
        same("log_probs", bc[t].log_probs, bg[t].log_probs);
        same("values", bc[t].values, bg[t].values);
        same("rewards", bc[t].rewards, bg[t].rewards);
        same("dones", bc[t].dones, bg[t].dones);
        same("resets", bc[t].resets, bg[t].resets);
        same("advantages", bc[t].advantages, bg[t].advantages);
        same("returns", bc[t].returns, bg[t].returns);
        same("hidden", hc[t], hg[t]);
      }
    }
    for (int t = 0; t < NT; ++t) {
      const auto a = cpu.episode_stats(t), b = gpu.episode_stats(t);
      same_d("pv_sum", a.pv_sum, b.pv_sum);
      same_d("slippage_sum", a.slippage_sum, b.slippage_sum);
      same_d("completion_sum", a.completion_sum, b.completion_sum);
      same_d("inventory_sq_sum", a.inventory_sq_sum, b.inventory_sq_sum);
      if (a.episodes != b.episodes || a.episodes == 0) {
        std::printf("MISMATCH episodes %lld vs %lld\n", (long long)a.episodes, (long long)b.episodes);
        ++g_fail;
      }
    }
    cpu.clear_episode_stats();
    gpu.clear_episode_stats();
  }

  // (2) train_loop: collect + ppo_update per type, three updates
  {
    std::vector<ippo::AdamState> ac(nets_c.size()), ag(nets_g.size());
    std::vector<ippo::UpdateMetrics> mc, mg;
    ippo::train_loop(cpu, nets_c, ac, lc, [&](int, std::span<const ippo::UpdateMetrics> m) {
      mc.insert(mc.end(), m.begin(), m.end());
    });
    ippo::train_loop(gpu, nets_g, ag, lc, [&](int, std::span<const ippo::UpdateMetrics> m) {
      mg.insert(mg.end(), m.begin(), m.end());
    });
    same("update metrics", mc, mg);
    for (std::size_t t = 0; t < nets_c.size(); ++t) {
      same("w_ih", nets_c[t].w_ih, nets_g[t].w_ih);
      same("w_hh", nets_c[t].w_hh, nets_g[t].w_hh);
      same("w_actor", nets_c[t].w_actor, nets_g[t].w_actor);
      same("w_critic", nets_c[t].w_critic, nets_g[t].w_critic);
      same_d("b_critic", nets_c[t].b_critic, nets_g[t].b_critic);
    }
  }
  if (g_fail) {
    std::printf("FAIL: %d mismatches\n", g_fail);
    return 1;
  }
  std::printf("OK: collect_rollout x3 + train_loop x3 over CudaMarketVecEnv == MarketVecEnv (%d envs)\n", n_envs);
  return 0;
}
