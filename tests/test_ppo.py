"""On-GPU PPO, ported from pkg/tests/test_ppo.py.  GAE, schedules, the update math and
checkpoints run on CPU tensors; the training loop and evaluation run on the GPU env."""

import numpy as np
import pytest
import torch

from conftest import build_slab_scene
from paper_2503_18616_b200.errors import CheckpointError, ValidationError
from paper_2503_18616_b200.ppo import (
    ActorCritic, PPOConfig, TrainStats, compute_gae, evaluate, linear_schedule, load_checkpoint, ppo_update,
    save_checkpoint, train,
)


class TestSchedule:
    def test_values(self):
        assert linear_schedule(2.5e-4, 0, 500_000) == 2.5e-4
        assert linear_schedule(2.5e-4, 500_000, 500_000) == 0.0
        assert linear_schedule(2.5e-4, 250_000, 500_000) == pytest.approx(1.25e-4)

    def test_out_of_range(self):
        with pytest.raises(ValidationError):
            linear_schedule(1.0, -1, 10)
        with pytest.raises(ValidationError):
            linear_schedule(1.0, 11, 10)


def mc_return_oracle(rewards, gamma):
    out = np.zeros(len(rewards))
    acc = 0.0
    for t in range(len(rewards) - 1, -1, -1):
        acc = rewards[t] + gamma * acc
        out[t] = acc
    return out


class TestGAE:
    def test_single_terminal_step(self):
        adv, ret = compute_gae([1.0], [0.0], [0.0], [True], 0.995, 0.95)
        assert adv[0] == pytest.approx(1.0) and ret[0] == pytest.approx(1.0)

    def test_two_step_hand_recursion(self):
        adv, ret = compute_gae([0.0, 1.0], [0.5, 0.5], [0.0], [False, True], 0.995, 0.95)
        assert adv[1] == pytest.approx(0.5, abs=1e-12)
        assert adv[0] == pytest.approx(0.470125, abs=1e-12)
        assert ret[0] == pytest.approx(0.970125, abs=1e-12)

    def test_lambda_zero_is_td_error(self):
        rng = np.random.default_rng(16)
        r, v = rng.normal(size=12), rng.normal(size=12)
        adv, _ = compute_gae(r, v, np.array([0.3]), np.zeros(12, bool), 0.9, 0.0)
        assert np.allclose(adv, r + 0.9 * np.append(v[1:], 0.3) - v, atol=1e-12)

    def test_lambda_one_equals_monte_carlo(self):
        rng = np.random.default_rng(17)
        for _ in range(20):
            n = int(rng.integers(2, 30))
            r, v = rng.normal(size=n), rng.normal(size=n)
            term = np.zeros(n, bool)
            term[-1] = True
            gamma = rng.uniform(0.9, 1.0)
            adv, ret = compute_gae(r, v, [0.0], term, gamma, 1.0)
            oracle = mc_return_oracle(r, gamma)
            assert np.abs(adv - (oracle - v)).max() < 1e-10 and np.abs(ret - oracle).max() < 1e-10

    def test_truncation_bootstraps_with_terminal_value(self):
        adv, _ = compute_gae(np.array([1.0, 1.0]), np.zeros(2), [9.9], np.array([False, False]), 1.0, 1.0,
                             truncated=np.array([False, True]), truncation_values=np.array([0.0, 5.0]))
        assert adv[1] == pytest.approx(6.0) and adv[0] == pytest.approx(1.0 + adv[1])

    def test_batched_matches_per_env(self):
        rng = np.random.default_rng(18)
        r, v = rng.normal(size=(16, 3)), rng.normal(size=(16, 3))
        term = rng.random((16, 3)) < 0.15
        boot = rng.normal(size=3)
        adv, ret = compute_gae(r, v, boot, term, 0.99, 0.9)
        for i in range(3):
            a1, r1 = compute_gae(r[:, i], v[:, i], [boot[i]], term[:, i], 0.99, 0.9)
            assert np.allclose(adv[:, i], a1, atol=1e-14) and np.allclose(ret[:, i], r1, atol=1e-14)


def tiny_batch(model, n=64, ratio=1.0, advantage=1.0, seed=0):
    g = torch.Generator().manual_seed(seed)
    obs = torch.randn(n, model.obs_dim, generator=g)
    actions = torch.randn(n, model.act_dim, generator=g)
    with torch.no_grad():
        log_probs, _, values = model.evaluate_actions(obs, actions)
    return (obs, actions, log_probs - float(np.log(ratio)), values.detach(), torch.full((n,), float(advantage)),
            values.detach() + advantage)


class TestPPOUpdate:
    def make(self):
        cfg = PPOConfig(steps_before_update=64, minibatch_size=64, epochs=1, normalize_advantages=False)
        torch.manual_seed(0)
        model = ActorCritic(6, 3)
        return cfg, model, torch.optim.Adam(model.parameters(), lr=cfg.learning_rate)

    def test_unit_ratio_surrogate_is_mean_advantage(self):
        cfg, model, opt = self.make()
        st = ppo_update(model, opt, tiny_batch(model, advantage=2.0), 0.1, 1e-9, cfg, torch.Generator().manual_seed(0))
        assert st["policy_loss"] == pytest.approx(-2.0, abs=1e-5)

    def test_clip_engages_above_ratio(self):
        cfg, model, opt = self.make()
        st = ppo_update(model, opt, tiny_batch(model, ratio=1.3), 0.1, 1e-9, cfg, torch.Generator().manual_seed(0))
        assert st["policy_loss"] == pytest.approx(-1.1, abs=1e-4)

    def test_post_clip_gradient_norm(self):
        cfg, model, opt = self.make()
        ppo_update(model, opt, tiny_batch(model, advantage=50.0), 0.1, 1e-3, cfg, torch.Generator().manual_seed(0))
        total = sum(float((p.grad ** 2).sum()) for p in model.parameters() if p.grad is not None)
        assert np.sqrt(total) <= cfg.max_grad_norm * (1.0 + 1e-6)

    def test_nonfinite_loss_aborts(self):
        cfg, model, opt = self.make()
        batch = list(tiny_batch(model))
        batch[4] = torch.full_like(batch[4], np.inf)
        batch[5] = batch[3] + batch[4]
        with pytest.raises(RuntimeError, match="non-finite"):
            ppo_update(model, opt, tuple(batch), 0.1, 1e-3, cfg, torch.Generator().manual_seed(0))


class TestConfig:
    def test_reference_defaults(self):
        cfg = PPOConfig()
        assert (cfg.total_steps, cfg.steps_before_update, cfg.minibatch_size, cfg.epochs) == (500_000, 1024, 256, 4)
        assert (cfg.gamma, cfg.gae_lambda, cfg.clip_range, cfg.value_clip) == (0.995, 0.95, 0.1, 0.2)
        assert (cfg.value_coef, cfg.entropy_coef, cfg.max_grad_norm, cfg.learning_rate) == (0.5, 0.0, 0.5, 2.5e-4)

    def test_large_batch_config_valid(self):
        cfg = PPOConfig.for_num_envs(4096).validate()
        assert cfg.steps_before_update % 4096 == 0 and cfg.steps_before_update // 4096 == 16

    def test_validation(self):
        with pytest.raises(ValidationError):
            PPOConfig(steps_before_update=1000, minibatch_size=256).validate()


class TestCheckpoint:
    def test_round_trip(self, tmp_path):
        torch.manual_seed(1)
        model = ActorCritic(6, 3)
        save_checkpoint(str(tmp_path / "p.pt"), model, PPOConfig())
        loaded, payload = load_checkpoint(str(tmp_path / "p.pt"), expect_obs_dim=6, expect_act_dim=3)
        obs = torch.randn(4, 6)
        assert torch.equal(model.act_greedy(obs), loaded.act_greedy(obs)) and payload["config"]["gamma"] == 0.995

    def test_dim_mismatch_named(self, tmp_path):
        save_checkpoint(str(tmp_path / "p.pt"), ActorCritic(4, 2))
        with pytest.raises(CheckpointError, match="expected 6.*has 4"):
            load_checkpoint(str(tmp_path / "p.pt"), expect_obs_dim=6)

    def test_missing(self):
        with pytest.raises(CheckpointError):
            load_checkpoint("nope.pt")

    def test_stats_csv_round_trip(self, tmp_path):
        s = TrainStats(horizon=4, num_envs=2)
        s.add_row(update=1, env_steps=8, mean_ep_reward=float("nan"), mean_ep_len=3.0, episodes=0, policy_loss=0.1,
                  value_loss=0.2, entropy=0.3, grad_norm=0.4, lr=1e-3, clip_range=0.1, sps=10.0)
        s.to_csv(str(tmp_path / "l.csv"))
        t = TrainStats.from_csv(str(tmp_path / "l.csv"))
        assert t.horizon == 4 and t.num_envs == 2 and t.rows[0]["env_steps"] == 8 and np.isnan(t.rows[0]["mean_ep_reward"])


def short_cfg(**kw):
    base = dict(total_steps=1024, steps_before_update=256, minibatch_size=64, epochs=2, seed=0)
    base.update(kw)
    return PPOConfig(**base)


@pytest.mark.gpu
class TestTrainGPU:
    def env(self, n=2, **over):
        from paper_2503_18616_b200 import EnvBatch
        mesh, rest, cfg = build_slab_scene()
        for k, v in over.items():
            setattr(cfg, k, v)
        return EnvBatch((mesh, rest, cfg), num_envs=n, seed=0, device="cuda:0")

    def test_horizon_split_and_schedules(self, tmp_path):
        stats = train(self.env(), short_cfg(), out_dir=str(tmp_path))
        assert stats.horizon == 128 and stats.rows[-1]["env_steps"] == 1024
        lrs = [r["lr"] for r in stats.rows]
        assert lrs[0] == pytest.approx(2.5e-4) and all(b <= a for a, b in zip(lrs, lrs[1:]))
        assert (tmp_path / "train_log.csv").exists() and (tmp_path / "policy.pt").exists()
        assert next(stats.model.parameters()).is_cuda

    def test_uneven_split_rejected(self):
        with pytest.raises(ValidationError):
            train(self.env(3), short_cfg())

    def test_deterministic_training(self):
        def run():
            stats = train(self.env(), short_cfg(total_steps=2048))
            return stats, {k: v.clone() for k, v in stats.model.state_dict().items()}
        sa, pa = run()
        sb, pb = run()
        assert all(torch.equal(pa[k], pb[k]) for k in pa)
        for ra, rb in zip(sa.rows, sb.rows):
            for col in TrainStats.columns:
                if col != "sps":
                    assert ra[col] == rb[col] or (np.isnan(ra[col]) and np.isnan(rb[col]))

    def test_evaluate_counts_episodes(self):
        env = self.env(max_episode_steps=5)
        torch.manual_seed(0)
        res = evaluate(env, ActorCritic(6, 3).to("cuda:0"), episodes=6, seed=0)
        assert 0.0 <= res["success_rate"] <= 1.0 and res["mean_length"] <= 5.0
        with pytest.raises(ValidationError):
            evaluate(env, ActorCritic(6, 3).to("cuda:0"), episodes=0)


@pytest.mark.gpu
def test_p8_reach_task_convergence_on_gpu():
    """Acceptance P8 (`/root/reference/pkg/tests/test_acceptance.py:186-200`) at the config-4 size:
    on-GPU PPO on 4096 reach_1170 envs crosses a trailing mean episode reward of 80 (the reference's
    stop rule: trailing-`stop_window`-episode mean held for `stop_patience` updates,
    ppo.py:405-413) within 120 updates (~2 M env steps, a few seconds on one B200), and the greedy
    policy then succeeds on >= 90% of 200 episodes, the reference's P8 bar."""
    from paper_2503_18616_b200 import EnvBatch
    from paper_2503_18616_b200.mesh import default_scene_path, load_scene
    env = EnvBatch(load_scene(default_scene_path()), num_envs=4096, seed=0, device="cuda:0")
    cfg = PPOConfig.for_num_envs(4096, stop_at_reward=80.0, stop_window=100, seed=0)
    cfg.total_steps = 120 * cfg.steps_before_update
    stats = train(env, cfg)
    assert stats.reward_crossed_at is not None, stats.rows[-3:]
    assert stats.reward_crossed_at <= 120 * cfg.steps_before_update
    res = evaluate(env, stats.model, episodes=200, seed=1)
    assert res["success_rate"] >= 0.90, res
    print(f"\nPASS P8 (GPU): reward > 80 at {stats.reward_crossed_at} env steps "
          f"({stats.reward_crossed_wall:.1f} s); greedy success {res['success_rate']:.2f}")
