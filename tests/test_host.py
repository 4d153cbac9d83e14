"""CPU tests of the product's host side: the C ABI library loads and exports
every symbol include/mlob.h declares, record layouts, defaults, config
validation, episode indexing and the host store builder (bit-identical to the
reference generator).  No compute call needs a GPU here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2511_02136_b200 import abi, env

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "mlob.h")).read()
    return sorted(set(re.findall(r"\b(mlob_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = env.lib()
    syms = declared_symbols()
    assert len(syms) > 50
    for s in syms:
        assert hasattr(L, s), s
    assert L.mlob_abi_version() == abi.ABI_VERSION


def test_defaults_match_reference_structs():
    L = env.lib()
    c = abi.EnvConfig()
    L.mlob_default_env_config(C.byref(c))
    assert bytes(c) == bytes(abi.env_config([]))
    s = abi.AgentSpec()
    L.mlob_default_agent_spec(C.byref(s))
    ref = abi.agent_spec(abi.MARKET_MAKER)
    assert bytes(s) == bytes(ref)
    sc = abi.SynthConfig()
    L.mlob_default_synth_config(C.byref(sc))
    assert bytes(sc) == bytes(abi.synth_config())


def test_arity_and_obs_size():
    L = env.lib()
    for spec, n in [(abi.agent_spec(abi.EXECUTOR), 12), (abi.agent_spec(abi.EXECUTOR, exec_complex=0), 4),
                    (abi.agent_spec(abi.DIRECTIONAL), 3), (abi.agent_spec(abi.MARKET_MAKER), 8),
                    (abi.agent_spec(abi.MARKET_MAKER, mm_space=abi.SPREAD_SKEW), 9),
                    (abi.agent_spec(abi.MARKET_MAKER, mm_space=abi.AVST), 4)]:
        assert L.mlob_action_arity(C.byref(spec)) == n == abi.action_arity(spec)
    assert L.mlob_observation_size(abi.OBS_MM_FULL, 5) == 28


def test_config_validation_mirrors_reference():
    L = env.lib()
    ok = abi.env_config([abi.agent_spec(abi.MARKET_MAKER)])
    assert L.mlob_validate_env_config(C.byref(ok)) == abi.MLOB_OK
    for kw in [dict(steps_per_episode=0), dict(messages_per_step=-1), dict(start_stride_steps=0),
               dict(book_capacity=0), dict(obs_depth=0)]:
        assert L.mlob_validate_env_config(C.byref(abi.env_config([], **kw))) == abi.MLOB_E_INVALID_ARGUMENT
    for p in [dict(lambda_=1.5), dict(rho=-1.0), dict(order_size=0), dict(inventory_cap=0)]:
        bad = abi.env_config([abi.agent_spec(abi.MARKET_MAKER, **p)])
        assert L.mlob_validate_env_config(C.byref(bad)) == abi.MLOB_E_INVALID_ARGUMENT
    bad = abi.env_config([abi.agent_spec(abi.EXECUTOR, task_size=0)])
    assert L.mlob_validate_env_config(C.byref(bad)) == abi.MLOB_E_INVALID_ARGUMENT
    assert b"task_size" in L.mlob_last_error()


def test_episode_index_arithmetic():  # test_data.cpp:115-156
    assert list(env.episode_index(12800, 64, 100, 64)) == [0, 6400]
    assert list(env.episode_index(12800, 64, 100, 32)) == [0, 3200, 6400]
    assert len(env.episode_index(6399, 64, 100, 64)) == 0
    assert list(env.episode_index(10, 4, 0, 4)) == [0]
    for stride in (1, 3, 17, 64):
        idx = env.episode_index(12800, 64, 100, stride)
        assert len(idx) and all(s + 6400 <= 12800 for s in idx)
    with pytest.raises(ValueError):
        env.episode_index(0, 64, 100, 64)


@pytest.mark.parametrize("kw,seed", [({}, 0), ({"state_sample_every": 100}, 11),
                                     ({"initial_mid": 100000, "band": 2000, "p_new_passive": 0.46,
                                       "p_new_cross": 0.04, "p_cancel": 0.30, "p_delete": 0.16,
                                       "p_execute": 0.02, "state_depth": 1000,
                                       "state_sample_every": 6400}, 0),
                                     ({"volatility": 0.0, "initial_mid": 500}, 3)])
def test_product_synth_matches_reference_generator(ref, kw, seed):
    cfg = abi.synth_config(n_messages=30000, **kw)
    mine = env.HostStore.synth(cfg, seed)
    theirs = ref.synth(cfg, seed)
    assert mine.messages().tobytes() == theirs.messages().tobytes()
    assert mine.states() == theirs.states()


def test_product_synth_matches_oracle_without_reference(orc):
    cfg = abi.synth_config(n_messages=20000, state_sample_every=500)
    assert env.HostStore.synth(cfg, 5).messages().tobytes() == orc.synth(cfg, 5).messages().tobytes()


def test_store_trim_front():
    s = env.synth_store(0, n_messages=3000, state_sample_every=100)
    msgs = s.messages()
    states = s.states()
    s.trim_front(1000)
    assert s.messages().tobytes() == msgs[1000:].tobytes()
    t = s.states()
    assert [x[0] for x in t] == [x[0] - 1000 for x in states if x[0] >= 1000]
    assert t[0][1:] == [x for x in states if x[0] == 1000][0][1:]


def test_store_roundtrip_through_host_create():
    s = env.synth_store(1, n_messages=2000, state_sample_every=200)
    r = env.HostStore.from_messages(s.messages(), s.states())
    assert r.messages().tobytes() == s.messages().tobytes()
    assert r.states() == s.states()


def test_synth_errors():
    with pytest.raises(ValueError):
        env.synth_store(0, n_messages=0)
    with pytest.raises(ValueError):
        env.synth_store(0, initial_mid=5)


def test_no_cpu_fallback_without_gpu():
    """Without a CUDA device the product fails loudly instead of stepping on
    the CPU (there is no CPU execution path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        env.DeviceStore(env.synth_store(0, n_messages=1000), 0)


def test_host_store_save_load_roundtrip(tmp_path):
    """mlob_host_store_save / _load: the binary image one rank per node writes
    for the others (bench.py host_store) carries messages and book states
    unchanged; a foreign or truncated file is a runtime_error."""
    from paper_2511_02136_b200.env import HostStore
    h = HostStore.synth(abi.synth_config(n_messages=30000, state_sample_every=100), 5)
    path = str(tmp_path / "store.bin")
    h.save(path)
    g = HostStore.load(path)
    assert g.n_messages == h.n_messages
    assert (g.messages() == h.messages()).all()
    assert g.states() == h.states()
    with open(path, "r+b") as f:
        f.truncate(1000)
    with pytest.raises(RuntimeError):
        HostStore.load(path)
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"not a store" * 10)
    with pytest.raises(RuntimeError):
        HostStore.load(str(bad))
