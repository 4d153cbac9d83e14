"""Pins the oracle: the C restatement (orc) against the reference's own
known-answer tests, the SURVEY §8c golden digests and the compiled reference
itself (ref).  CPU only."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from oracle.oracle import (OBook, OEnv, OVecEnv, bench_run, random_stream)
from paper_2511_02136_b200 import abi
from tests import kat
from tests.common import (compare_env_state, random_direct_action, scenario_configs,
                          small_store)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---- core/rng.hpp KATs ------------------------------------------

def test_rng_known_answers(orc):
    assert orc.splitmix64(0) == 0xE220A8397B1DCDAF
    w = (C.c_uint64 * 1)(1)
    assert orc.make_key(0, 1, w) == 0x253E9F2719612DB2
    d = (C.c_uint64 * 2)()
    orc.crng_draws(0x253E9F2719612DB2, 2, d)
    # SURVEY §8c lists this pair in the opposite order; the reference's own
    # CounterRng (rng.hpp:46, compiled and run here) yields fb26.. first.
    assert list(d) == [0xFB2670E9E34C2FB4, 0x223D0D1686DC2F76]
    # the pure-Python test helper agrees
    assert kat.make_key(0, 1) == 0x253E9F2719612DB2
    r = kat.CounterRng(kat.make_key(0, 1))
    assert [r.next(), r.next()] == [0xFB2670E9E34C2FB4, 0x223D0D1686DC2F76]


# ---- golden digests ------------------------------------------------------------

@pytest.mark.parametrize("name", ["exec_only", "mm_exec"])
def test_config_a_golden(orc, name):
    golden = json.load(open(os.path.join(GOLDEN, "kat_config_a.json")))[name]
    got = kat.config_a_digest("orc", name)
    assert got == golden


def test_config_a_matches_survey_digests():
    """The committed golden file equals the numbers SURVEY §8c quotes."""
    g = json.load(open(os.path.join(GOLDEN, "kat_config_a.json")))
    assert g["exec_only"]["trade_fnv"] == "2bd2e489b75a7f38"
    assert g["exec_only"]["book_fnv"] == "895762ebbef83f71"
    assert (g["exec_only"]["messages"], g["exec_only"]["trades"]) == (10027, 3269)
    assert g["exec_only"]["sum_reward"] == -1030.0
    assert g["exec_only"]["sum_obs"] == 968.13458584172008
    assert g["mm_exec"]["trade_fnv"] == "aa48d18e732bbcf8"
    assert g["mm_exec"]["book_fnv"] == "eea0275d797c136d"
    assert g["mm_exec"]["next_seq"] == 4518
    assert g["mm_exec"]["sum_reward"] == -4686.0559935155188


@pytest.mark.parametrize("name", ["exec_only", "mm_exec"])
def test_config_a_reference_matches_golden(ref, name):
    golden = json.load(open(os.path.join(GOLDEN, "kat_config_a.json")))[name]
    assert kat.config_a_digest("ref", name) == golden


# ---- test_lob.cpp KATs on the restated book -----------------------------------

def nl(side, price, qty, oid, trader=0, time=0):
    return abi.Message(time, oid, price, qty, abi.NEW_LIMIT, side, (C.c_uint8 * 2)(), trader)


def mk(kind, side, oid, qty=0):
    return abi.Message(0, oid, 0, qty, kind, side, (C.c_uint8 * 2)(), 0)


@pytest.fixture(params=["orc", "ref"])
def lib(request):
    from oracle.oracle import Oracle, available
    if request.param == "ref" and not available("ref"):
        pytest.skip("no _ref")
    return Oracle(request.param)


def test_lob_price_time_kat(lib):  # test_lob.cpp:100-129
    b = OBook(lib, 100)
    b.process(nl(abi.ASK, 1000, 5, 10))
    b.process(nl(abi.ASK, 1000, 3, 11))
    t = b.process(nl(abi.BID, 1001, 6, 12, 1))
    assert list(t["quantity"]) == [5, 1] and list(t["passive_order_id"]) == [10, 11]
    assert list(t["price"]) == [1000, 1000] and t["aggressor_trader_id"][0] == 1
    asks = b.orders(abi.ASK)
    assert asks[-1]["quantity"] == 2 and len(b.orders(abi.BID)) == 0


def test_lob_init_and_noops(lib):  # test_lob.cpp:61-98, 131-164
    b = OBook(lib, 100)
    b.init_from_l2([(1000, 5), (999, 7)], [], 1000)
    o = b.orders(abi.BID)
    assert o[-1]["price"] == 1000 and o[-1]["arrival_seq"] < o[0]["arrival_seq"]
    with pytest.raises(ValueError):
        OBook(lib, 100).init_from_l2([(2000 - i, 1) for i in range(101)], [], 0)
    b = OBook(lib, 100)
    b.process(nl(abi.ASK, 1005, 10, 7))
    before = b.orders(abi.ASK).tobytes()
    assert len(b.process(mk(abi.DELETE, abi.BID, 42))) == 0
    b.process(mk(abi.EXECUTE_HIDDEN, abi.ASK, 7, 3))
    b.process(mk(abi.CROSS, abi.BID, 0, 1))
    assert b.orders(abi.ASK).tobytes() == before
    assert len(b.process(mk(abi.EXECUTE_VISIBLE, abi.ASK, 7, 3))) == 0
    assert b.orders(abi.ASK)[-1]["quantity"] == 7
    b.process(mk(abi.CANCEL_PARTIAL, abi.ASK, 7, 7))
    assert len(b.orders(abi.ASK)) == 0


def test_lob_mid_and_l2(lib):  # test_lob.cpp:179-213
    b = OBook(lib, 100)
    assert b.mid_half(1001) == 1001
    b.process(nl(abi.BID, 1000, 5, 1))
    b.process(nl(abi.ASK, 1002, 5, 2))
    assert b.mid_half(0) == 2002
    b.process(nl(abi.BID, 1000, 5, 3))
    bids, _ = b.l2(5)
    assert bids == [(1000, 10)]
    b.process(nl(abi.ASK, 1003, 1, 4))
    b.process(nl(abi.ASK, 1001, 2, 5))
    assert b.l2(2)[1] == [(1001, 2), (1002, 5)]


def test_lob_eviction(lib):  # test_lob.cpp:215-256
    def two():
        b = OBook(lib, 2)
        b.process(nl(abi.BID, 10, 1, 1))
        b.process(nl(abi.BID, 9, 1, 2))
        return b
    b = two()
    b.process(nl(abi.BID, 11, 1, 3))
    o = b.orders(abi.BID)
    assert len(o) == 2 and o[-1]["price"] == 11 and o[0]["price"] == 10
    b = two()
    b.process(nl(abi.BID, 9, 1, 3))
    o = b.orders(abi.BID)
    assert list(o["order_id"]) == [2, 1] and b.next_seq == 2
    t = OBook(lib, 2)
    for oid, p in ((5, 20), (6, 20), (7, 19)):
        t.process(nl(abi.ASK, p, 1, oid))
    assert list(t.orders(abi.ASK)["order_id"]) == [6, 7]
    b = OBook(lib, 4)
    for i in range(32):
        b.process(nl(abi.BID, 100 + i, 1, i, i % 3))
        assert len(b.orders(abi.BID)) <= 4
    assert b.orders(abi.BID)[-1]["price"] == 131


def test_random_streams_match_naive_book(orc, ref):  # test_lob.cpp:258-281
    for seed in range(25):
        msgs = random_stream(orc, seed, n_messages=4000)
        assert msgs.tobytes() == random_stream(ref, seed, n_messages=4000).tobytes()
        b, r = OBook(orc, 1 << 15), OBook(ref, 1 << 15)
        naive = ref.naive_create()
        tr = (abi.Trade * 4096)()
        for m in msgs:
            t1, t2 = b.process(m), r.process(m)
            mm = abi.Message.from_buffer_copy(m.tobytes())
            n = ref.naive_process(naive, C.byref(mm), tr, 4096)
            t3 = np.frombuffer(bytes(tr)[: n * 56], dtype=t1.dtype)
            assert t1.tobytes() == t2.tobytes() == t3.tobytes()
        assert b.orders(0).tobytes() == r.orders(0).tobytes()
        assert b.orders(1).tobytes() == r.orders(1).tobytes()
        lv = (abi.Level * 8192)()
        for side in (0, 1):
            n = ref.naive_l2_full(naive, side, lv, 8192)
            full = b.l2(1 << 15)[side]
            assert full == [(lv[i].price, lv[i].quantity) for i in range(n)]
        ref.naive_free(naive)


@pytest.mark.parametrize("capacity", [8, 64, 1 << 15])
def test_duplicate_live_ids_match_reference(orc, ref, capacity):
    """Resting orders sharing ids: reduce / remove take the first match in the
    reference's storage order (book.hpp:191-206); with evictions at small
    capacities.  C restatement vs the compiled reference, message by message."""
    from oracle.oracle import dup_id_stream
    for seed in range(6):
        msgs = dup_id_stream(orc, seed, n_messages=3000)
        b, r = OBook(orc, capacity), OBook(ref, capacity)
        for m in msgs:
            assert b.process(m).tobytes() == r.process(m).tobytes()
        assert b.orders(0).tobytes() == r.orders(0).tobytes()
        assert b.orders(1).tobytes() == r.orders(1).tobytes()


# ---- synthetic store -----------------------------------------------------------

@pytest.mark.parametrize("kw,seed", [({}, 0), ({"state_sample_every": 100}, 11),
                                     ({"initial_mid": 100000, "band": 2000,
                                       "p_new_passive": 0.46, "p_new_cross": 0.04,
                                       "p_cancel": 0.30, "p_delete": 0.16, "p_execute": 0.02,
                                       "state_depth": 1000, "state_sample_every": 6400}, 0),
                                     ({"volatility": 0.0, "initial_mid": 500}, 3)])
def test_synth_matches_reference(orc, ref, kw, seed):
    cfg = abi.synth_config(n_messages=20000, **kw)
    a, b = orc.synth(cfg, seed), ref.synth(cfg, seed)
    assert a.messages().tobytes() == b.messages().tobytes()
    assert a.states() == b.states()


def test_synth_errors(orc):
    with pytest.raises(ValueError):
        orc.synth(abi.synth_config(n_messages=0), 0)
    with pytest.raises(ValueError):
        orc.synth(abi.synth_config(initial_mid=9), 0)


# ---- environment differential: orc vs ref on every output, every step ----------

@pytest.mark.parametrize("scenario", list(scenario_configs().keys()))
def test_env_differential(orc, ref, scenario):
    cfg, synth_kw, n_steps = scenario_configs()[scenario]
    so, sr = small_store(orc, synth_kw), small_store(ref, synth_kw)
    rng = kat.CounterRng(kat.make_key(99, len(scenario)))
    for env_index in (0, 3):
        eo, er = OEnv(orc, so, cfg, 5, env_index), OEnv(ref, sr, cfg, 5, env_index)
        n_ep = eo.n_episodes
        assert n_ep == er.n_episodes
        for ep in range(min(2, n_ep)):
            eo.reset(ep)
            er.reset(ep)
            compare_env_state(eo, er, ref_side=True)
            for t in range(n_steps):
                if rng.below(4) == 0:
                    acts = [random_direct_action(rng) for _ in range(eo.n_agents)]
                    eo.step(acts)
                    er.step(acts)
                else:
                    ids = [rng.below(abi.action_arity(cfg.specs[s])) for s in eo.flat]
                    eo.step_ids(ids)
                    er.step_ids(ids)
                compare_env_state(eo, er, ref_side=True)


def test_env_errors(orc, ref):
    cfg = abi.env_config([abi.agent_spec(abi.MARKET_MAKER)], steps_per_episode=4,
                         messages_per_step=10, start_stride_steps=4)
    for o in (orc, ref):
        st = small_store(o, {})
        e = OEnv(o, st, cfg, 1, 0)
        with pytest.raises(RuntimeError):  # logic_error: step before reset
            e.step_ids([0])
        with pytest.raises(IndexError):
            e.reset(e.n_episodes)
        e.reset(0)
        with pytest.raises(ValueError):
            e.step_ids([0, 0])
        with pytest.raises(IndexError):
            e.step_ids([8])
        bad = abi.env_config([abi.agent_spec(abi.MARKET_MAKER, lambda_=1.5)])
        with pytest.raises(ValueError):
            OEnv(o, st, bad, 0, 0)


def test_vec_env_differential(orc, ref):
    cfg = abi.env_config([abi.agent_spec(abi.MARKET_MAKER, count=2), abi.agent_spec(abi.EXECUTOR)],
                         steps_per_episode=8, messages_per_step=20, start_stride_steps=3)
    so, sr = small_store(orc, {"state_sample_every": 20}), small_store(ref, {"state_sample_every": 20})
    vo, vr = OVecEnv(orc, so, cfg, 3, 5), OVecEnv(ref, sr, cfg, 3, 5, workers=3)
    vo.reset_all()
    vr.reset_all()
    rng = kat.CounterRng(123)
    for t in range(30):
        for ty in range(cfg.n_specs):
            oo, ro = vo.gather(ty), vr.gather(ty)
            assert oo[0].tobytes() == ro[0].tobytes() and oo[1].tobytes() == ro[1].tobytes()
            for s in range(5 * cfg.specs[ty].count):
                a = rng.below(abi.action_arity(cfg.specs[ty]))
                vo.set_action(ty, s, a)
                vr.set_action(ty, s, a)
        vo.step_all()
        vr.step_all()
        for ty in range(cfg.n_specs):
            for s in range(5 * cfg.specs[ty].count):
                assert vo.reward(ty, s) == vr.reward(ty, s)
                assert vo.done(ty, s) == vr.done(ty, s)
    for ty in range(cfg.n_specs):
        a, b = vo.episode_stats(ty), vr.episode_stats(ty)
        assert bytes(a) == bytes(b) and a.episodes == 15
    vo.clear_episode_stats()
    assert vo.episode_stats(0).episodes == 0


def test_bench_harness_counts(orc, ref):
    cfg = abi.env_config([abi.agent_spec(abi.MARKET_MAKER), abi.agent_spec(abi.EXECUTOR)],
                         steps_per_episode=16, messages_per_step=20, start_stride_steps=16)
    so, sr = small_store(orc, {"state_sample_every": 16}), small_store(ref, {"state_sample_every": 16})
    a = bench_run(orc, so, cfg, 8, 32, 2, 1, 0, 20, 1)
    b = bench_run(ref, sr, cfg, 8, 32, 2, 2, 0, 20, 1)
    assert a.env_steps == b.env_steps == 8 * 32
    assert a.messages == b.messages > 8 * 32 * 20


def test_evaluate_matrix_matches_reference(orc, ref):
    """Scripted cross-play (evaluate.hpp:104-217, twap.hpp, avst.hpp): the C
    restatement against the reference's own evaluate_matrix, bit for bit."""
    from tests.common import crossplay_case
    cfg, synth_kw, eps, t0, t1 = crossplay_case()
    a = orc.evaluate(small_store(orc, synth_kw), cfg, eps, t0, t1, 7)
    b = ref.evaluate(small_store(ref, synth_kw), cfg, eps, t0, t1, 7)
    assert len(a) == len(t0) * len(t1)
    assert [bytes(x) for x in a] == [bytes(x) for x in b]
    assert any(c.per_type[1].completion_mean > 0 for c in a)      # TWAP executes
    assert any(c.per_type[0].filled_total > 0 for c in a)         # AvSt quotes fill


def test_evaluate_matrix_errors(orc, ref):
    from tests.common import crossplay_case
    cfg, synth_kw, eps, t0, t1 = crossplay_case()
    for o in (orc, ref):
        st = small_store(o, synth_kw)
        with pytest.raises(ValueError):   # evaluate.hpp:112 (empty episodes)
            o.evaluate(st, cfg, [], t0, t1, 0)
        with pytest.raises(ValueError):   # evaluate.hpp:114-117 (learned without a net)
            o.evaluate(st, cfg, eps, [abi.policy(abi.POLICY_LEARNED)], t1, 0)
        with pytest.raises(IndexError):   # avst.hpp:21-23
            o.evaluate(st, cfg, eps, [abi.policy(abi.POLICY_AVST, gamma_index=4)], t1, 0)
        one = abi.env_config([abi.agent_spec(abi.EXECUTOR)], steps_per_episode=12,
                             messages_per_step=25, start_stride_steps=12)
        with pytest.raises(ValueError):   # evaluate.hpp:110-111 (two types)
            o.evaluate(st, one, eps, t0, t1, 0)


def test_collect_rollout_matches_reference(orc, ref):
    """make_policy_net (net.hpp:80-104) and collect_rollout (rollout.hpp:41-124:
    GRU forward, ActionSample draws, env steps with auto-reset, bootstrap, GAE)
    of the C restatement against the reference, two consecutive updates."""
    from tests.common import rollout_case
    got = {}
    for o in (orc, ref):
        cfg, synth_kw, nets = rollout_case(o)
        v = OVecEnv(o, small_store(o, synth_kw), cfg, 3, 5)
        v.reset_all()
        out = [n.flat.tobytes() for n in nets]
        for upd in (1, 2):
            v.collect_rollout(nets, 12, 0.99, 0.95, 77, upd)
            out += [v.rollout(t, f).tobytes() for t in range(2) for f in range(11)]
        got[o.kind] = out
    assert got["orc"] == got["ref"]
    with pytest.raises(ValueError):  # net.hpp:86-87
        orc.make_policy_net(8, 513, 8, 0)


def test_evaluate_matrix_learned_matches_reference(orc, ref):
    """Learned options (evaluate.hpp:80-90: policy_forward + argmax, hidden zeroed
    per episode) in the cross-play grid: C restatement vs the reference."""
    from tests.common import crossplay_learned_case
    cfg, synth_kw, eps, t0, t1 = crossplay_learned_case(orc)
    a = orc.evaluate(small_store(orc, synth_kw), cfg, eps, t0, t1, 5)
    b = ref.evaluate(small_store(ref, synth_kw), cfg, eps, t0, t1, 5)
    assert [bytes(x) for x in a] == [bytes(x) for x in b]


def _msgs(store):
    """message records with the (uninitialised in the reference) padding zeroed"""
    m = store.messages()
    m["_pad"] = b"\x00\x00"
    return m.tobytes()


def _lobster_files(tmp_path, name, msg, book):
    m, b = tmp_path / f"{name}_msg.csv", tmp_path / f"{name}_book.csv"
    m.write_text(msg)
    b.write_text(book)
    return str(m), str(b)


def test_lobster_matches_reference(orc, ref, tmp_path):
    """load_lobster (lobster.hpp:119-193): C restatement vs the reference on the
    test_data.cpp KAT, edge-case inputs and a synthetic day written like
    write_lobster; malformed inputs raise the same class and text."""
    from tests.lobster_util import ACCEPTED, MALFORMED, write_lobster
    for name, msg, book, upt, every in ACCEPTED:
        m, b = _lobster_files(tmp_path, name, msg, book)
        a, r = orc.lobster(m, b, upt, every), ref.lobster(m, b, upt, every)
        assert _msgs(a) == _msgs(r), name
        assert a.states() == r.states(), name
    kat = orc.lobster(*_lobster_files(tmp_path, "kat2", ACCEPTED[0][1], ACCEPTED[0][2]), 100, 1)
    m0 = kat.messages()[0]                    # test_data.cpp:54-82
    assert (m0["kind"], m0["side"], m0["price"], m0["quantity"], m0["order_id"], m0["time"]) == \
        (abi.NEW_LIMIT, abi.BID, 31480, 10, 42, 34200000123000)
    assert kat.states() == [(0, [], []), (1, [(31480, 10)], [(31490, 5)])]
    for name, msg, book, upt, every in MALFORMED:
        m, b = _lobster_files(tmp_path, name, msg, book)
        errs = []
        for o in (orc, ref):
            with pytest.raises(Exception) as ei:
                o.lobster(m, b, upt, every)
            errs.append((type(ei.value), str(ei.value)))
        assert errs[0] == errs[1], name
    synth = orc.synth(abi.synth_config(n_messages=3000, state_sample_every=100), 1)
    m, b = str(tmp_path / "day_msg.csv"), str(tmp_path / "day_book.csv")
    write_lobster(orc, synth.messages(), m, b, upt=100, depth=5)
    a, r = orc.lobster(m, b, 100, 100), ref.lobster(m, b, 100, 100)
    assert _msgs(a) == _msgs(r)
    assert a.states() == r.states() and len(a.states()) == 30
