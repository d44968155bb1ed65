"""CPU checks of bench.py's host-side logic: the reference arm must not load
this repo's package (its process mapped our libraries), both arms
derive one `config`, and the uplink-relay planner pairs ranks sensibly on the
box classes seen on the GPU pool (profiles/r02_bench_n4_*)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_reference_arm_helpers_do_not_import_the_package():
    code = ("import sys; sys.path.insert(0, %r); import bench; bench.bench_config(1, 32); "
            "bench.load_workloads().llama_layer_sample(layers=2); "
            "print([m for m in sys.modules if m.startswith('paper_2406_10707_b200')])" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True).stdout
    assert out.strip() == "[]"


def test_both_arms_share_one_config():
    a = bench.bench_config(4, bench.headline_layers(32, 4))
    b = bench.bench_config(4, bench.headline_layers(32, 4))
    assert json.dumps(a, sort_keys=True) == json.dumps(b, sort_keys=True)
    assert a["tensors"] == 36 * bench.headline_layers(32, 4) + 3 * 4  # 9 tensors x 4 states per layer + 3 others
    assert 1 <= bench.sample_layers(20, 5) <= 4


def test_relay_plan_shared_uplink_pair():
    # ranks 0-1 share an uplink (r02_bench_n4_shared_uplink_relay.json)
    plan = bench.relay_plan([27.1, 27.1, 44.5, 44.7], "auto")
    owners = {o for o, _, _ in plan["pairs"]}
    helpers = {h for _, h, _ in plan["pairs"]}
    assert owners == {0, 1} and helpers == {2, 3}
    for o, h, x in plan["pairs"]:
        assert 0.15 < x < 0.3
        # equal finishing times under the model, before damping
        assert abs((1 - x / 0.9) / 27.1 - (1 + x / 0.9) / 44.6) < 0.002


def test_relay_plan_three_owners_one_helper():
    plan = bench.relay_plan([21.9, 21.9, 21.9, 46.2], "auto")
    assert sorted(o for o, _, _ in plan["pairs"]) == [0, 1, 2]
    assert {h for _, h, _ in plan["pairs"]} == {3}


def test_relay_plan_symmetric_and_off():
    assert bench.relay_plan([18.4] * 4, "auto")["pairs"] == []
    assert bench.relay_plan([27.0, 44.0], "off")["pairs"] == []
    assert bench.relay_plan([57.0] * 4, "force")["pairs"] == [(0, 1, 0.3), (2, 3, 0.3)]


def test_refine_moves_toward_equal_times():
    plan = {"mode": "auto", "rates_gbps": [46, 46, 46, 33.9], "pairs": [(3, 0, 0.14)]}
    # the owner (rank 3) still finishes last: its share must grow
    refined = bench.refine_relay(plan, [2.2, 2.0, 2.0, 2.55])
    assert refined["pairs"][0][2] > 0.14
    # the helper finishes last: the share must shrink
    refined = bench.refine_relay(plan, [2.8, 2.0, 2.0, 2.3])
    assert refined["pairs"][0][2] < 0.14


def test_tune_relay_never_keeps_a_slower_plan():
    """If every relayed plan measures slower than no relay, the relay goes off."""
    armed = []
    plan = bench.relay_plan([27.0, 27.0, 44.0, 44.0], "auto")
    base = [1 / 27.0, 1 / 27.0, 1 / 44.0, 1 / 44.0]
    res = bench.tune_relay(plan, base, measure=lambda: [0.1, 0.1, 0.1, 0.1], arm=armed.append)
    assert res["pairs"] == [] and armed[-1]["pairs"] == []
    # and keeps a plan that beats it
    res = bench.tune_relay(plan, base, measure=lambda: [0.03, 0.03, 0.03, 0.03], arm=armed.append)
    assert res["pairs"] and armed[-1]["pairs"] == res["pairs"]


def test_relay_plan_eight_ranks_two_uplink_classes():
    """N=8 node where ranks 0-3 share uplinks in pairs and 4-7 have their own:
    every owner gets exactly one helper, helpers are never owners, and every
    share is within the cap."""
    rates = [27.0, 27.2, 26.9, 27.1, 56.0, 55.5, 56.2, 55.8]
    plan = bench.relay_plan(rates, "auto")
    owners = [o for o, _, _ in plan["pairs"]]
    helpers = {h for _, h, _ in plan["pairs"]}
    assert sorted(owners) == [0, 1, 2, 3] and helpers == {4, 5, 6, 7}
    assert not helpers & set(owners)
    assert all(0 < x <= 0.45 for _, _, x in plan["pairs"])
    assert bench.relay_plan(rates, "force")["pairs"] == [(0, 1, 0.3), (2, 3, 0.3), (4, 5, 0.3), (6, 7, 0.3)]


def test_configs2_skips_when_host_ram_is_short(monkeypatch):
    monkeypatch.setattr(bench, "fits_host", lambda b, w: False)

    class W:
        @staticmethod
        def llama13b_shard(dp, rank):
            class S:
                total_bytes = 30 << 30
            return S()
    out = bench.run_configs2(None, None, W, 0, "/tmp", 0, 8, lambda: None, max, sum, lambda x: [x] * 8, None)
    assert "skipped" in out


def test_tune_relay_survives_a_failing_relay():
    """A plan whose steps fail (measured as inf) is never kept, and refining
    from it does not divide by zero."""
    plan = bench.relay_plan([27.0, 27.0, 44.0, 44.0], "auto")
    base = [1 / 27.0, 1 / 27.0, 1 / 44.0, 1 / 44.0]
    armed = []
    res = bench.tune_relay(plan, base, measure=lambda: [float("inf")] * 4, arm=armed.append)
    assert res["pairs"] == [] and armed[-1]["pairs"] == []


def test_tune_relay_needs_a_margin_over_no_relay():
    """A relayed plan within 2 % of "no relay" is noise: no relay is kept."""
    plan = bench.relay_plan([57.0, 39.3], "auto")
    base = [0.537, 0.780]
    armed = []
    res = bench.tune_relay(plan, base, measure=lambda: [0.537, 0.777], arm=armed.append)
    assert res["pairs"] == [] and armed[-1]["pairs"] == []
    res = bench.tune_relay(plan, base, measure=lambda: [0.60, 0.70], arm=armed.append)
    assert res["pairs"]


def test_relay_plan_mildly_uneven_pair():
    """57.0 vs 48.9 GB/s (a 2-GPU box seen in the pool): rank 1 hands ~7 % to rank 0."""
    plan = bench.relay_plan([57.0, 48.9], "auto")
    assert [(o, h) for o, h, _ in plan["pairs"]] == [(1, 0)]
    assert 0.04 < plan["pairs"][0][2] < 0.1
    assert bench.relay_plan([57.0, 54.0], "auto")["pairs"] == []
