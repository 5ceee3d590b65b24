"""Bit-exact replay parity of the B200 engine against reference goldens.

Length-trace replay mode (north star): scheduling, abort and recycle
decisions and buffer contents must be bit-exact.  Each step's canonical
record (tests/canon.py) from the GPU run is compared field for field with
the record the reference produced on the same configuration.
"""

import numpy as np
import pytest

import canon
import goldens
from product_runs import product_replay, product_toy

pytestmark = pytest.mark.gpu

SMALL = ["C1", "E_samples", "E_const", "E_pool", "E_cap", "C3"]


def _strip(r):
    return {k: v for k, v in r.items() if k != "rollout_wall_time"}


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("mode", ["april", "baseline"])
def test_fused_replay_matches_reference(name, mode):
    g = goldens.replay(name, mode)
    if g is None:
        pytest.skip("no golden for this mode")
    recs, _ = product_replay(canon.CONFIGS[name], mode, len(g["records"]))
    for mine, ref in zip(recs, g["records"]):
        ref = _strip(ref)
        assert mine == ref, canon.first_diff(mine, ref)


@pytest.mark.parametrize("name", ["C1", "E_samples", "E_pool"])
def test_event_path_replay_matches_reference(name):
    """The build's Scheduler in per-event mode (`_fused=False`: the reference's loop shape, one
    decode_until_event per finish, scheduler.py:272-283) over the GPU engine.  The reference's OWN
    Scheduler driving the GPU engine is tests/test_reference_drives_gpu.py."""
    g = goldens.replay(name, "april")
    recs, _ = product_replay(canon.CONFIGS[name], "april", len(g["records"]), fused=False)
    for mine, ref in zip(recs, g["records"]):
        ref = _strip(ref)
        assert mine == ref, canon.first_diff(mine, ref)


@pytest.mark.parametrize("name", ["C2", "C4_1.5", "C4_3", "C5"])
def test_fused_replay_large_configs_digests(name):
    dg = goldens.digests()[f"{name}/april"]
    recs, _ = product_replay(canon.CONFIGS[name], "april", len(dg))
    assert [canon.digest(r) for r in recs] == dg


@pytest.mark.parametrize("mode", ["april", "baseline"])
def test_toy_policy_tokens_match_reference(mode):
    """Context-free policy on the GPU: Philox draws, inverse CDF, STOP/max-len."""
    g = goldens.load(f"toy_{mode}.json.gz")["records"]
    recs = product_toy(mode, g, len(g))
    for k, (mine, ref) in enumerate(zip(recs, g)):
        ref = _strip(ref)
        # behaviour logprobs: CUDA vs glibc log/exp differ at most in the last ulps
        for a, b in zip(mine["samples"], ref["samples"]):
            np.testing.assert_allclose(a[6], b[6], rtol=1e-13, atol=1e-15)
            a[6] = b[6]
        np.testing.assert_allclose(mine["advantages"], ref["advantages"], rtol=0, atol=1e-14)
        mine["advantages"] = ref["advantages"]
        assert mine == ref, f"step {k}: " + str(canon.first_diff(mine, ref))
