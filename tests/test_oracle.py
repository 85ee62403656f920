"""Pins the CPU oracle against outputs frozen from the unmodified reference
(tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

from oracle import ckks_oracle as O


def h(arr) -> str:
    a = np.ascontiguousarray(np.asarray(arr, dtype=np.uint64))
    return hashlib.sha256(a.astype("<u8").tobytes()).hexdigest()


@pytest.fixture(scope="module")
def small(golden_small):
    P = O.OParams.build(256, 50, 40, 4, 50, 2)
    assert P.qs == golden_small["q"].tolist() and P.ps == golden_small["p"].tolist()
    K = O.keygen(P, np.random.default_rng(3), rotations=[1, 2, 4])
    return P, K


def test_psi_and_ntt(small, golden_small):
    P, _ = small
    assert [O.twiddles(q, P.n)[3] for q in P.ext] == golden_small["psi"].tolist()
    out = O.ntt(golden_small["ntt_in"], P.ext)
    assert np.array_equal(out, golden_small["ntt_out"])
    assert np.array_equal(O.intt(out, P.ext), golden_small["ntt_in"])


def test_base_convert_and_automorphism(small, golden_small):
    P, _ = small
    got = O.base_convert(golden_small["ntt_in"][:3], P.qs[:3], P.ps + P.qs[3:4])
    assert np.array_equal(got, golden_small["bc_out"])
    assert np.array_equal(O.automorphism(golden_small["ntt_in"], 5, P.ext), golden_small["auto5"])


def test_keys(small, golden_small):
    _, K = small
    assert np.array_equal(K.sk, golden_small["sk"])
    assert np.array_equal(K.pk_b, golden_small["pk_b"])
    assert np.array_equal(K.rlk[0], golden_small["rlk_b"])
    assert np.array_equal(K.rlk[1], golden_small["rlk_a"])
    for s in (1, 2, 4):
        assert np.array_equal(K.gks[s][0], golden_small[f"gk{s}_b"])


def test_scheme_ops(small, golden_small):
    P, K = small
    pt, sc = O.encode(golden_small["v1"], P, P.L)
    assert np.array_equal(pt, golden_small["pt1"])
    ct1, _ = O.encrypt(pt, sc, K, np.random.default_rng(77))
    pt2, _ = O.encode(golden_small["v2"], P, P.L)
    ct2, _ = O.encrypt(pt2, sc, K, np.random.default_rng(78))
    assert np.array_equal(ct1, golden_small["ct1"])
    hm = O.hmult(ct1, ct2, K)
    assert np.array_equal(hm, golden_small["hmult"])
    rs = O.rescale(hm, P)
    assert np.array_equal(rs, golden_small["rescale"])
    dec = O.decode(O.decrypt(rs, K), sc * sc / P.qs[P.L], P)
    np.testing.assert_array_equal(dec, golden_small["dec_hmult"])
    for k in (1, 3, -1, 4):
        assert np.array_equal(O.rotate(ct1, k, K), golden_small[f"rot{k}"])
    assert np.array_equal(O.pmult(ct1, pt, P.qs), golden_small["pmult"])


def test_desk_a_hashes(golden_hashes):
    g = golden_hashes["deskA"]
    P = O.OParams.build(1 << 13, 59, 40, 10, 59, 2)
    assert P.qs == g["params"]["q"] and P.ps == g["params"]["p"]
    K = O.keygen(P, np.random.default_rng(g["key_seed"]), rotations=[1, 4])
    assert h(K.sk) == g["sk"]
    assert h(np.stack([K.rlk[0], K.rlk[1]])) == g["rlk"]
    # gks[1] is generated first in both (rotation order 1, 2, 4, ...)
    assert h(np.stack([K.gks[1][0], K.gks[1][1]])) == g["gks"]["1"]
    vrng = np.random.default_rng(12345)
    v1 = vrng.uniform(-1, 1, P.slots)
    v2 = vrng.uniform(-1, 1, P.slots)
    pt, sc = O.encode(v1, P, P.L)
    assert h(pt) == g["pt1"]
    coeff_rng = np.random.default_rng(0)
    coeff = np.stack([coeff_rng.integers(0, q, size=P.n, dtype=np.uint64) for q in P.ext])
    assert h(O.ntt(coeff, P.ext)) == g["ntt_out_seed0"]


def test_cpu_bench_sampler_and_extrapolation():
    """bench.py's CPU-baseline leg: the pinned single-threaded sampler runs
    the reference's five primitives per level (oracle/cpu_bench.py) and the
    extrapolation multiplies a per-layer tally by level-interpolated times."""
    from oracle import cpu_bench
    from oracle import ckks_oracle as O
    P = O.OParams.build(256, 50, 40, 5, 50, 2)
    spec = {"n": P.n, "qs": P.qs, "ps": P.ps, "delta": P.delta, "levels": [1, 5], "reps": 1}
    out = cpu_bench.launch(spec, sorted(__import__("os").sched_getaffinity(0))[:1])[0]
    assert out["threads"] == 1 and set(out["levels"]) == {"1", "5"}
    for lv in out["levels"].values():
        assert all(lv[op] > 0 for op in cpu_bench.OPS)
    fake = {"1": {op: 1.0 for op in cpu_bench.OPS}, "5": {op: 3.0 for op in cpu_bench.OPS}}
    rows = [{"entry_level": 3, "tally": {"rotations": 2, "hadds": 1}},
            {"entry_level": 5, "tally": {"pmults": 4}}, {"entry_level": 0, "tally": {"rescales": 1}}]
    x = cpu_bench.extrapolate(fake, rows)
    # level 3 -> 2.0 s per op; level 5 -> 3.0; level 0 -> 0.5 (linear below the lowest sample)
    assert x["s_per_image"] == 2 * 2.0 + 1 * 2.0 + 4 * 3.0 + 0.5
