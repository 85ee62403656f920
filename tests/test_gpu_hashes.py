"""Bit-exact parity at the BASELINE configs: desk-A (config 1) and N=2^16
with 25 q-limbs and 4 specials (config 2).  The reference's residues are
frozen as sha256 digests (tests/golden/make_golden.py scheme_hashes); the
engine regenerates keys/ciphertexts from the same seeds and must hash
identically."""

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def h(arr) -> str:
    a = np.ascontiguousarray(np.asarray(arr, dtype=np.uint64))
    return hashlib.sha256(a.astype("<u8").tobytes()).hexdigest()


def _ct(ct):
    return np.stack(ct.host_residues())


def _run(params, gold):
    from paper_2310_16530_b200 import ckks, ring
    from paper_2310_16530_b200.engine import to_host_u64

    assert [m.q for m in params.q_mods] == gold["params"]["q"]
    assert [m.q for m in params.p_mods] == gold["params"]["p"]
    ks = ckks.keygen(params, np.random.default_rng(gold["key_seed"]), rotations=gold["rotations"])
    assert h(ks.sk.coeffs) == gold["sk"]
    assert h(np.stack([ks.pk[0].coeffs, ks.pk[1].coeffs])) == gold["pk"]
    assert h(np.stack([to_host_u64(ks.rlk.rows_b), to_host_u64(ks.rlk.rows_a)])) == gold["rlk"]
    for s, want in gold["gks"].items():
        k = ks.gks[int(s)]
        assert h(np.stack([to_host_u64(k.rows_b), to_host_u64(k.rows_a)])) == want, f"gk {s}"
    vrng = np.random.default_rng(12345)
    v1 = vrng.uniform(-1, 1, params.slots)
    v2 = vrng.uniform(-1, 1, params.slots)
    L = params.max_level
    pt1 = ckks.encode(v1, params, L)
    assert h(pt1.poly.coeffs) == gold["pt1"]
    ct1 = ckks.encrypt(pt1, ks, np.random.default_rng(77))
    ct2 = ckks.encrypt(ckks.encode(v2, params, L), ks, np.random.default_rng(78))
    assert h(_ct(ct1)) == gold["ct1"]
    assert h(_ct(ct2)) == gold["ct2"]
    coeff_rng = np.random.default_rng(0)
    ext = params.q_mods + params.p_mods
    coeff = np.stack([coeff_rng.integers(0, m.q, size=params.n, dtype=np.uint64) for m in ext])
    assert h(coeff) == gold["ntt_in_seed0"]
    f = ring.ntt_forward(ring.RnsPoly(ext, coeff, ring.Domain.COEFF, params.ctx))
    assert h(f.coeffs) == gold["ntt_out_seed0"]
    assert np.array_equal(ring.ntt_inverse(f).coeffs, coeff)
    hm = ckks.hmult(ct1, ct2, ks)
    assert h(_ct(hm)) == gold["hmult"]
    rs = ckks.rescale(hm, params)
    assert h(_ct(rs)) == gold["rescale"]
    dec = ckks.decode(ckks.decrypt(rs, ks), params)
    assert [float(x) for x in dec[:8]] == gold["dec_hmult_head"]
    for k, want in gold["rot"].items():
        assert h(_ct(ckks.rotate(ct1, int(k), ks))) == want, f"rotate {k}"


def test_desk_a_bit_exact(golden_hashes):
    from paper_2310_16530_b200 import ckks
    _run(ckks.desk_a(), golden_hashes["deskA"])


def test_bench16_bit_exact(golden_hashes):
    from paper_2310_16530_b200 import ckks
    _run(ckks.bench16(), golden_hashes["bench16"])
