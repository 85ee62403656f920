"""HCNK containers (reference io.py).  The committed
containers under tests/golden were written by the unmodified reference
(make_golden.py hcnk) for the unit-small key set and ciphertexts whose
residues golden_small.npz holds."""

import io as pyio
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def params():
    from paper_2310_16530_b200 import ckks
    return ckks.CkksParams.build("unit-small", 256, 50, 40, 4, 50, 2)


def test_host_parse_reference_keyset(params, golden_small):
    """byte-level parse of the reference-written key set (no GPU)"""
    from paper_2310_16530_b200 import io as hio
    with open(GOLD / "hcnk_unit_small.keyset", "rb") as f:
        hio.read_header(f, hio.KIND_KEYSET, params)
        sk, pk_b, pk_a = (hio.read_poly(f, params) for _ in range(3))
        assert (sk.n_q, sk.n_p, sk.eval_domain) == (5, 2, True)
        assert np.array_equal(sk.coeffs, golden_small["sk"])
        assert np.array_equal(pk_b.coeffs, golden_small["pk_b"])
        assert np.array_equal(pk_a.coeffs, golden_small["pk_a"])
        n_dig = hio._u32(f)
        rows = [(hio.read_array(f), hio.read_array(f)) for _ in range(n_dig)]
        assert np.array_equal(np.stack([b for b, _ in rows]), golden_small["rlk_b"])
        assert np.array_equal(np.stack([a for _, a in rows]), golden_small["rlk_a"])
        steps = []
        for _ in range(hio._u32(f)):
            step = hio._u32(f)
            steps.append(step)
            n_dig = hio._u32(f)
            rows = [(hio.read_array(f), hio.read_array(f)) for _ in range(n_dig)]
            assert np.array_equal(np.stack([b for b, _ in rows]), golden_small[f"gk{step}_b"])
        assert steps == [1, 2, 4]
        assert f.read() == b""


def test_host_parse_reference_ciphertext(params, golden_small):
    import struct
    from paper_2310_16530_b200 import io as hio
    with open(GOLD / "hcnk_unit_small_ct1.ct", "rb") as f:
        hio.read_header(f, hio.KIND_CIPHERTEXT, params)
        struct.unpack("<d", f.read(8))
        c0, c1 = hio.read_poly(f, params), hio.read_poly(f, params)
    assert np.array_equal(np.stack([c0.coeffs, c1.coeffs]), golden_small["ct1"])


def test_header_checks(params):
    from paper_2310_16530_b200 import ckks, io as hio
    from paper_2310_16530_b200.errors import SerializationError
    raw = (GOLD / "hcnk_unit_small_ct1.ct").read_bytes()
    with pytest.raises(SerializationError, match="digest"):
        hio.read_header(pyio.BytesIO(raw), hio.KIND_CIPHERTEXT, ckks.CkksParams.build("x", 256, 50, 40, 3, 50, 2))
    with pytest.raises(SerializationError, match="expected keyset"):
        hio.read_header(pyio.BytesIO(raw), hio.KIND_KEYSET, params)
    with pytest.raises(SerializationError, match="not an HCNK"):
        hio.read_header(pyio.BytesIO(b"XXXX" + raw[4:]), hio.KIND_CIPHERTEXT, params)
    f = pyio.BytesIO(raw[:200])
    hio.read_header(f, hio.KIND_CIPHERTEXT, params)
    f.read(8)
    with pytest.raises(SerializationError, match="truncated"):
        hio.read_poly(f, params)


@pytest.mark.gpu
def test_device_round_trip_is_byte_identical(params, golden_small, tmp_path):
    """load (to HBM) and save (from HBM) reproduce the reference's bytes."""
    import torch
    from paper_2310_16530_b200 import ckks, io as hio
    ks = hio.load_keyset(str(GOLD / "hcnk_unit_small.keyset"), params)
    assert np.array_equal(ks.sk.data.cpu().numpy().view(np.uint64), golden_small["sk"])
    assert np.array_equal(ks.gks[4].rows_a.cpu().numpy().view(np.uint64), golden_small["gk4_a"])
    hio.save_keyset(str(tmp_path / "k"), ks)
    assert (tmp_path / "k").read_bytes() == (GOLD / "hcnk_unit_small.keyset").read_bytes()
    for name in ("hcnk_unit_small_ct1.ct", "hcnk_unit_small_ct1_l2.ct"):
        ct = hio.load_ciphertext(str(GOLD / name), params)
        hio.save_ciphertext(str(tmp_path / name), ct, params)
        assert (tmp_path / name).read_bytes() == (GOLD / name).read_bytes()
    ct = hio.load_ciphertext(str(GOLD / "hcnk_unit_small_ct1.ct"), params)
    assert np.array_equal(np.stack(ct.host_residues()), golden_small["ct1"])
    # the loaded keys compute: rotate the loaded ciphertext, match the reference's rot1
    got = ckks.rotate(ct, 1, ks)
    assert np.array_equal(np.stack(got.host_residues()), golden_small["rot1"])
    pt = hio.load_packed_tensor(str(GOLD / "hcnk_unit_small.packed"), params)
    hio.save_packed_tensor(str(tmp_path / "p"), pt, params)
    assert (tmp_path / "p").read_bytes() == (GOLD / "hcnk_unit_small.packed").read_bytes()
    assert pt.fmt.variant == "B" and (pt.shape.c, pt.shape.h, pt.shape.w) == (8, 2, 2)
    assert torch.equal(pt.cts[0].data, ct.data)


@pytest.mark.gpu
def test_bootstrap_keyset_trailer(tmp_path):
    """a bootstrapping key set keeps its conjugation key and secret weight
    in the HCX1 trailer, which the reference's reader never reaches"""
    import torch
    from paper_2310_16530_b200 import ckks, io as hio
    params = ckks.CkksParams.build("unit-small", 256, 50, 40, 4, 50, 2)
    ks = ckks.keygen(params, np.random.default_rng(5), rotations=[1], secret_weight=16, conjugation=True)
    hio.save_keyset(str(tmp_path / "b"), ks)
    back = hio.load_keyset(str(tmp_path / "b"), params)
    assert back.secret_weight == 16
    assert torch.equal(back.conj.rows_b, ks.conj.rows_b) and torch.equal(back.conj.rows_a, ks.conj.rows_a)
