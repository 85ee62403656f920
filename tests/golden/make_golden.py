"""Generate the committed golden fixtures from the UNMODIFIED reference.

Runs only in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py [small|deskA|bench16|layers|host|hcnk ...]

Outputs (all small enough to commit):
  golden_small.npz      full residue arrays at a 256-ring (the reference's
                        own small_setup params, test_ckks.py:46-52)
  golden_hashes.json    sha256 of residue arrays at desk-A (cfg 1) and at
                        N=2^16 (cfg 2, CkksParams.build("bench16",...)),
                        plus layer-level outputs (conv / basic block /
                        tiny-cnn) with their decrypted values
A hash is sha256 over the C-contiguous little-endian uint64 bytes.
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

os.environ.setdefault("HCNN_TEST_MODE", "1")
sys.setrecursionlimit(10000)

from hcnn import ckks, graph, packing, ring  # noqa: E402  (reference package)

HERE = Path(__file__).resolve().parent


def h(arr) -> str:
    import hashlib
    a = np.ascontiguousarray(np.asarray(arr, dtype=np.uint64))
    return hashlib.sha256(a.astype("<u8").tobytes()).hexdigest()


def ct_arr(ct) -> np.ndarray:
    return np.stack([ct.c0.coeffs, ct.c1.coeffs])


def key_arr(k) -> tuple[np.ndarray, np.ndarray]:
    return np.stack(k.rows_b), np.stack(k.rows_a)


def load_json():
    p = HERE / "golden_hashes.json"
    return json.loads(p.read_text()) if p.exists() else {}


def save_json(obj):
    (HERE / "golden_hashes.json").write_text(json.dumps(obj, indent=1, sort_keys=True) + "\n")


def meta():
    return {"numpy": np.__version__, "reference": "hcnn 0.1.0 @ /root/reference/pkg"}


# ---------------------------------------------------------------------------
def gen_small():
    params = ckks.CkksParams.build("unit-small", 256, 50, 40, 4, 50, 2)
    ext = params.q_mods + params.p_mods
    out = {"q": np.array([m.q for m in params.q_mods], np.uint64),
           "p": np.array([m.q for m in params.p_mods], np.uint64),
           "psi": np.array([ring.get_twiddles(m, params.n).psi for m in ext], np.uint64)}
    rng = np.random.default_rng(0)
    coeff = np.stack([rng.integers(0, m.q, size=params.n, dtype=np.uint64) for m in ext])
    p = ring.RnsPoly(ext, coeff.copy(), ring.Domain.COEFF)
    out["ntt_in"] = coeff
    out["ntt_out"] = ring.ntt_forward(p).coeffs
    # base conversion q0..q2 -> specials + q3
    src = params.q_mods[:3]
    dst = params.p_mods + params.q_mods[3:4]
    bc_in = ring.RnsPoly(src, coeff[:3].copy(), ring.Domain.COEFF)
    out["bc_out"] = ring.base_convert(bc_in, dst).coeffs
    # coefficient-domain automorphism
    out["auto5"] = ring.automorphism(p, 5).coeffs
    out["auto_g"] = ring.automorphism(p, ckks.galois_element(3, params.n)).coeffs

    ks = ckks.keygen(params, np.random.default_rng(3), rotations=[1, 2, 4])
    out["sk"] = ks.sk.coeffs
    out["pk_b"], out["pk_a"] = ks.pk[0].coeffs, ks.pk[1].coeffs
    out["rlk_b"], out["rlk_a"] = key_arr(ks.rlk)
    for s in (1, 2, 4):
        out[f"gk{s}_b"], out[f"gk{s}_a"] = key_arr(ks.gks[s])
    vrng = np.random.default_rng(12345)
    v1 = vrng.uniform(-1, 1, params.slots)
    v2 = vrng.uniform(-1, 1, params.slots)
    L = params.max_level
    pt1 = ckks.encode(v1, params, L)
    out["v1"], out["v2"] = v1, v2
    out["pt1"] = pt1.poly.coeffs
    ct1 = ckks.encrypt(pt1, ks, np.random.default_rng(77))
    ct2 = ckks.encrypt(ckks.encode(v2, params, L), ks, np.random.default_rng(78))
    out["ct1"], out["ct2"] = ct_arr(ct1), ct_arr(ct2)
    hm = ckks.hmult(ct1, ct2, ks)
    out["hmult"] = ct_arr(hm)
    out["rescale"] = ct_arr(ckks.rescale(hm, params))
    for k in (1, 3, -1, 4):
        out[f"rot{k}"] = ct_arr(ckks.rotate(ct1, k, ks))
    out["dec_hmult"] = ckks.decode(ckks.decrypt(ckks.rescale(hm, params), ks), params)
    out["pmult"] = ct_arr(ckks.pmult(ct1, pt1))
    out["hadd"] = ct_arr(ckks.hadd(ct1, ct2))
    out["padd"] = ct_arr(ckks.padd(ct1, pt1))
    np.savez_compressed(HERE / "golden_small.npz", **out)
    print("small done")


# ---------------------------------------------------------------------------
def scheme_hashes(params, key_seed, rotations, rot_tests, tag):
    t0 = time.time()
    ks = ckks.keygen(params, np.random.default_rng(key_seed), rotations=rotations)
    t_key = time.time() - t0
    res = {"params": {"n": params.n, "q": [m.q for m in params.q_mods], "p": [m.q for m in params.p_mods]},
           "key_seed": key_seed, "rotations": list(rotations)}
    res["sk"] = h(ks.sk.coeffs)
    res["pk"] = h(np.stack([ks.pk[0].coeffs, ks.pk[1].coeffs]))
    b, a = key_arr(ks.rlk)
    res["rlk"] = h(np.stack([b, a]))
    res["gks"] = {}
    for s in sorted(ks.gks):
        b, a = key_arr(ks.gks[s])
        res["gks"][str(s)] = h(np.stack([b, a]))
    vrng = np.random.default_rng(12345)
    v1 = vrng.uniform(-1, 1, params.slots)
    v2 = vrng.uniform(-1, 1, params.slots)
    L = params.max_level
    pt1 = ckks.encode(v1, params, L)
    res["pt1"] = h(pt1.poly.coeffs)
    ct1 = ckks.encrypt(pt1, ks, np.random.default_rng(77))
    ct2 = ckks.encrypt(ckks.encode(v2, params, L), ks, np.random.default_rng(78))
    res["ct1"], res["ct2"] = h(ct_arr(ct1)), h(ct_arr(ct2))
    coeff_rng = np.random.default_rng(0)
    ext = params.q_mods + params.p_mods
    coeff = np.stack([coeff_rng.integers(0, m.q, size=params.n, dtype=np.uint64) for m in ext])
    res["ntt_in_seed0"] = h(coeff)
    res["ntt_out_seed0"] = h(ring.ntt_forward(ring.RnsPoly(ext, coeff, ring.Domain.COEFF)).coeffs)
    t0 = time.time()
    hm = ckks.hmult(ct1, ct2, ks)
    t_hm = time.time() - t0
    res["hmult"] = h(ct_arr(hm))
    t0 = time.time()
    rs = ckks.rescale(hm, params)
    t_rs = time.time() - t0
    res["rescale"] = h(ct_arr(rs))
    dec = ckks.decode(ckks.decrypt(rs, ks), params)
    res["dec_hmult_err"] = float(np.max(np.abs(dec - v1 * v2)))
    res["dec_hmult_head"] = [float(x) for x in dec[:8]]
    res["rot"] = {}
    t_rot = None
    for k in rot_tests:
        t0 = time.time()
        r = ckks.rotate(ct1, k, ks)
        if t_rot is None:
            t_rot = time.time() - t0
        res["rot"][str(k)] = h(ct_arr(r))
    res["ref_cpu_seconds"] = {"keygen": t_key, "hmult": t_hm, "rescale": t_rs, "rotate_first": t_rot}
    res["meta"] = meta()
    print(tag, "done", res["ref_cpu_seconds"])
    return res


def gen_deska():
    obj = load_json()
    obj["deskA"] = scheme_hashes(ckks.desk_a(), 0xA11CE, [1 << i for i in range(12)], [1, 5, -1, 2048], "deskA")
    save_json(obj)


def gen_bench16():
    obj = load_json()
    p = ckks.CkksParams.build("bench16", 1 << 16, 59, 40, 24, 59, 4)
    obj["bench16"] = scheme_hashes(p, 1, [1, 4], [1, 5], "bench16")
    save_json(obj)


# ---------------------------------------------------------------------------
def gen_layers():
    """Layer-level goldens: the acceptance suite's desk-A basic block (gate 4
    setup, test_acceptance.py:73-93, 282-309) and one desk-B tiny-cnn
    inference (gate 7 setup, test_acceptance.py:96-105, 415-449)."""
    obj = load_json()
    res = {}
    params = ckks.desk_a()
    stack_fx = graph.gen_fixture("basic-block-stack(1)", 21, params)
    stack_g = graph.build_graph("basic-block-stack(1)", stack_fx, multiplex=8)
    steps = sorted(graph.required_rotation_steps(stack_g, params.slots))
    t0 = time.time()
    ks = ckks.keygen(params, np.random.default_rng(0xACCE), rotations=steps)
    plan = graph.plan_levels(stack_g, params.max_level)
    x = np.asarray(stack_fx["golden"][0]["input"])
    packed = packing.encrypt_tensor(x, stack_g.input_format, ks, np.random.default_rng(0xACC4),
                                    plan.entry_levels[0])
    t1 = time.time()
    out, rep = graph.execute(stack_g, plan, packed, ks, "encrypted")
    t_exec = time.time() - t1
    dec = packing.decrypt_tensor(out, ks)
    ref, _ = graph.execute(stack_g, plan, x, mode="plaintext-ref")
    res["block"] = {
        "steps": steps, "key_seed": 0xACCE, "enc_seed": 0xACC4,
        "input": h(np.stack([ct_arr(c) for c in packed.cts])),
        "output": h(np.stack([ct_arr(c) for c in out.cts])),
        "entries": [r["entry_level"] for r in rep.per_layer],
        "tally": rep.totals().as_dict(),
        "per_layer_out": [],
        "dec_max_err_vs_plain": float(np.max(np.abs(dec - ref))),
        "dec_head": [float(v) for v in dec.ravel()[:16]],
        "ref_cpu_seconds": t_exec,
    }
    # first conv alone
    layer = stack_g.layers[0]
    conv_out = packing.conv2d(packed, layer.spec, ks, None, {}, tag=layer.name)
    res["block"]["conv1_out"] = h(np.stack([ct_arr(c) for c in conv_out.cts]))
    print("block done", time.time() - t0)

    # tiny-cnn at desk-B, one inference
    params = ckks.desk_b()
    fx = graph.gen_fixture("tiny-cnn", 42, params)
    g = graph.build_graph("tiny-cnn", fx, multiplex=8)
    plan = graph.plan_levels(g, params.max_level)
    steps = sorted(graph.required_rotation_steps(g, params.slots))
    ks = ckks.keygen(params, np.random.default_rng(0xB0B), rotations=steps)
    rng = np.random.default_rng(0xACC7)
    x = rng.uniform(-1.0, 1.0, (1, 8, 8))
    packed = packing.encrypt_tensor(x, g.input_format, ks, rng, plan.entry_levels[0])
    t1 = time.time()
    out, rep = graph.execute(g, plan, packed, ks, "encrypted", cache={})
    t_exec = time.time() - t1
    logits = packing.read_logits(out, g.n_classes, g.formats[-1], ks)
    ref, _ = graph.execute(g, plan, x, mode="plaintext-ref")
    res["tiny"] = {
        "steps": steps, "key_seed": 0xB0B, "input_seed": 0xACC7,
        "plan": plan.as_dict(),
        "output": h(ct_arr(out)),
        "logits": [float(v) for v in logits],
        "plain_logits": [float(v) for v in ref],
        "tally": rep.totals().as_dict(),
        "ref_cpu_seconds": t_exec,
    }
    res["meta"] = meta()
    obj["layers"] = res
    save_json(obj)
    print("tiny done", time.time() - t0)


def hf(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.float64)).astype("<f8").tobytes()).hexdigest()


def gen_host():
    """Host-side goldens (CPU tests): fixtures, folds, plans, rotation-step
    sets, layouts -- everything the GPU path consumes as plaintext input."""
    from hcnn import aespa
    obj = load_json()
    res = {"hermite2": list(aespa.hermite_coeffs(2).f_hat), "hermite4": list(aespa.hermite_coeffs(4).f_hat)}
    fixtures = {}
    for topo, seed, pname in (("tiny-cnn", 42, "desk-B"), ("basic-block-stack(1)", 21, "desk-A"),
                              ("basic-block-stack(2)", 7, "desk-A")):
        params = ckks.params_by_name(pname)
        fx = graph.gen_fixture(topo, seed, params, golden_count=2)
        g = graph.build_graph(topo, fx, multiplex=8)
        ent = {"digest": graph.weights_digest(fx), "golden": fx["golden"],
               "plan": graph.plan_levels(g, params.max_level).as_dict(),
               "plan_t5": graph.plan_levels(g, 7, 5).as_dict(),
               "steps": sorted(graph.required_rotation_steps(g, params.slots)),
               "steps_fixed": sorted(graph.required_rotation_steps(g, params.slots, include_fixed=True)),
               "layers": []}
        for L in g.layers:
            row = {"kind": L.kind, "fold_forward": L.fold_forward}
            if L.kind == "conv":
                row["eff_w"] = hf(L.spec.effective_weights())
                row["bias_map"] = None if L.spec.bias_map is None else hf(L.spec.bias_map)
                row["low_scale_out"] = L.spec.low_scale_out
            if L.kind == "act":
                row["quads"] = [[q.a, q.b, q.c] for q in L.quads]
            ent["layers"].append(row)
        x = np.asarray(fx["golden"][0]["input"])
        plan = graph.plan_levels(g, params.max_level)
        ent["plain_out"] = hf(graph.execute(g, plan, x, mode="plaintext-ref")[0])
        fixtures[f"{topo}|{seed}|{pname}"] = ent
    res["fixtures"] = fixtures
    lay = {}
    rng = np.random.default_rng(11)
    for fa, shape, slots in ((("B", 4, 1, 4), (4, 2, 2), 32), (("A", 4, 1, 16), (4, 4, 4), 256),
                             (("B", 2, 2, 16), (3, 2, 2), 256), (("B", 8, 2, 64), (12, 4, 4), 1024)):
        fmt = packing.PackingFormat(*fa)
        t = rng.uniform(-1, 1, shape)
        L = packing.Layout(fmt, packing.TensorShape(*shape), slots)
        lay["|".join(map(str, fa + shape + (slots,)))] = {
            "input": t.tolist(),
            "pack": [hf(v) for v in packing.pack(t, fmt, slots)],
            "occ": [hf(L.occupancy(i)) for i in range(L.n_cts)],
            "pool_fc_steps": sorted(packing.pool_fc_rotation_steps(packing.TensorShape(*shape), fmt, slots,
                                                                   shape[0], 3)),
        }
    res["layouts"] = lay
    res["meta"] = meta()
    obj["host"] = res
    save_json(obj)
    print("host done")


# ---------------------------------------------------------------------------
def gen_hcnk():
    """HCNK containers written by the reference's io.py (io.py:54-249) for the
    unit-small key set and ciphertexts of gen_small: the device loader must
    read them, and the device writer must reproduce them byte for byte."""
    from hcnn import io as hio
    params = ckks.CkksParams.build("unit-small", 256, 50, 40, 4, 50, 2)
    ks = ckks.keygen(params, np.random.default_rng(3), rotations=[1, 2, 4])
    vrng = np.random.default_rng(12345)
    v1 = vrng.uniform(-1, 1, params.slots)
    L = params.max_level
    ct1 = ckks.encrypt(ckks.encode(v1, params, L), ks, np.random.default_rng(77))
    hio.save_keyset(str(HERE / "hcnk_unit_small.keyset"), ks)
    hio.save_ciphertext(str(HERE / "hcnk_unit_small_ct1.ct"), ct1, params)
    hio.save_ciphertext(str(HERE / "hcnk_unit_small_ct1_l2.ct"), ckks.mod_drop(ct1, 2), params)
    from hcnn.packing import PackedTensor, PackingFormat, TensorShape
    pt = PackedTensor(cts=[ct1, ckks.mod_drop(ct1, L)], fmt=PackingFormat("B", 4, 1, 4),
                      shape=TensorShape(8, 2, 2))
    hio.save_packed_tensor(str(HERE / "hcnk_unit_small.packed"), pt, params)
    print("hcnk done")


# ---------------------------------------------------------------------------
def gen_packing():
    """Layer goldens on the reference's own packing-unit setup
    (test_packing.py:74-119, pack-unit N=512, L=7) for every HyPHEN layer
    function on the ResNet20 path that the layer digests do not already
    cover: stride-2 conv in both directions (test_packing.py:363-383),
    downsample (packing.py:714-740, test_packing.py:515-525),
    conv2d_fixed_baseline (packing.py:620-673, test_packing.py:447-477),
    he_activation / avgpool / fc (test_packing.py:483-575); plus
    cost_report_compare on the graph-unit tiny-cnn (graph.py:637-682,
    test_graph.py:86-117, 504-508)."""
    from hcnn import packing as P
    from hcnn.aespa import AespaChannelParams, fold_channels, hermite_coeffs
    obj = load_json()
    res = {}
    params = ckks.CkksParams.build("pack-unit", 512, 50, 40, 7, 50, 2)
    slots = params.slots
    A, B = P.FORMAT_A, P.FORMAT_B
    m4A, m4B = P.PackingFormat(A, 4, 1, 16), P.PackingFormat(B, 4, 1, 16)
    m2A, m2B = P.PackingFormat(A, 2, 1, 16), P.PackingFormat(B, 2, 1, 16)
    m2A2, m2B2 = P.PackingFormat(A, 2, 2, 16), P.PackingFormat(B, 2, 2, 16)
    w4, w2 = np.ones((4, 4, 3, 3)), np.ones((2, 2, 3, 3))
    sh4, sh2 = P.TensorShape(4, 4, 4), P.TensorShape(2, 4, 4)
    layers = [
        (P.ConvLayerSpec(w4, 1, m4A, m4B), sh4, False),
        (P.ConvLayerSpec(w4, 1, m4A, m4A), sh4, True),
        (P.ConvLayerSpec(w2, 2, m2A, m2B2), sh2, False),
        (P.ConvLayerSpec(w2, 2, m2B, m2A2), sh2, False),
        (P.ConvLayerSpec(w2, 1, m2B2, m2A2), P.TensorShape(2, 2, 2), False),
        (P.ConvLayerSpec(w2, 1, m2A2, m2B2), P.TensorShape(2, 2, 2), False),
    ]
    steps = set()
    for layer, shape, fixed in layers:
        steps |= P.conv_rotation_steps(layer, shape, slots, fixed=fixed)
    steps |= P.pool_fc_rotation_steps(sh4, m4A, slots, 4, 3)
    steps |= P.pool_fc_rotation_steps(sh4, m4B, slots, 4, 3)
    steps = sorted(steps)
    ks = ckks.keygen(params, np.random.default_rng(0xBEEF), rotations=steps)
    res["params"] = {"n": params.n, "q": [m.q for m in params.q_mods], "p": [m.q for m in params.p_mods]}
    res["steps"], res["key_seed"] = steps, 0xBEEF

    def cts(x):
        return h(np.stack([ct_arr(c) for c in x.cts]))

    def rec(name, x_in, y, tally=None, extra=None):
        d = {"input": cts(x_in), "output": cts(y) if hasattr(y, "cts") else h(ct_arr(y)),
             "level": y.level, "scale": y.scale}
        if hasattr(y, "cts"):
            d["fmt"] = [y.fmt.variant, y.fmt.multiplex, y.fmt.gap, y.fmt.span]
            d["shape"] = [y.shape.c, y.shape.h, y.shape.w]
            d["dec"] = [float(v) for v in P.decrypt_tensor(y, ks).ravel()]
        if tally is not None:
            d["tally"] = tally.as_dict()
        if extra:
            d.update(extra)
        res[name] = d

    # stride 2, A -> B (test_packing.py:363-374) and B -> A
    for name, seed, fin, fout in (("stride2_a2b", 11, m2A, m2B2), ("stride2_b2a", 13, m2B, m2A2)):
        rng = np.random.default_rng(seed)
        t = rng.standard_normal((2, 4, 4))
        w = rng.standard_normal((2, 2, 3, 3)) * 0.4
        b = rng.standard_normal(2) * 0.2
        x = P.encrypt_tensor(t, fin, ks, rng, params.max_level)
        tally = P.OpTally()
        y = P.conv2d(x, P.ConvLayerSpec(w, 2, fin, fout, bias=b), ks, tally)
        rec(name, x, y, tally)
    # conv at the doubled gap (test_packing.py:376-383), both directions
    rng = np.random.default_rng(12)
    t = rng.standard_normal((2, 4, 4))
    w = rng.standard_normal((2, 2, 3, 3)) * 0.4
    x = P.encrypt_tensor(t, m2A, ks, rng, params.max_level)
    mid = P.conv2d(x, P.ConvLayerSpec(w, 2, m2A, m2B2), ks)
    tally = P.OpTally()
    out = P.conv2d(mid, P.ConvLayerSpec(w, 1, m2B2, m2A2), ks, tally)
    rec("gap2_b2a", mid, out, tally)
    tally = P.OpTally()
    out2 = P.conv2d(out, P.ConvLayerSpec(w, 1, m2A2, m2B2), ks, tally)
    rec("gap2_a2b", out, out2, tally)
    # fixed baseline (test_packing.py:447-477)
    rng = np.random.default_rng(21)
    t = rng.standard_normal((4, 4, 4))
    w = rng.standard_normal((4, 4, 3, 3)) * 0.4
    b = rng.standard_normal(4) * 0.2
    xa = P.encrypt_tensor(t, m4A, ks, rng, params.max_level)
    t_alt, t_fix = P.OpTally(), P.OpTally()
    y_alt = P.conv2d(xa, P.ConvLayerSpec(w, 1, m4A, m4B, bias=b), ks, t_alt)
    y_fix = P.conv2d_fixed_baseline(xa, P.ConvLayerSpec(w, 1, m4A, m4A, bias=b), ks, t_fix)
    rec("alt_a2b", xa, y_alt, t_alt)
    rec("fixed", xa, y_fix, t_fix)
    rng = np.random.default_rng(22)
    t = rng.standard_normal((4, 4, 4))
    w = rng.standard_normal((4, 4, 3, 3)) * 0.4
    x = P.encrypt_tensor(t, m4A, ks, rng, 4)
    tally = P.OpTally()
    y = P.conv2d_fixed_baseline(x, P.ConvLayerSpec(w, 1, m4A, m4A), ks, tally)
    rec("fixed_l4", x, y, tally)
    # activation (test_packing.py:483-500)
    rng = np.random.default_rng(31)
    t = rng.standard_normal((4, 4, 4))
    chans = [AespaChannelParams(gamma=0.8 + 0.1 * i, beta=0.05 * i, mu=(0.1, -0.05, 0.02),
                                sigma2=(1.1, 0.9, 1.3)) for i in range(4)]
    quads = fold_channels(chans, hermite_coeffs(2))
    x = P.encrypt_tensor(t, m4B, ks, rng, 4)
    tally = P.OpTally()
    y = P.he_activation(x, quads, ks, tally)
    rec("act", x, y, tally)
    # downsample (test_packing.py:515-525) on both formats
    for name, seed, fmt in (("down_a", 32, m2A), ("down_b", 36, m2B)):
        rng = np.random.default_rng(seed)
        t = rng.standard_normal((2, 4, 4))
        x = P.encrypt_tensor(t, fmt, ks, rng, 4)
        tally = P.OpTally()
        y = P.downsample(x, ks, tally)
        rec(name, x, y, tally)
    # pool + fc (test_packing.py:537-562)
    for variant in (A, B):
        rng = np.random.default_rng(34)
        t = rng.standard_normal((4, 4, 4))
        wfc = rng.standard_normal((3, 4)) * 0.5
        bfc = rng.standard_normal(3) * 0.2
        fmt = P.PackingFormat(variant, 4, 1, 16)
        x = P.encrypt_tensor(t, fmt, ks, rng, 4)
        tally = P.OpTally()
        pooled = P.avgpool_global(x, ks, tally)
        rec(f"pool_{variant}", x, pooled, tally)
        tally = P.OpTally()
        out = P.fully_connected(pooled, wfc, bfc, ks, tally)
        rec(f"fc_{variant}", pooled, out, tally,
            {"logits": [float(v) for v in P.read_logits(out, 3, fmt, ks)]})

    # cost_report_compare on the graph-unit tiny-cnn (test_graph.py:86-117, 504-508)
    gp = ckks.CkksParams.build("graph-unit", 2048, 50, 40, 11, 50, 2)
    fx = graph.gen_fixture("tiny-cnn", 7, gp, golden_count=2)
    g = graph.build_graph("tiny-cnn", fx, multiplex=4)
    gsteps = sorted(graph.required_rotation_steps(g, gp.slots, include_fixed=True))
    gks = ckks.keygen(gp, np.random.default_rng(0xD00D), rotations=gsteps)
    plan = graph.plan_levels(g, gp.max_level)
    x = np.array(fx["golden"][0]["input"])
    cmp = graph.cost_report_compare(g, plan, x, gks, np.random.default_rng(9))
    res["compare"] = {"steps": gsteps, "key_seed": 0xD00D, "report": cmp}
    res["meta"] = meta()
    obj["packing"] = res
    save_json(obj)
    print("packing done")


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "deskA", "bench16", "layers", "host", "hcnk"]
    for w in which:
        {"small": gen_small, "deskA": gen_deska, "bench16": gen_bench16, "layers": gen_layers,
         "host": gen_host, "hcnk": gen_hcnk, "packing": gen_packing}[w]()
