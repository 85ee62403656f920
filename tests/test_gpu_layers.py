"""Layer-level drop-in parity: the HyPHEN conv / AESPA activation / pool /
dense head and the graph executor on device ciphertexts reproduce the
reference's residues bit for bit (digests frozen by
tests/golden/make_golden.py gen_layers from the unmodified reference:
the acceptance suite's desk-A basic block and one desk-B tiny-cnn
inference), with identical op tallies and decrypted values."""

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def h(arr) -> str:
    a = np.ascontiguousarray(np.asarray(arr, dtype=np.uint64))
    return hashlib.sha256(a.astype("<u8").tobytes()).hexdigest()


def _cts(cts):
    return np.stack([np.stack(c.host_residues()) for c in cts])


def test_basic_block_bit_exact(golden_hashes):
    from paper_2310_16530_b200 import ckks, graph, packing
    gold = golden_hashes["layers"]["block"]
    params = ckks.desk_a()
    fx = graph.gen_fixture("basic-block-stack(1)", 21, params)
    g = graph.build_graph("basic-block-stack(1)", fx, multiplex=8)
    steps = sorted(graph.required_rotation_steps(g, params.slots))
    assert steps == gold["steps"]
    ks = ckks.keygen(params, np.random.default_rng(gold["key_seed"]), rotations=steps)
    plan = graph.plan_levels(g, params.max_level)
    x = np.asarray(fx["golden"][0]["input"])
    packed = packing.encrypt_tensor(x, g.input_format, ks, np.random.default_rng(gold["enc_seed"]),
                                    plan.entry_levels[0])
    assert h(_cts(packed.cts)) == gold["input"]
    conv1 = packing.conv2d(packed, g.layers[0].spec, ks, None, {}, tag=g.layers[0].name)
    assert h(_cts(conv1.cts)) == gold["conv1_out"]
    out, rep = graph.execute(g, plan, packed, ks, "encrypted")
    assert [r["entry_level"] for r in rep.per_layer] == gold["entries"]
    assert rep.totals().as_dict() == gold["tally"]
    assert h(_cts(out.cts)) == gold["output"]
    dec = packing.decrypt_tensor(out, ks)
    assert [float(v) for v in dec.ravel()[:16]] == gold["dec_head"]


def test_tiny_cnn_desk_b_bit_exact(golden_hashes):
    from paper_2310_16530_b200 import ckks, graph, packing
    gold = golden_hashes["layers"]["tiny"]
    params = ckks.desk_b()
    fx = graph.gen_fixture("tiny-cnn", 42, params)
    g = graph.build_graph("tiny-cnn", fx, multiplex=8)
    plan = graph.plan_levels(g, params.max_level)
    assert plan.as_dict() == gold["plan"]
    steps = sorted(graph.required_rotation_steps(g, params.slots))
    assert steps == gold["steps"]
    ks = ckks.keygen(params, np.random.default_rng(gold["key_seed"]), rotations=steps)
    rng = np.random.default_rng(gold["input_seed"])
    x = rng.uniform(-1.0, 1.0, (1, 8, 8))
    packed = packing.encrypt_tensor(x, g.input_format, ks, rng, plan.entry_levels[0])
    out, rep = graph.execute(g, plan, packed, ks, "encrypted", cache={})
    assert rep.totals().as_dict() == gold["tally"]
    assert h(np.stack(out.host_residues())) == gold["output"]
    logits = packing.read_logits(out, g.n_classes, g.formats[-1], ks)
    assert [float(v) for v in logits] == gold["logits"]
    ref, _ = graph.execute(g, plan, x, mode="plaintext-ref")
    assert np.max(np.abs(logits - ref)) < 1e-2
    assert int(np.argmax(logits)) == int(np.argmax(ref))


def test_execute_many_matches_single_images(golden_hashes):
    """graph.execute_many (B images in lockstep, bench.py --images-per-gpu)
    gives each image exactly its single-image residues and op tally on a
    graph without refresh points (the acceptance basic block, desk-A)."""
    import torch
    from paper_2310_16530_b200 import ckks, graph, packing
    gold = golden_hashes["layers"]["block"]
    params = ckks.desk_a()
    fx = graph.gen_fixture("basic-block-stack(1)", 21, params)
    g = graph.build_graph("basic-block-stack(1)", fx, multiplex=8)
    steps = sorted(graph.required_rotation_steps(g, params.slots))
    ks = ckks.keygen(params, np.random.default_rng(gold["key_seed"]), rotations=steps)
    plan = graph.plan_levels(g, params.max_level)
    assert not plan.refresh_points
    rng = np.random.default_rng(5)
    xs = [packing.encrypt_tensor(rng.uniform(-1, 1, (8, 8, 8)), g.input_format, ks, rng, plan.entry_levels[0])
          for _ in range(3)]
    cache: dict = {}
    many = graph.execute_many(g, plan, xs, ks, cache=cache)
    for x, (out, rep) in zip(xs, many):
        one, rep1 = graph.execute(g, plan, x, ks, "encrypted", cache=cache)
        assert rep.totals().as_dict() == rep1.totals().as_dict()
        assert all(torch.equal(a.data, b.data) for a, b in zip(out.cts, one.cts))
    assert h(_cts(many[0][0].cts)) != h(_cts(many[1][0].cts))


def test_stacked_images_match_single_images(golden_hashes):
    """graph.stack_images: ciphertexts holding B images ([B, 2, l+1, N]) run
    through the executor once (bench.py --images-per-gpu B, batch-mode
    stack); every image's residues and tally equal its single-image run."""
    import torch
    from paper_2310_16530_b200 import ckks, graph, packing
    gold = golden_hashes["layers"]["block"]
    params = ckks.desk_a()
    fx = graph.gen_fixture("basic-block-stack(1)", 21, params)
    g = graph.build_graph("basic-block-stack(1)", fx, multiplex=8)
    steps = sorted(graph.required_rotation_steps(g, params.slots))
    ks = ckks.keygen(params, np.random.default_rng(gold["key_seed"]), rotations=steps)
    plan = graph.plan_levels(g, params.max_level)
    rng = np.random.default_rng(6)
    xs = [packing.encrypt_tensor(rng.uniform(-1, 1, (8, 8, 8)), g.input_format, ks, rng, plan.entry_levels[0])
          for _ in range(3)]
    cache: dict = {}
    out, rep = graph.execute(g, plan, graph.stack_images(xs), ks, "encrypted", cache=cache)
    assert ckks.image_batch() == 1  # the image-batch context is scoped to the call
    for x, o in zip(xs, graph.unstack_images(out)):
        one, rep1 = graph.execute(g, plan, x, ks, "encrypted", cache=cache)
        assert rep.totals().as_dict() == rep1.totals().as_dict()
        assert all(torch.equal(a.data, b.data) for a, b in zip(o.cts, one.cts))
