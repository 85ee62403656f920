"""Where a bootstrap loses precision: decrypts the CtS output y and the
EvalMod output of an N=2^16 bootstrap and compares the latter with the host
evaluation of the same polynomial (bootstrap.evalmod_plain) on the decrypted
y.  argv: Chebyshev degree, EvalMod baby steps."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2310_16530_b200 import bootstrap as bt, ckks
    degree = int(sys.argv[1]) if len(sys.argv) > 1 else 31
    baby = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    cfg = bt.BootConfig(degree=degree)
    params = bt.boot_params("boot16", 1 << 16, 8, cfg)
    b = bt.Bootstrapper(params, cfg)
    ks = b.keygen(np.random.default_rng(16), rotations=[1])
    rng = np.random.default_rng(3)
    v = rng.uniform(-1, 1, params.slots)
    ct = ckks.encrypt(ckks.encode(v, params, 0), ks, rng)
    u, delta1 = b.coeff_to_slot(ct, ks)
    uc = ckks.conjugate(u, ks)
    ev = bt._Exact(params, ks)
    y = ev.add(u, uc)
    yd = np.real(ckks.decode(ckks.decrypt(y, ks), params, imag_tol=None))
    evx = bt._Exact(params, ks, fused=cfg.fused_moddown_rescale)
    c = bt.eval_chebyshev(evx, y, b.cheb, b.eval_scale, baby=baby)
    cd = np.real(ckks.decode(ckks.decrypt(c, ks), params, imag_tol=None))
    want_c = np.polynomial.chebyshev.chebval(yd, b.cheb)
    out = c
    for _ in range(cfg.double_angle):
        out = evx.cheb_product(out, out, None)
    od = np.real(ckks.decode(ckks.decrypt(out, ks), params, imag_tol=None))
    want_o = bt.evalmod_plain(cfg, yd)
    lg = lambda e: round(-float(np.log2(np.max(np.abs(e)) + 1e-300)), 2)
    print(json.dumps({"degree": degree, "baby": baby, "y_max": float(np.max(np.abs(yd))),
                      "y_scale_log2": round(float(np.log2(y.scale)), 3), "y_level": y.level,
                      "cheb_bits": lg(cd - want_c), "cheb_level": c.level,
                      "evalmod_bits": lg(od - want_o), "out_level": out.level,
                      "powers": sorted(bt.bsgs_powers(bt.bsgs_split(b.cheb, baby), baby))}), flush=True)


if __name__ == "__main__":
    main()
