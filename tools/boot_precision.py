"""Bootstrap precision (bits, max-abs over all 32768 slots) of N=2^16
chains with different prime sizes: the default boot16 chain (58-bit
CtS/EvalMod primes, 61-bit specials) against narrow ones whose every limb but
q0 (and one special) fits the FP64 NTT network (q < 2^41).  Prints a JSON
line per chain: bits for two inputs and ms per bootstrap (eager)."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2310_16530_b200 import bootstrap as bt, ckks
    chains = {"wide": dict(big_bits=58, special_bits=61, n_special=4),
              "narrow": dict(big_bits=40, special_bits=(61, 40, 40, 40), n_special=4),
              "big40": dict(big_bits=40, special_bits=61, n_special=4),
              "mixsp": dict(big_bits=58, special_bits=(61, 40, 40, 40), n_special=4)}
    degree = int(sys.argv[1]) if len(sys.argv) > 1 else 59
    pick = sys.argv[2].split(",") if len(sys.argv) > 2 else list(chains)
    r = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    for name in pick:
        kw = chains[name]
        cfg = bt.BootConfig(degree=degree, double_angle=r)
        params = bt.boot_params("boot16", 1 << 16, 8, cfg, **kw)
        b = bt.Bootstrapper(params, cfg)
        ks = b.keygen(np.random.default_rng(16), rotations=[1])
        rng = np.random.default_rng(3)
        bits = []
        for _ in range(2):
            v = rng.uniform(-1, 1, params.slots)
            ct = ckks.encrypt(ckks.encode(v, params, 0), ks, rng)
            out = b.bootstrap(ct, ks)
            d = ckks.decode(ckks.decrypt(out, ks), params, imag_tol=None)
            e = np.abs(np.real(d) - v)
            bits.append({"max": round(-float(np.log2(e.max())), 2),
                         "p999": round(-float(np.log2(np.quantile(e, 0.999))), 2),
                         "median": round(-float(np.log2(np.median(e))), 2),
                         "imag_max": round(-float(np.log2(np.max(np.abs(np.imag(d))) + 1e-300)), 2),
                         "worst_slots": [int(i) for i in np.argsort(e)[-3:]]})
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            b.bootstrap(ct, ks)
        torch.cuda.synchronize()
        print(json.dumps({"chain": name, "degree": degree, "double_angle": r, **{k: str(v) for k, v in kw.items()}, "bits": bits,
                          "ms_eager": round((time.perf_counter() - t) / 5 * 1e3, 2)}), flush=True)
        del b, ks
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
