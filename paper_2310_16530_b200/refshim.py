"""Reference-side drop-in: run the reference package's own HyPHEN layers and
graph executor (``hcnn.packing`` / ``hcnn.graph``) over this engine's
HBM-resident ciphertexts.

The reference's layers reach the scheme through ``ckks.<fn>`` attribute
lookups plus a few name-bound imports:

* ``packing.py:34`` binds ``Ciphertext``; ``packing.py:36`` binds
  ``to_mont_rows`` / ``zero_poly``; ``_zero_ct`` (``packing.py:314-321``)
  builds a host zero ciphertext with ``Ciphertext(c0=..., c1=...)``;
* ``graph.py:41`` binds ``Ciphertext`` (``isinstance`` at ``graph.py:666``).

``enable(ckks, packing, graph)`` patches exactly those names on the
reference modules passed in (nothing here imports the reference), so a
reference maintainer switches backends with::

    from hcnn import ckks, packing, graph
    from paper_2310_16530_b200 import refshim
    refshim.enable(ckks, packing, graph)

after which ``hcnn.graph.execute`` and every ``hcnn.packing`` layer issue
their ciphertext arithmetic to the CUDA engine.  ``disable()`` restores the
originals.  Without a CUDA device the patched calls raise ``NativeError``
(no CPU fallback).
"""

from __future__ import annotations

from . import ckks as _gpu
from . import ring as _ring

# the scheme surface packing.py / graph.py call through ``ckks.<fn>``
# (packing.py:282-852, graph.py:435-572), plus keys and parameter presets
CKKS_NAMES = ("encode", "decode", "encrypt", "decrypt", "keygen", "hadd", "hsub", "padd", "pmult",
              "pmult_mont", "hmult", "square", "rescale", "mod_drop", "rotate", "rotation_plan",
              "galois_element", "debug_refresh", "mask_scale_for", "CkksParams", "Ciphertext", "Plaintext",
              "KeySet", "desk_a", "desk_b", "unit", "params_by_name")

_saved: list[tuple[object, str, object]] = []


def _zero_ct(params, level: int, scale: float, n: int):
    """packing.py:314-321 on the device: a zero ciphertext at `level`."""
    return _gpu.Ciphertext(params.ctx.zeros(2, level + 1, params.n), scale, n, params)


def _set(mod, name: str, value) -> None:
    _saved.append((mod, name, getattr(mod, name, None)))
    setattr(mod, name, value)


def enable(ckks, packing, graph) -> None:
    """Patch the reference modules (hcnn.ckks, hcnn.packing, hcnn.graph)."""
    if _saved:
        return
    for name in CKKS_NAMES:
        _set(ckks, name, getattr(_gpu, name))
    # name-bound hooks
    _set(packing, "Ciphertext", _gpu.Ciphertext)
    _set(packing, "CkksParams", _gpu.CkksParams)
    _set(packing, "KeySet", _gpu.KeySet)
    _set(packing, "mask_scale_for", _gpu.mask_scale_for)
    _set(packing, "to_mont_rows", _ring.to_mont_rows)
    _set(packing, "zero_poly", _ring.zero_poly)
    _set(packing, "_zero_ct", _zero_ct)
    _set(graph, "Ciphertext", _gpu.Ciphertext)
    _set(graph, "CkksParams", _gpu.CkksParams)
    _set(graph, "KeySet", _gpu.KeySet)
    _set(graph, "mask_scale_for", _gpu.mask_scale_for)


def disable() -> None:
    while _saved:
        mod, name, old = _saved.pop()
        setattr(mod, name, old)


def enabled() -> bool:
    return bool(_saved)
