"""Device context: one CkksParams (or one bare modulus chain) resident in HBM.

Thin host wrapper over the C ABI.  Residue tensors are torch int64 tensors
on the CUDA device holding the uint64 bit patterns, shaped [npolys, nlimbs, N]
(or [nlimbs, N] for a single polynomial), limb-major exactly like
RnsPoly.coeffs in the reference (ring.py:204-213).  Everything is enqueued on
torch's current CUDA stream; torch's caching allocator provides outputs and
scratch, so calls allocate nothing from the driver in steady state.
"""

from __future__ import annotations

import ctypes
import threading
from typing import Sequence

import numpy as np
import torch

from . import _native
from .errors import BasisError, LevelError, NativeError

_ctx_cache: dict[tuple, "DeviceContext"] = {}
_ctx_lock = threading.Lock()


def _require_cuda(device: int) -> None:
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device visible: the hcnn-b200 engine has no CPU fallback")


def _ptr(t: torch.Tensor | None) -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(0)
    return ctypes.c_void_p(t.data_ptr())


def _stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def to_device_u64(arr: np.ndarray, device: int | torch.device = 0) -> torch.Tensor:
    """uint64 numpy array -> int64 CUDA tensor with the same bits."""
    a = np.ascontiguousarray(arr, dtype=np.uint64)
    return torch.from_numpy(a.view(np.int64)).to(device=f"cuda:{device}" if isinstance(device, int) else device)


def to_host_u64(t: torch.Tensor) -> np.ndarray:
    """int64 CUDA tensor -> uint64 numpy array (synchronising copy)."""
    return t.detach().to("cpu").contiguous().numpy().view(np.uint64)


class DeviceContext:
    """An hcnn_ctx: moduli constants, twiddles (reference psi) and the
    lazily built base-conversion tables for one ring degree and chain."""

    def __init__(self, n: int, q_list: Sequence[int], p_list: Sequence[int] = (), device: int = 0):
        _require_cuda(device)
        self.lib = _native.load()
        self.n = int(n)
        self.logn = self.n.bit_length() - 1
        self.q_list = tuple(int(q) for q in q_list)
        self.p_list = tuple(int(p) for p in p_list)
        self.Lq = len(self.q_list)
        self.K = len(self.p_list)
        self.device = device
        self.torch_device = torch.device(f"cuda:{device}")
        h = ctypes.c_void_p()
        with torch.cuda.device(device):
            _native.check(self.lib.hcnn_ctx_create(
                ctypes.byref(h), device, self.n,
                _native.u64_array(self.q_list), self.Lq,
                _native.u64_array(self.p_list) if self.p_list else None, self.K))
        self.handle = h
        self.launches = 0

    def __del__(self):
        try:
            if getattr(self, "handle", None) and self.handle.value:
                self.lib.hcnn_ctx_destroy(self.handle)
        except Exception:
            pass

    # -- helpers -----------------------------------------------------------
    def empty(self, *shape) -> torch.Tensor:
        return torch.empty(shape, dtype=torch.int64, device=self.torch_device)

    def zeros(self, *shape) -> torch.Tensor:
        return torch.zeros(shape, dtype=torch.int64, device=self.torch_device)

    def psi(self, mod_index: int) -> int:
        v = ctypes.c_uint64()
        _native.check(self.lib.hcnn_ctx_psi(self.handle, mod_index, ctypes.byref(v)))
        return int(v.value)

    def _chk(self, rc: int) -> None:
        self.launches += 1
        _native.check(rc)

    @staticmethod
    def _npolys(t: torch.Tensor, nq: int, np_: int, n: int) -> int:
        nl = nq + np_
        total = t.numel()
        if total % (nl * n):
            raise BasisError(f"tensor of {total} residues is not a batch over {nl} limbs of {n}")
        if not t.is_contiguous():
            raise BasisError("residue tensors must be contiguous")
        return total // (nl * n)

    # -- ring.py level ops ----------------------------------------------------
    def ntt(self, t: torch.Tensor, nq: int, np_: int = 0, inverse: bool = False) -> torch.Tensor:
        """In-place forward (coeff->eval) or inverse NTT of every limb."""
        npolys = self._npolys(t, nq, np_, self.n)
        fn = self.lib.hcnn_ntt_inverse if inverse else self.lib.hcnn_ntt_forward
        self._chk(fn(self.handle, _ptr(t), nq, np_, npolys, _stream()))
        return t

    def binop(self, op: str, a: torch.Tensor, b: torch.Tensor, nq: int, np_: int = 0,
              out: torch.Tensor | None = None, plain_c0: bool = False) -> torch.Tensor:
        """plain_c0: a holds ciphertexts ([.., 2, limbs, N]), b one plaintext
        poly added to every c0; every c1 is copied (hcnn_poly_add b_broadcast 2)."""
        npolys = self._npolys(a, nq, np_, self.n)
        nb = self._npolys(b, nq, np_, self.n)
        if plain_c0:
            if nb != 1 or npolys % 2 or op not in ("add", "sub"):
                raise BasisError("plain_c0: one plaintext poly against whole ciphertexts")
            bcast = 2
        else:
            bcast = 1 if (nb == 1 and npolys > 1) else 0
        if not bcast and nb != npolys:
            raise BasisError("operand batch sizes differ")
        if out is None:
            out = torch.empty_like(a)
        fn = {
            "add": self.lib.hcnn_poly_add,
            "sub": self.lib.hcnn_poly_sub,
            "mul": self.lib.hcnn_poly_mul,
            "mul_mont": self.lib.hcnn_poly_mul_mont,
            "mac_mont": self.lib.hcnn_poly_mac_mont,
        }[op]
        self._chk(fn(self.handle, _ptr(out), _ptr(a), _ptr(b), nq, np_, npolys, bcast, _stream()))
        return out

    def unop(self, op: str, a: torch.Tensor, nq: int, np_: int = 0,
             out: torch.Tensor | None = None) -> torch.Tensor:
        npolys = self._npolys(a, nq, np_, self.n)
        if out is None:
            out = torch.empty_like(a)
        fn = {
            "neg": self.lib.hcnn_poly_neg,
            "to_mont": self.lib.hcnn_to_mont,
            "from_mont": self.lib.hcnn_from_mont,
        }[op]
        self._chk(fn(self.handle, _ptr(out), _ptr(a), nq, np_, npolys, _stream()))
        return out

    def scalar_mul(self, a: torch.Tensor, consts: Sequence[int], nq: int, np_: int = 0,
                   out: torch.Tensor | None = None, add: bool = False) -> torch.Tensor:
        """limb i times consts[i] (or, with add=True, plus consts[i])."""
        npolys = self._npolys(a, nq, np_, self.n)
        if len(consts) != nq + np_:
            raise BasisError("one constant per limb required")
        if out is None:
            out = torch.empty_like(a)
        fn = self.lib.hcnn_scalar_add if add else self.lib.hcnn_scalar_mul
        self._chk(fn(self.handle, _ptr(out), _ptr(a), _native.u64_array(consts), nq, np_, npolys, _stream()))
        return out

    def from_signed(self, rows: torch.Tensor, nq: int, np_: int = 0, mont: bool = False) -> torch.Tensor:
        """int64 rows [npolys, N] -> residues [npolys, nlimbs, N] (Montgomery form if mont)."""
        rows = rows.contiguous()
        npolys = rows.numel() // self.n
        out = self.empty(npolys, nq + np_, self.n)
        fn = self.lib.hcnn_from_signed_mont if mont else self.lib.hcnn_from_signed
        self._chk(fn(self.handle, _ptr(out), _ptr(rows), nq, np_, npolys, _stream()))
        return out

    def ntt_from_signed(self, rows: torch.Tensor, nq: int, mont: bool = False) -> torch.Tensor:
        """int64 rows [npolys, N] -> evaluation residues [npolys, nq, N] (Montgomery if mont), one fused pass."""
        rows = rows.contiguous()
        npolys = rows.numel() // self.n
        out = self.empty(npolys, nq, self.n)
        self._chk(self.lib.hcnn_ntt_from_signed(self.handle, _ptr(out), _ptr(rows), nq, npolys, 1 if mont else 0,
                                                _stream()))
        return out

    def automorphism(self, a: torch.Tensor, g: int, nq: int, np_: int = 0, eval_domain: bool = True,
                     out: torch.Tensor | None = None) -> torch.Tensor:
        npolys = self._npolys(a, nq, np_, self.n)
        if out is None:
            out = torch.empty_like(a)
        self._chk(self.lib.hcnn_automorphism(self.handle, _ptr(out), _ptr(a), int(g), 1 if eval_domain else 0,
                                             nq, np_, npolys, _stream()))
        return out

    def base_convert(self, a: torch.Tensor, src_mods: Sequence[int], dst_mods: Sequence[int]) -> torch.Tensor:
        """Centred FBC between arbitrary modulus-index lists (coefficient domain)."""
        ns, nt = len(src_mods), len(dst_mods)
        npolys = a.numel() // (ns * self.n)
        out = self.empty(npolys, nt, self.n)
        self._chk(self.lib.hcnn_base_convert(self.handle, _ptr(out), _ptr(a.contiguous()),
                                             _native.u32_array(src_mods), ns, _native.u32_array(dst_mods), nt,
                                             npolys, _stream()))
        return out

    # -- ckks.py level ops ----------------------------------------------------
    def ks_workspace(self, level: int, nb: int = 1) -> torch.Tensor:
        nbytes = int(self.lib.hcnn_ks_workspace_bytes_batch(self.handle, level, nb))
        return self.empty(nbytes // 8)

    def keyswitch(self, x_eval: torch.Tensor, level: int, key_b: torch.Tensor, key_a: torch.Tensor):
        out = self.empty(2, level + 1, self.n)
        ws = self.ks_workspace(level)
        self._chk(self.lib.hcnn_keyswitch(self.handle, _ptr(out[0]), _ptr(out[1]), _ptr(x_eval), level,
                                          _ptr(key_b), _ptr(key_a), _ptr(ws), _stream()))
        return out

    def _batch(self, ct: torch.Tensor, level: int) -> int:
        """entries of a ciphertext ([2,l+1,N]) or batch ([nb,2,l+1,N]) tensor"""
        if not ct.is_contiguous() or ct.shape[-3:] != (2, level + 1, self.n) or ct.dim() not in (3, 4):
            raise BasisError(f"expected a contiguous [(nb,) 2, {level + 1}, {self.n}] ciphertext tensor")
        return 1 if ct.dim() == 3 else int(ct.shape[0])

    def hmult(self, a: torch.Tensor, b: torch.Tensor, level: int, key_b: torch.Tensor,
              key_a: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """tensor + relinearise one ciphertext or a batch ([nb,2,l+1,N]; one key)."""
        nb = self._batch(a, level)
        if b.shape != a.shape or not b.is_contiguous():
            raise BasisError("hmult operands differ in shape")
        if out is None:
            out = torch.empty_like(a)
        ws = self.ks_workspace(level, nb)
        self._chk(self.lib.hcnn_hmult_batch(self.handle, _ptr(out), _ptr(a), _ptr(b), level, nb, _ptr(key_b),
                                            _ptr(key_a), _ptr(ws), _stream()))
        return out

    def rotate_hoisted(self, ct: torch.Tensor, level: int, galois: Sequence[int],
                       keys: Sequence[tuple[torch.Tensor, torch.Tensor]]) -> list[torch.Tensor]:
        """rotations of one ciphertext or a batch sharing one ModUp; outs[i] has ct's shape."""
        nb = self._batch(ct, level)
        n_rot = len(galois)
        outs = [torch.empty_like(ct) for _ in range(n_rot)]
        if n_rot == 0:
            return outs
        ws = self.empty(int(self.lib.hcnn_ks_workspace_bytes_rot(self.handle, level, nb, n_rot)) // 8)
        P = ctypes.c_void_p * n_rot
        outs_p = P(*[o.data_ptr() for o in outs])
        kb = P(*[k[0].data_ptr() for k in keys])
        ka = P(*[k[1].data_ptr() for k in keys])
        self._chk(self.lib.hcnn_rotate_hoisted_batch(self.handle, outs_p, _ptr(ct), level, nb, n_rot,
                                                     _native.u64_array(galois), kb, ka, self._key_lqs(keys),
                                                     _ptr(ws), _stream()))
        return outs

    def _key_lqs(self, keys):
        """q-limb rows of each key (a truncated key stores a prefix; see KeySet.truncate_rotations)"""
        return _native.u32_array([int(k[0].shape[-2]) - self.K for k in keys])

    def mac_terms_multi(self, cts: Sequence[torch.Tensor], masks: Sequence[Sequence[torch.Tensor | None]],
                        level: int, outs: Sequence[torch.Tensor] | None = None,
                        accumulate: bool = False) -> list[torch.Tensor]:
        """outs[g] (+)= sum_t cts[t] (.) masks[g][t] (None: no term), one ciphertext read per 4 outputs.
        A mask may be an int64 [l+1, N] Montgomery row tensor or a uint8 packed mask (pack_masks)."""
        G, T = len(masks), len(cts)
        if T and cts[0].dim() == 4:
            # image batches [B, 2, l+1, N] sharing the masks (ckks.image_batched):
            # one launch set per image
            B = int(cts[0].shape[0])
            for c in cts:
                if not c.is_contiguous() or c.shape != (B, 2, level + 1, self.n):
                    raise BasisError("mac_terms_multi image batches must be contiguous [B, 2, l+1, N]")
            if outs is None:
                outs = [self.empty(B, 2, level + 1, self.n) for _ in range(G)]
            b = 0
            while b < B:
                if b + 1 < B and self.n % 256 == 0:  # two images per launch: each mask tile read once for both
                    self._mac_multi_call([c[b] for c in cts], masks, level, [o[b] for o in outs], accumulate, 2)
                    b += 2
                else:
                    self._mac_multi_call([c[b] for c in cts], masks, level, [o[b] for o in outs], accumulate, 1)
                    b += 1
            return list(outs)
        for c in cts:
            if not c.is_contiguous() or c.shape != (2, level + 1, self.n):
                raise BasisError("mac_terms_multi ciphertexts must be contiguous [2, l+1, N]")
        if outs is None:
            outs = [self.empty(2, level + 1, self.n) for _ in range(G)]
        self._mac_multi_call(cts, masks, level, outs, accumulate, 1)
        return list(outs)

    def _mac_multi_call(self, cts, masks, level, outs, accumulate, n_images):
        """hcnn_mac_terms_multi_images; with n_images = 2, cts[t] / outs[g] are
        the first of two images stored back to back."""
        G, T = len(masks), len(cts)
        P = ctypes.c_void_p
        flat = [m for row in masks for m in row]
        ptrs = [(m.data_ptr() if m is not None else None) for m in flat]
        packed = [1 if (m is not None and m.dtype == torch.uint8) else 0 for m in flat]
        pk = (ctypes.c_ubyte * max(len(packed), 1))(*packed) if any(packed) else None
        self._chk(self.lib.hcnn_mac_terms_multi_images(self.handle, (P * max(G, 1))(*[o.data_ptr() for o in outs]),
                                                       (P * max(T, 1))(*[c.data_ptr() for c in cts]),
                                                       (P * max(G * T, 1))(*ptrs), pk, G, T, level, n_images,
                                                       1 if accumulate else 0, _stream()))

    def packed_mask_bytes(self, level: int) -> int:
        """limb 0 as u64, limbs 1..level as u32 low words + a u8 (q < 2^40) or u16 high plane"""
        return (8 + 4 * level + sum(2 if q >> 40 else 1 for q in self.q_list[1:level + 1])) * self.n

    def masks_packable(self, level: int) -> bool:
        return level < 63 and all(q < (1 << 48) for q in self.q_list[1:level + 1])  # nq <= 63 (hcnn_pack_masks)

    def pack_masks(self, rows: torch.Tensor, level: int) -> torch.Tensor:
        """Montgomery rows [k, l+1, N] -> uint8 [k, packed_mask_bytes(l)] (lossless 40/48-bit planes)."""
        rows = rows.contiguous()
        k = rows.numel() // ((level + 1) * self.n)
        out = torch.empty(k, self.packed_mask_bytes(level), dtype=torch.uint8, device=self.torch_device)
        self._chk(self.lib.hcnn_pack_masks(self.handle, _ptr(out), _ptr(rows), k, level, _stream()))
        return out

    def unpack_mask(self, packed: torch.Tensor, level: int) -> torch.Tensor:
        out = self.empty(level + 1, self.n)
        self._chk(self.lib.hcnn_unpack_mask(self.handle, _ptr(out), _ptr(packed), level, _stream()))
        return out

    # -- extended basis Q_l||P (double-hoisted linear transforms) --------------
    def rotate_hoisted_ext(self, ct: torch.Tensor, level: int, galois: Sequence[int],
                           keys: Sequence[tuple[torch.Tensor, torch.Tensor]]) -> list[torch.Tensor]:
        """rotations kept in Q_l||P (no ModDown): outs[i] [(nb,) 2, l+1+K, N]."""
        nb = self._batch(ct, level)
        shape = tuple(ct.shape[:-2]) + (level + 1 + self.K, self.n)
        outs = [self.empty(*shape) for _ in galois]
        if not outs:
            return outs
        ws = self.ks_workspace(level, nb)
        P = ctypes.c_void_p * len(outs)
        self._chk(self.lib.hcnn_rotate_hoisted_ext_batch(
            self.handle, P(*[o.data_ptr() for o in outs]), _ptr(ct), level, nb, len(outs),
            _native.u64_array(galois), P(*[k[0].data_ptr() for k in keys]), P(*[k[1].data_ptr() for k in keys]),
            self._key_lqs(keys), _ptr(ws), _stream()))
        return outs

    def mac_terms_ext(self, cts: Sequence[torch.Tensor], masks: Sequence[torch.Tensor], level: int,
                      out: torch.Tensor | None = None, accumulate: bool = False) -> torch.Tensor:
        """mac_terms over Q_l||P ciphertexts and masks (nq + K limbs)."""
        nl = level + 1 + self.K
        for c in cts:
            if not c.is_contiguous() or c.shape != cts[0].shape or c.shape[-2:] != (nl, self.n):
                raise BasisError("mac_terms_ext operands must be contiguous [(nb,) 2, l+1+K, N]")
        nb = 1 if cts[0].dim() == 3 else int(cts[0].shape[0])
        if out is None:
            out = self.empty(*cts[0].shape)
        P = ctypes.c_void_p * max(len(cts), 1)
        self._chk(self.lib.hcnn_mac_terms_ext_batch(self.handle, _ptr(out), P(*[c.data_ptr() for c in cts]),
                                                    P(*[m.data_ptr() for m in masks]), len(cts), level, nb,
                                                    1 if accumulate else 0, _stream()))
        return out

    def moddown(self, ext: torch.Tensor, level: int) -> torch.Tensor:
        """Q_l||P ciphertext(s) -> Q_l (ext's P limbs are clobbered)."""
        if not ext.is_contiguous() or ext.shape[-2:] != (level + 1 + self.K, self.n):
            raise BasisError("moddown expects a contiguous [(nb,) 2, l+1+K, N] tensor")
        nb = 1 if ext.dim() == 3 else int(ext.shape[0])
        out = self.empty(*ext.shape[:-2], level + 1, self.n)
        ws = self.ks_workspace(level, nb)
        self._chk(self.lib.hcnn_moddown_batch(self.handle, _ptr(out), _ptr(ext), level, nb, _ptr(ws), _stream()))
        return out

    def hmult_rescale(self, a: torch.Tensor, b: torch.Tensor, level: int, key_b: torch.Tensor,
                      key_a: torch.Tensor) -> torch.Tensor:
        """rescale(hmult(a, b)) with the relinearisation's ModDown and the rescale fused
        (one rounding; bootstrapping only).  -> [(nb,) 2, l, N]"""
        nb = self._batch(a, level)
        if b.shape != a.shape or not b.is_contiguous():
            raise BasisError("hmult operands differ in shape")
        if level < 1:
            raise LevelError("no limb left to rescale away")
        out = self.empty(*a.shape[:-2], level, self.n)
        ws = self.empty(int(self.lib.hcnn_hmult_rescale_workspace_bytes(self.handle, level, nb)) // 8)
        self._chk(self.lib.hcnn_hmult_rescale_batch(self.handle, _ptr(out), _ptr(a), _ptr(b), level, nb,
                                                    _ptr(key_b), _ptr(key_a), _ptr(ws), _stream()))
        return out

    def moddown_rescale(self, ext: torch.Tensor, level: int) -> torch.Tensor:
        """Q_l||P ciphertext(s) -> round(x / (P q_l)) over Q_{l-1} in one base conversion (ext clobbered)."""
        if not ext.is_contiguous() or ext.shape[-2:] != (level + 1 + self.K, self.n):
            raise BasisError("moddown_rescale expects a contiguous [(nb,) 2, l+1+K, N] tensor")
        if level < 1:
            raise LevelError("no limb left to rescale away")
        nb = 1 if ext.dim() == 3 else int(ext.shape[0])
        out = self.empty(*ext.shape[:-2], level, self.n)
        ws = self.ks_workspace(level, nb)
        self._chk(self.lib.hcnn_moddown_rescale_batch(self.handle, _ptr(out), _ptr(ext), level, nb, _ptr(ws),
                                                      _stream()))
        return out

    def mac_terms(self, cts: Sequence[torch.Tensor], masks: Sequence[torch.Tensor], level: int,
                  out: torch.Tensor | None = None, accumulate: bool = False) -> torch.Tensor:
        """out (+)= sum_t cts[t] (.) masks[t] (Montgomery masks), one fused kernel.
        cts[t] may be batches [nb,2,l+1,N] sharing the masks."""
        nb = self._batch(cts[0], level) if cts else (1 if out is None or out.dim() == 3 else out.shape[0])
        if out is None:
            out = self.empty(2, level + 1, self.n) if nb == 1 and (not cts or cts[0].dim() == 3) \
                else self.empty(nb, 2, level + 1, self.n)
        n = len(cts)
        for c in cts:
            if c.shape != cts[0].shape or not c.is_contiguous():
                raise BasisError("mac_terms ciphertexts differ in shape")
        P = ctypes.c_void_p * max(n, 1)
        cp = P(*[c.data_ptr() for c in cts])
        mp = P(*[m.data_ptr() for m in masks])
        self._chk(self.lib.hcnn_mac_terms_batch(self.handle, _ptr(out), cp, mp, n, level, nb,
                                                1 if accumulate else 0, _stream()))
        return out

    def scalar_mac(self, srcs: Sequence[torch.Tensor], consts: Sequence[Sequence[int]], level: int,
                   out: torch.Tensor | None = None, accumulate: bool = False, c0_add: int | None = None
                   ) -> torch.Tensor:
        """out[2, level+1, N] (+)= sum_t consts[t][r] * srcs[t] per limb r;
        srcs[t] are contiguous [2, >=level+1, N] ciphertext tensors (a longer
        one is read as its level-dropped prefix).  c0_add: integer added to
        every c0 (even poly) -- a plaintext constant in the same pass."""
        nq = level + 1
        lead = tuple(srcs[0].shape[:-2]) if srcs else (tuple(out.shape[:-2]) if out is not None else (2,))
        if out is None:
            out = self.empty(*lead, nq, self.n)
        n = len(srcs)
        for s in srcs:
            if not s.is_contiguous() or tuple(s.shape[:-2]) != lead or s.shape[-2] < nq:
                raise BasisError("scalar_mac sources must be contiguous [..., >=level+1, N] of one shape")
        flat = [int(v) % self.q_list[r] for row in consts for r, v in enumerate(row[:nq])]
        if any(len(row) < nq for row in consts) or len(consts) != n:
            raise BasisError("scalar_mac needs one constant per limb per source")
        P = ctypes.c_void_p * max(n, 1)
        L = ctypes.c_uint32 * max(n, 1)
        sp = P(*[s.data_ptr() for s in srcs])
        npolys = int(np.prod(lead))
        sl = L(*[s.shape[-2] for s in srcs])
        add = None if c0_add is None else _native.u64_array([int(c0_add) % self.q_list[r] for r in range(nq)])
        self._chk(self.lib.hcnn_scalar_mac(self.handle, _ptr(out), sp, sl, _native.u64_array(flat or [0]), n, nq,
                                           npolys, 1 if accumulate else 0, add, _stream()))
        return out

    def rescale(self, a: torch.Tensor, level: int) -> torch.Tensor:
        npolys = self._npolys(a, level + 1, 0, self.n)
        out = self.empty(*a.shape[:-2], level, self.n)
        ws = self.empty(npolys * self.n)
        self._chk(self.lib.hcnn_rescale(self.handle, _ptr(out), _ptr(a), level, npolys, _ptr(ws), _stream()))
        return out


def context_for(n: int, q_list: Sequence[int], p_list: Sequence[int] = (),
                device: int | None = None) -> DeviceContext:
    """The (cached) context for a chain on `device` (default: torch's current device)."""
    if device is None:
        _require_cuda(0)
        device = torch.cuda.current_device()
    key = (int(n), tuple(int(q) for q in q_list), tuple(int(p) for p in p_list), device)
    ctx = _ctx_cache.get(key)
    if ctx is None:
        with _ctx_lock:
            ctx = _ctx_cache.get(key)
            if ctx is None:
                ctx = DeviceContext(n, key[1], key[2], device)
                _ctx_cache[key] = ctx
    return ctx
