"""B200-native batched NTT engine (D. Harvey, arXiv:1205.2926) -- Python binding.

Thin ctypes marshalling over the C ABI in ``include/ntt_b200.h``; every step of
the transform runs in the CUDA kernels of ``libntt_b200.so``.  There is no CPU
fallback: importing this module without the built library raises.  PyTorch is
used only for device memory and streams (tensors are passed as raw pointers).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# NTT_B200_LIB: a library path, or "audit" for the range-audit debug build (libntt_b200_audit.so)
_LIB_ENV = os.environ.get("NTT_B200_LIB", "")
LIB_PATH = (os.path.join(_HERE, "libntt_b200_audit.so") if _LIB_ENV == "audit"
            else (_LIB_ENV or os.path.join(_HERE, "libntt_b200.so")))

NTT_SCALE_INV_L = 1
NTT_OP_FORWARD = 1
NTT_OP_INVERSE = 2

_STATUS = {
    0: "NTT_OK", -1: "NTT_ERR_ARG", -2: "NTT_ERR_MODULUS", -3: "NTT_ERR_ROOT", -4: "NTT_ERR_LENGTH",
    -5: "NTT_ERR_WORD", -6: "NTT_ERR_CUDA", -7: "NTT_ERR_NOMEM", -8: "NTT_ERR_UNSUPPORTED", -9: "NTT_ERR_RANGE",
}


class NttError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        name = _STATUS.get(status, str(status))
        msg = f"{where}: {name} ({_lib.ntt_status_str(status).decode()})"
        if status == -6:
            msg += f" [{_lib.ntt_last_cuda_error().decode()}]"
        super().__init__(msg)


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("p", ctypes.c_uint64), ("omega", ctypes.c_uint64), ("omega_inv", ctypes.c_uint64), ("L_inv", ctypes.c_uint64),
        ("ell", ctypes.c_uint), ("log2_beta", ctypes.c_uint), ("word_bytes", ctypes.c_uint),
        ("n_passes", ctypes.c_uint), ("pass_log2", ctypes.c_uint * 4), ("device", ctypes.c_int),
    ]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, u64, uint, sz, c_int = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint, ctypes.c_size_t, ctypes.c_int
    sig = {
        "ntt_plan_create": [ctypes.POINTER(vp), u64, u64, uint, uint, c_int],
        "ntt_plan_create_ex": [ctypes.POINTER(vp), u64, u64, uint, uint, c_int, uint],
        "ntt_plan_destroy": [vp],
        "ntt_plan_info": [vp, ctypes.POINTER(PlanInfo)],
        "ntt_forward": [vp, vp, sz, vp],
        "ntt_inverse": [vp, vp, sz, vp],
        "ntt_transform_pass": [vp, vp, sz, uint, uint, vp],
        "ntt_pointwise_mul": [vp, vp, vp, vp, sz, uint, vp],
        "ntt_cyclic_convolve": [vp, vp, vp, sz, vp],
        "ntt_plan_twiddles": [vp, vp, vp],
        "ntt_fourstep_cols": [vp, uint, vp, uint, uint, vp],
        "ntt_fourstep_rows": [vp, uint, vp, vp, uint, uint, vp],
        "ntt_fourstep_cols_inv": [vp, uint, vp, uint, uint, vp],
        "ntt_fourstep_cols_p2p": [vp, uint, vp, ctypes.POINTER(u64), uint, uint, vp],
        "ntt_fourstep_rows_inv_p2p": [vp, uint, vp, ctypes.POINTER(u64), uint, uint, vp],
        "ntt_fourstep_rows_inv": [vp, uint, vp, vp, uint, uint, vp],
        "ntt_block_transpose": [vp, vp, sz, sz, sz, uint, vp],
        "ntt_crt3": [vp, vp, vp, vp, sz, uint, uint, uint, vp],
        "ntt_synth_uniform": [vp, sz, uint, u64, u64, u64, u64, uint, vp],
        "ntt_debug_butterfly": [vp, c_int, vp, vp, vp, vp, sz, vp],
        "ntt_execute_host": [vp, uint, vp, vp, sz, vp, sz, vp],
        "ntt_calibrate_butterfly": [uint, u64, u64, u64, uint, vp, ctypes.POINTER(u64), vp],
        "ntt_audit_counts": [c_int, ctypes.POINTER(u64)],
        "ntt_plan_table": [vp, uint, uint, vp, sz, ctypes.POINTER(sz)],
        "ntt_audit_reset": [c_int, c_int],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = c_int
    lib.ntt_status_str.argtypes = [c_int]
    lib.ntt_status_str.restype = ctypes.c_char_p
    lib.ntt_last_cuda_error.restype = ctypes.c_char_p
    lib.ntt_last_launch_count.restype = uint
    lib.ntt_set_range_checks.argtypes = [uint]
    lib.ntt_set_range_checks.restype = uint
    lib.ntt_abi_version.restype = uint
    lib.ntt_build_flags.restype = uint
    return lib


_lib = _load()

EXPORTED = (
    "ntt_plan_create", "ntt_plan_create_ex", "ntt_plan_destroy", "ntt_plan_info", "ntt_forward", "ntt_inverse", "ntt_transform_pass", "ntt_pointwise_mul",
    "ntt_cyclic_convolve", "ntt_execute_host", "ntt_plan_twiddles", "ntt_plan_table", "ntt_fourstep_cols", "ntt_fourstep_rows",
    "ntt_fourstep_cols_inv", "ntt_fourstep_rows_inv", "ntt_fourstep_cols_p2p",
    "ntt_fourstep_rows_inv_p2p", "ntt_block_transpose", "ntt_crt3", "ntt_synth_uniform",
    "ntt_debug_butterfly", "ntt_calibrate_butterfly", "ntt_set_range_checks", "ntt_build_flags", "ntt_audit_counts", "ntt_audit_reset", "ntt_last_launch_count", "ntt_status_str", "ntt_last_cuda_error", "ntt_abi_version",
)


def lib() -> ctypes.CDLL:
    return _lib


def _check(status: int, where: str):
    if status != 0:
        raise NttError(status, where)


def _ptr(t) -> int:
    """Device pointer of a torch tensor (or an int pointer)."""
    if t is None:
        return 0
    if isinstance(t, int):
        return t
    return t.data_ptr()


try:  # the current stream's raw handle without building a torch.cuda.Stream object (~1 us per call)
    import torch as _torch
    _raw_stream = _torch._C._cuda_getCurrentRawStream
    _cur_dev = _torch._C._cuda_getDevice
except Exception:  # no torch build with CUDA: the legacy default stream
    _raw_stream = _cur_dev = None


def _stream(stream) -> int:
    if stream is None:
        if _raw_stream is None:
            return 0
        try:
            return _raw_stream(_cur_dev())
        except Exception:  # no device: legacy default stream
            return 0
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def set_range_checks(on: bool) -> bool:
    """ntt_set_range_checks: debugging mode validating transform inputs (returns the previous setting)."""
    return bool(_lib.ntt_set_range_checks(1 if on else 0))


def audit_build() -> bool:
    """True when the loaded library is the range-audit debug build (NTT_B200_LIB=audit)."""
    return bool(_lib.ntt_build_flags() & 1)


def audit_counts(device: int = 0) -> int:
    """ntt_audit_counts: range violations counted since the last audit_reset (audit build only)."""
    v = ctypes.c_uint64()
    _check(_lib.ntt_audit_counts(device, ctypes.byref(v)), "ntt_audit_counts")
    return int(v.value)


def audit_reset(device: int = 0, mutate: bool = False, stress: bool = False):
    """ntt_audit_reset: zero the counters; mutate drops Algorithm 3's "+2p"; stress adds per-warp random
    delays at every round (audit build only)."""
    _check(_lib.ntt_audit_reset(device, (1 if mutate else 0) | (2 if stress else 0)), "ntt_audit_reset")


def last_launch_count() -> int:
    return int(_lib.ntt_last_launch_count())


class Plan:
    """ntt_plan_create(p, omega, ell, log2_beta, device) (include/ntt_b200.h)."""

    def __init__(self, p: int, omega: int, ell: int, log2_beta: int, device: int = 0, butterfly: int = 3):
        h = ctypes.c_void_p()
        _check(_lib.ntt_plan_create_ex(ctypes.byref(h), p, omega, ell, log2_beta, device, butterfly),
               "ntt_plan_create_ex")
        self.butterfly = butterfly
        self._h = h
        self.p, self.omega, self.ell, self.log2_beta, self.device = p, omega, ell, log2_beta, device
        self.L = 1 << ell
        self.word_bytes = log2_beta // 8

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.ntt_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def info(self) -> PlanInfo:
        out = PlanInfo()
        _check(_lib.ntt_plan_info(self._h, ctypes.byref(out)), "ntt_plan_info")
        return out

    def _batch(self, x, batch):
        if batch is not None:
            return batch
        n = x.numel()
        if n % self.L:
            raise ValueError(f"buffer of {n} words is not a multiple of L = {self.L}")
        return n // self.L

    def forward(self, x, batch=None, stream=None):
        _check(_lib.ntt_forward(self._h, _ptr(x), self._batch(x, batch), _stream(stream)), "ntt_forward")
        return x

    def inverse(self, x, batch=None, stream=None):
        _check(_lib.ntt_inverse(self._h, _ptr(x), self._batch(x, batch), _stream(stream)), "ntt_inverse")
        return x

    def transform_pass(self, x, pass_index, inverse=False, batch=None, stream=None):
        """One kernel pass of the schedule (ntt_transform_pass): forward passes 0..n-1 in order
        equal forward(); inverse passes n-1..0 in order equal inverse()."""
        _check(_lib.ntt_transform_pass(self._h, _ptr(x), self._batch(x, batch), 1 if inverse else 0, pass_index,
                                       _stream(stream)), "ntt_transform_pass")
        return x

    def pointwise_mul(self, c, a, b, batch=None, scale_inv_L=False, stream=None):
        flags = NTT_SCALE_INV_L if scale_inv_L else 0
        _check(_lib.ntt_pointwise_mul(self._h, _ptr(c), _ptr(a), _ptr(b), self._batch(a, batch), flags,
                                      _stream(stream)), "ntt_pointwise_mul")
        return c

    def cyclic_convolve(self, a, b, batch=None, stream=None):
        _check(_lib.ntt_cyclic_convolve(self._h, _ptr(a), _ptr(b), self._batch(a, batch), _stream(stream)),
               "ntt_cyclic_convolve")
        return a

    def execute_host(self, ops, host_in, host_out, dev_buf, batch=None, stream=None):
        """ntt_execute_host: host (pinned) tensors in/out, device scratch dev_buf."""
        nb = dev_buf.numel() * dev_buf.element_size()
        _check(_lib.ntt_execute_host(self._h, ops, _ptr(host_in), _ptr(host_out), self._batch(host_in, batch),
                                     _ptr(dev_buf), nb, _stream(stream)), "ntt_execute_host")
        return host_out

    def twiddles(self):
        """(W, W') host arrays of the forward table, e < L/2 (numpy)."""
        import numpy as np
        dt = np.uint64 if self.word_bytes == 8 else np.uint32
        half = self.L // 2
        W = np.zeros(max(half, 1), dtype=dt)
        Wp = np.zeros(max(half, 1), dtype=dt)
        _check(_lib.ntt_plan_twiddles(self._h, W.ctypes.data, Wp.ctypes.data), "ntt_plan_twiddles")
        return W[:half], Wp[:half]

    def table(self, kind: int, pass_index: int = 0):
        """ntt_plan_table: a device-resident twiddle table as a numpy array, shape (n, 2) of
        (W, W') pairs (or (n,) one-word Montgomery entries for Algorithm 5 forward tables)."""
        import numpy as np
        nb = ctypes.c_size_t()
        _check(_lib.ntt_plan_table(self._h, kind, pass_index, None, 0, ctypes.byref(nb)), "ntt_plan_table")
        buf = np.empty(nb.value // self.word_bytes, dtype=np.uint64 if self.word_bytes == 8 else np.uint32)
        _check(_lib.ntt_plan_table(self._h, kind, pass_index, buf.ctypes.data, nb.value, ctypes.byref(nb)),
               "ntt_plan_table")
        mont = self.butterfly == 5 and kind in (0, 1, 2, 3)
        return buf.astype(np.uint64) if mont else buf.astype(np.uint64).reshape(-1, 2)

    def fourstep_cols(self, ell1, x_shard, rank, world, stream=None):
        _check(_lib.ntt_fourstep_cols(self._h, ell1, _ptr(x_shard), rank, world, _stream(stream)),
               "ntt_fourstep_cols")

    def fourstep_rows(self, ell1, recv, out, rank, world, stream=None):
        _check(_lib.ntt_fourstep_rows(self._h, ell1, _ptr(recv), _ptr(out), rank, world, _stream(stream)),
               "ntt_fourstep_rows")

    def fourstep_cols_p2p(self, ell1, x_shard, peer_ptrs, rank, world, stream=None):
        """ntt_fourstep_cols_p2p: peer_ptrs = the `world` receive-buffer device addresses (ints)."""
        arr = (ctypes.c_uint64 * len(peer_ptrs))(*[int(q) for q in peer_ptrs])
        _check(_lib.ntt_fourstep_cols_p2p(self._h, ell1, _ptr(x_shard), arr, rank, world, _stream(stream)),
               "ntt_fourstep_cols_p2p")

    def fourstep_rows_inv_p2p(self, ell1, x_rows, peer_ptrs, rank, world, stream=None):
        """ntt_fourstep_rows_inv_p2p: peer_ptrs = the `world` receive-buffer device addresses (ints)."""
        arr = (ctypes.c_uint64 * len(peer_ptrs))(*[int(q) for q in peer_ptrs])
        _check(_lib.ntt_fourstep_rows_inv_p2p(self._h, ell1, _ptr(x_rows), arr, rank, world, _stream(stream)),
               "ntt_fourstep_rows_inv_p2p")

    def fourstep_rows_inv(self, ell1, x_rows, send, rank, world, stream=None):
        _check(_lib.ntt_fourstep_rows_inv(self._h, ell1, _ptr(x_rows), _ptr(send), rank, world, _stream(stream)),
               "ntt_fourstep_rows_inv")

    def fourstep_cols_inv(self, ell1, x_shard, rank, world, stream=None):
        _check(_lib.ntt_fourstep_cols_inv(self._h, ell1, _ptr(x_shard), rank, world, _stream(stream)),
               "ntt_fourstep_cols_inv")

    def debug_butterfly(self, alg, W, Wp, X, Y, stream=None):
        _check(_lib.ntt_debug_butterfly(self._h, alg, _ptr(W), _ptr(Wp), _ptr(X), _ptr(Y), X.numel(),
                                        _stream(stream)), "ntt_debug_butterfly")


def calibrate_butterfly(log2_beta: int, p: int, W: int, Wp: int, iters: int, sink, stream=None) -> int:
    """Launch the register-only Alg. 3 loop; returns the number of butterflies it performs."""
    n = ctypes.c_uint64()
    _check(_lib.ntt_calibrate_butterfly(log2_beta, p, W, Wp, iters, _ptr(sink), ctypes.byref(n), _stream(stream)),
           "ntt_calibrate_butterfly")
    return int(n.value)


def block_transpose(dst, src, n0: int, n1: int, n2: int, stream=None):
    """ntt_block_transpose: dst[j][i][k] = src[i][j][k] (device tensors of 4- or 8-byte words)."""
    _check(_lib.ntt_block_transpose(_ptr(dst), _ptr(src), n0, n1, n2, src.element_size(), _stream(stream)),
           "ntt_block_transpose")
    return dst


def crt3(out, r0, r1, r2, primes, stream=None):
    """ntt_crt3: out (uint64 device tensor of 2n words: lo, hi per coefficient) = the CRT lift of the
    three uint32 residue tensors r0, r1, r2 (n words each) modulo primes = (p0, p1, p2)."""
    n = r0.numel()
    if r1.numel() != n or r2.numel() != n or out.numel() < 2 * n:
        raise ValueError("crt3: size mismatch")
    _check(_lib.ntt_crt3(_ptr(out), _ptr(r0), _ptr(r1), _ptr(r2), n, *primes, _stream(stream)), "ntt_crt3")
    return out


def synth_uniform(x, seed: int, tensor_id: int, start: int = 0, bound: int = 0, bits: int = 0, stream=None):
    """Fill device tensor x with the seeded stream of synth/__init__.py (same definition)."""
    wb = x.element_size()
    _check(_lib.ntt_synth_uniform(_ptr(x), x.numel(), wb, seed, tensor_id, start, bound, bits, _stream(stream)),
           "ntt_synth_uniform")
    return x
