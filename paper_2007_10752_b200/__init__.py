"""B200-native bitsliced 3DES-EDE ECB (arXiv 2007.10752 hot path).

Thin ctypes binding over the C ABI in ``include/tdes.h`` / ``include/tdes_bench.h``
(``libtdes_b200.so``, built for sm_100a by ``__graft_entry__.build()``).  This
module only marshals arguments: every step of the cipher runs in the CUDA
kernels; there is no CPU fallback.  If the shared library is missing, importing
this package raises ``ImportError``.

PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TDES_LIB_PATH") or os.path.join(_HERE, "libtdes_b200.so")  # override: experiments only

TDES_OK = 0
ERRORS = {-1: "TDES_ERR_INVALID_ARG", -2: "TDES_ERR_MISALIGNED", -3: "TDES_ERR_OVERLAP",
          -4: "TDES_ERR_CUDA", -5: "TDES_ERR_WORKSPACE"}


class TdesError(RuntimeError):
    def __init__(self, code: int, what: str):
        msg = f"{what}: {ERRORS.get(code, code)} ({_lib.tdes_strerror(code).decode()})"
        if code == -4:
            msg += f", cudaError={_lib.tdes_last_cuda_error()}"
        super().__init__(msg)
        self.code = code


class TdesSchedule(ctypes.Structure):
    """Mirror of ``tdes_schedule`` (include/tdes.h)."""
    _fields_ = [("subkey", (ctypes.c_uint64 * 16) * 3),
                ("mask", ((ctypes.c_uint32 * 48) * 48) * 2)]


class DesSchedule(ctypes.Structure):
    """Mirror of ``des_schedule`` (include/tdes.h)."""
    _fields_ = [("subkey", ctypes.c_uint64 * 16),
                ("mask", ((ctypes.c_uint32 * 48) * 16) * 2)]


class KernelInfo(ctypes.Structure):
    _fields_ = [("sbox_lop3_total", ctypes.c_int), ("sbox_lop3", ctypes.c_int * 8),
                ("threads_per_cta", ctypes.c_int), ("blocks_per_thread", ctypes.c_int),
                ("min_ctas_per_sm", ctypes.c_int)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, sz, u8p = ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_uint8)
    sig = {
        "tdes_key_schedule": ([u8p, u8p, u8p, ctypes.POINTER(TdesSchedule)], ctypes.c_int),
        "tdes_ecb_encrypt": ([ctypes.POINTER(TdesSchedule), vp, vp, sz, vp], ctypes.c_int),
        "tdes_ecb_decrypt": ([ctypes.POINTER(TdesSchedule), vp, vp, sz, vp], ctypes.c_int),
        "des_key_schedule": ([u8p, ctypes.POINTER(DesSchedule)], ctypes.c_int),
        "des_ecb_encrypt": ([ctypes.POINTER(DesSchedule), vp, vp, sz, vp], ctypes.c_int),
        "des_ecb_decrypt": ([ctypes.POINTER(DesSchedule), vp, vp, sz, vp], ctypes.c_int),
        "tdes_ecb_crypt_host": ([ctypes.POINTER(TdesSchedule), ctypes.c_int, vp, vp, sz, vp, sz, sz,
                                 ctypes.POINTER(vp), ctypes.c_int], ctypes.c_int),
        "tdes_get_kernel_info": ([ctypes.POINTER(KernelInfo)], ctypes.c_int),
        "tdes_strerror": ([ctypes.c_int], ctypes.c_char_p),
        "tdes_last_cuda_error": ([], ctypes.c_int),
        "tdes_fill_splitmix64": ([vp, sz, ctypes.c_uint64, ctypes.c_uint64, vp], ctypes.c_int),
        "tdes_sum64": ([vp, sz, vp, vp], ctypes.c_int),
        "tdes_count_mismatch": ([vp, vp, sz, vp, vp], ctypes.c_int),
        "tdes_lop3_peak": ([vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                            ctypes.POINTER(ctypes.c_uint64), vp], ctypes.c_int),
        "tdes_device_geometry": ([ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)],
                                 ctypes.c_int),
        "tdes_paper_ecb": ([vp, vp, vp, sz, ctypes.c_int, vp, sz, vp], ctypes.c_int),
        "tdes_ecb_crypt_mode": ([ctypes.POINTER(TdesSchedule), ctypes.c_int, vp, vp, sz, ctypes.c_int, vp],
                                ctypes.c_int),
        "tdes_fold_operands": ([ctypes.POINTER(TdesSchedule), ctypes.c_int, vp, sz, ctypes.POINTER(sz),
                                ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    }
    for name, (argtypes, restype) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = restype
    return lib


_lib = _load()

# Every symbol include/tdes.h and include/tdes_bench.h declare.
EXPORTS = ("tdes_key_schedule", "tdes_ecb_encrypt", "tdes_ecb_decrypt", "des_key_schedule",
           "des_ecb_encrypt", "des_ecb_decrypt", "tdes_ecb_crypt_host", "tdes_get_kernel_info",
           "tdes_strerror", "tdes_last_cuda_error", "tdes_fill_splitmix64", "tdes_sum64",
           "tdes_count_mismatch", "tdes_lop3_peak", "tdes_device_geometry", "tdes_paper_ecb",
           "tdes_ecb_crypt_mode", "tdes_fold_operands")

MODE_AUTO, MODE_THROUGHPUT, MODE_SPLIT, MODE_DEVKEYS = 0, 1, 2, 3


def _check(rc: int, what: str):
    if rc != TDES_OK:
        raise TdesError(rc, what)


def _key_bytes(k) -> bytes:
    if isinstance(k, str):
        s = k.strip()
        if len(s) != 16:
            raise ValueError(f"key must be 16 hex digits, got {len(s)}")
        try:
            k = bytes.fromhex(s)
        except ValueError as e:
            raise ValueError(f"key is not hex: {s!r}") from e
    k = bytes(k)
    if len(k) != 8:
        raise ValueError("key must be 8 bytes")
    return k


def _u8(b: bytes):
    return (ctypes.c_uint8 * 8).from_buffer_copy(b)


def key_schedule(k1, k2, k3) -> TdesSchedule:
    """3DES key schedule (bytes or 16-hex-digit strings; FIPS bit 1 = MSB of byte 0)."""
    s = TdesSchedule()
    _check(_lib.tdes_key_schedule(_u8(_key_bytes(k1)), _u8(_key_bytes(k2)), _u8(_key_bytes(k3)),
                                  ctypes.byref(s)), "tdes_key_schedule")
    return s


def des_key_schedule(k) -> DesSchedule:
    s = DesSchedule()
    _check(_lib.des_key_schedule(_u8(_key_bytes(k)), ctypes.byref(s)), "des_key_schedule")
    return s


def subkeys(s: TdesSchedule) -> list[list[int]]:
    return [[int(s.subkey[k][r]) for r in range(16)] for k in range(3)]


# Per-call host cost matters for small launches (a C1 launch is ~12 us of device
# time): the public torch.cuda.current_stream() and torch.cuda.device() cost ~2.2 and
# ~1.5 us per call (tools/exp/binding_overhead.py), so the binding uses torch's raw
# accessors when they exist and enters the device context only when the tensor is
# not on the current device.
_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_GET_DEVICE = getattr(torch._C, "_cuda_getDevice", None)


def _launch(device: torch.device, call, stream):
    """Run ``call(stream_handle)`` with ``device`` current (the C ABI launches on the
    current device) on ``stream`` (default: that device's current stream)."""
    idx = device.index
    h = _RAW_STREAM(idx) if stream is None and _RAW_STREAM is not None else _stream_handle(stream, device)
    if _GET_DEVICE is not None and _GET_DEVICE() == idx:
        return call(h)
    with torch.cuda.device(device):
        return call(h)


def _stream_handle(stream, device=None) -> int:
    """The raw handle of `stream` (default: the current stream of `device`).

    The C ABI launches on the *current* device, so every call below runs inside
    ``torch.cuda.device(x.device)``; an explicit stream must live on that device."""
    if stream is None:
        return int(torch.cuda.current_stream(device).cuda_stream)
    if device is not None and stream.device != torch.device(device):
        raise ValueError(f"stream is on {stream.device}, the tensors on {device}")
    return int(stream.cuda_stream)


def _prep(x: torch.Tensor, out):
    if not x.is_cuda:
        raise ValueError("input must be a CUDA tensor (use ecb_crypt_host for host buffers)")
    if not x.is_contiguous() or x.dtype != torch.uint8 or x.numel() % 8:
        raise ValueError("input must be a contiguous uint8 CUDA tensor with numel % 8 == 0")
    if out is None:
        out = torch.empty_like(x)
    if not (out.is_cuda and out.is_contiguous() and out.dtype == torch.uint8 and out.numel() == x.numel()):
        raise ValueError("out must be a contiguous uint8 CUDA tensor of the input's size")
    if out.device != x.device:
        raise ValueError(f"out is on {out.device}, the input on {x.device}")
    return out


def _crypt(fn, sched, x, out, stream, what):
    out = _prep(x, out)
    _check(_launch(x.device, lambda h: fn(ctypes.byref(sched), x.data_ptr(), out.data_ptr(), x.numel() // 8, h),
                   stream), what)
    return out


def ecb_encrypt(x: torch.Tensor, sched: TdesSchedule, out: torch.Tensor | None = None, stream=None):
    """3DES-EDE ECB encrypt of a uint8 CUDA tensor (numel % 8 == 0) on ``stream``."""
    return _crypt(_lib.tdes_ecb_encrypt, sched, x, out, stream, "tdes_ecb_encrypt")


def ecb_decrypt(x: torch.Tensor, sched: TdesSchedule, out: torch.Tensor | None = None, stream=None):
    return _crypt(_lib.tdes_ecb_decrypt, sched, x, out, stream, "tdes_ecb_decrypt")


def des_ecb_encrypt(x, sched: DesSchedule, out=None, stream=None):
    """Single DES (the K1=K2=K3 case, 16 rounds) -- never reported as 3DES."""
    return _crypt(_lib.des_ecb_encrypt, sched, x, out, stream, "des_ecb_encrypt")


def des_ecb_decrypt(x, sched: DesSchedule, out=None, stream=None):
    return _crypt(_lib.des_ecb_decrypt, sched, x, out, stream, "des_ecb_decrypt")


def ecb_crypt_mode(x: torch.Tensor, sched: TdesSchedule, mode: int, decrypt=False, out=None, stream=None):
    """3DES ECB with an explicit kernel choice (MODE_AUTO / MODE_THROUGHPUT / MODE_SPLIT / MODE_DEVKEYS)."""
    out = _prep(x, out)
    _check(_launch(x.device, lambda h: _lib.tdes_ecb_crypt_mode(ctypes.byref(sched), int(bool(decrypt)), x.data_ptr(),
                                                               out.data_ptr(), x.numel() // 8, mode, h), stream),
           "tdes_ecb_crypt_mode")
    return out


def ecb_encrypt_ptr(sched: TdesSchedule, in_ptr: int, out_ptr: int, nblocks: int, stream_handle: int = 0):
    """Raw-pointer form of tdes_ecb_encrypt (device pointers)."""
    _check(_lib.tdes_ecb_encrypt(ctypes.byref(sched), in_ptr, out_ptr, nblocks, stream_handle),
           "tdes_ecb_encrypt")


def ecb_decrypt_ptr(sched: TdesSchedule, in_ptr: int, out_ptr: int, nblocks: int, stream_handle: int = 0):
    _check(_lib.tdes_ecb_decrypt(ctypes.byref(sched), in_ptr, out_ptr, nblocks, stream_handle),
           "tdes_ecb_decrypt")


class HostPipeline:
    """End-to-end host->device->host 3DES (tdes_ecb_crypt_host) with its own workspace and streams."""

    def __init__(self, chunk_blocks: int = 1 << 22, nstreams: int = 3, device=None):
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.chunk_blocks = int(chunk_blocks) + (int(chunk_blocks) & 1)
        self.streams = [torch.cuda.Stream(device=self.device) for _ in range(nstreams)]
        self.workspace = torch.empty(nstreams * self.chunk_blocks * 8, dtype=torch.uint8, device=self.device)
        self._handles = (ctypes.c_void_p * nstreams)(*[s.cuda_stream for s in self.streams])

    def run(self, sched: TdesSchedule, host_in: torch.Tensor, host_out: torch.Tensor, decrypt=False):
        for t in (host_in, host_out):
            if t.is_cuda or not t.is_contiguous() or t.dtype != torch.uint8:
                raise ValueError("host buffers must be contiguous uint8 CPU tensors")
        if host_in.numel() % 8 or host_out.numel() != host_in.numel():
            raise ValueError("size mismatch or not a whole number of blocks")
        with torch.cuda.device(self.device):   # the C ABI launches on the current device
            # order the caller's current stream before ours (inputs may be produced on it)
            cur = torch.cuda.current_stream(self.device)
            for s in self.streams:
                s.wait_stream(cur)
            _check(_lib.tdes_ecb_crypt_host(ctypes.byref(sched), int(bool(decrypt)), host_in.data_ptr(),
                                            host_out.data_ptr(), host_in.numel() // 8,
                                            self.workspace.data_ptr(), self.workspace.numel(),
                                            self.chunk_blocks, self._handles, len(self.streams)),
                   "tdes_ecb_crypt_host")
        return host_out


def kernel_info() -> KernelInfo:
    k = KernelInfo()
    _check(_lib.tdes_get_kernel_info(ctypes.byref(k)), "tdes_get_kernel_info")
    return k


def fold_operands(sched: TdesSchedule, decrypt=False) -> dict:
    """Host-side key operands of the 3DES throughput kernel (mask folding; no GPU needed).

    Returns numpy uint32 arrays s, k [48, stride], d [48, dstride], fix_s, fix_k
    [3, dstride], fin_s, fin_k [64] and the geometry (include/tdes_bench.h)."""
    import numpy as np
    words = ctypes.c_size_t()
    geom = (ctypes.c_int * 4)()
    _lib.tdes_fold_operands(ctypes.byref(sched), int(bool(decrypt)), None, 0, ctypes.byref(words), geom)
    buf = np.zeros(words.value, dtype=np.uint32)
    _check(_lib.tdes_fold_operands(ctypes.byref(sched), int(bool(decrypt)), buf.ctypes.data, buf.size,
                                   ctypes.byref(words), geom), "tdes_fold_operands")
    slots, stride, nfree, dstride = list(geom)
    out, o = {"slots": slots, "stride": stride, "nfree": nfree, "dstride": dstride}, 0
    for name, shape in (("s", (48, stride)), ("k", (48, stride)), ("d", (48, dstride)), ("fix_s", (3, dstride)),
                        ("fix_k", (3, dstride)), ("fin_s", (64,)), ("fin_k", (64,))):
        n = int(np.prod(shape))
        out[name] = buf[o:o + n].reshape(shape)
        o += n
    return out


def device_geometry() -> tuple[int, int]:
    a, b = ctypes.c_int(), ctypes.c_int()
    _check(_lib.tdes_device_geometry(ctypes.byref(a), ctypes.byref(b)), "tdes_device_geometry")
    return a.value, b.value


class PaperBaseline:
    """The paper's own kernel design on this GPU (include/tdes_paper.h; comparison only).

    Key-generation kernel (3 CTAs x 56 threads) + three launches of a
    64-thread-CTA-per-block, char-per-bit crypt kernel (§IV).
    """

    def __init__(self, k1, k2, k3, device=None):
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        keys = _key_bytes(k1) + _key_bytes(k2) + _key_bytes(k3)
        self.keys = torch.tensor(list(keys), dtype=torch.uint8, device=dev)
        self.workspace = torch.empty(3 * 16 * 48, dtype=torch.uint8, device=dev)

    def run(self, x: torch.Tensor, decrypt=False, out=None, stream=None):
        out = _prep(x, out)
        if x.device != self.keys.device:
            raise ValueError(f"input on {x.device}, PaperBaseline built for {self.keys.device}")
        with torch.cuda.device(x.device):
            _check(_lib.tdes_paper_ecb(self.keys.data_ptr(), x.data_ptr(), out.data_ptr(), x.numel() // 8,
                                       int(bool(decrypt)), self.workspace.data_ptr(), self.workspace.numel(),
                                       _stream_handle(stream, x.device)), "tdes_paper_ecb")
        return out


# ------------------------------------------------------ bench helpers -----

def fill_splitmix64(x: torch.Tensor, first_index: int = 0, seed: int = 20071075, stream=None):
    """Synthetic plaintext (DESIGN.md input recipe) generated on the device."""
    if not (x.is_cuda and x.is_contiguous() and x.numel() % 8 == 0):
        raise ValueError("x must be a contiguous CUDA tensor of whole 8-byte blocks")
    with torch.cuda.device(x.device):
        _check(_lib.tdes_fill_splitmix64(x.data_ptr(), x.numel() // 8, first_index, seed,
                                         _stream_handle(stream, x.device)), "tdes_fill_splitmix64")
    return x


def sum64(x: torch.Tensor, stream=None) -> int:
    """Sum of the little-endian uint64 blocks mod 2^64 (synchronizes)."""
    if not (x.is_cuda and x.is_contiguous()):
        raise ValueError("x must be a contiguous CUDA tensor")
    with torch.cuda.device(x.device):
        res = torch.zeros(1, dtype=torch.int64, device=x.device)
        _check(_lib.tdes_sum64(x.data_ptr(), x.numel() // 8, res.data_ptr(), _stream_handle(stream, x.device)),
               "tdes_sum64")
    return int(res.item()) & ((1 << 64) - 1)


def count_mismatch(a: torch.Tensor, b: torch.Tensor, stream=None) -> int:
    if not (a.is_cuda and a.is_contiguous() and b.is_contiguous()) or a.device != b.device \
            or a.numel() != b.numel():
        raise ValueError("a and b must be contiguous CUDA tensors of one size on one device")
    with torch.cuda.device(a.device):
        res = torch.zeros(1, dtype=torch.int64, device=a.device)
        _check(_lib.tdes_count_mismatch(a.data_ptr(), b.data_ptr(), a.numel() // 8, res.data_ptr(),
                                        _stream_handle(stream, a.device)), "tdes_count_mismatch")
    return int(res.item())


def lop3_peak_launch(sink: torch.Tensor, grid: int, cta: int, iters: int, stream=None) -> int:
    ops = ctypes.c_uint64()
    with torch.cuda.device(sink.device):
        _check(_lib.tdes_lop3_peak(sink.data_ptr(), grid, cta, iters, ctypes.byref(ops),
                                   _stream_handle(stream, sink.device)), "tdes_lop3_peak")
    return ops.value
