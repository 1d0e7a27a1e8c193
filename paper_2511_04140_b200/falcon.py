"""ctypes binding of the C ABI in include/falcon_b200.h (libfalcon_b200.so).

This is plumbing for tests, bench and Python users; the product is the CUDA library
behind it.  There is no CPU fallback: if the shared library is missing or no GPU is
present, the calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._build import LIB

F64, F32 = 0, 1
DEFAULT_CHUNK_N = 1025
DEFAULT_BATCH_VALUES = 1025 * 1024 * 4  # pipeline.hpp:71-72

OK, ERR_INVALID, ERR_CORRUPT, ERR_IO, ERR_CUDA, ERR_CALLBACK, ERR_CAPACITY, ERR_UNSUPPORTED = range(8)
STAGE_COMPRESS, STAGE_STORE, STAGE_DECODE = 0, 1, 2
KINDS = {"walk": 0, "decimal": 1, "signflip": 2, "outlier": 3, "bits": 4, "mixed": 5, "field": 6}

EXPORTED = [
    "falcon_abi_version", "falcon_last_error", "falcon_default_options", "falcon_ctx_create",
    "falcon_ctx_destroy", "falcon_max_encoded_chunk_size", "falcon_compress_bound",
    "falcon_write_header", "falcon_read_header", "falcon_compress_device",
    "falcon_compress_device_async", "falcon_decompress_device", "falcon_decompress_device_async",
    "falcon_decompress_device_chained", "falcon_archive_index", "falcon_decompress_device_range",
    "falcon_ctx_sync", "falcon_compress_stream", "falcon_decompress_stream", "falcon_compress_host",
    "falcon_decompress_host", "falcon_compress_chunk", "falcon_decompress_chunk", "falcon_synth_fill",
    "falcon_ctx_set_kernel_events", "falcon_selftest_dp", "falcon_selftest_div",
    "falcon_synth_fill_at", "falcon_synth_device", "falcon_compress_host_multi", "falcon_decompress_host_multi",
    "falcon_compress_device_frames", "falcon_compress_file", "falcon_decompress_file",
]


class FalconError(RuntimeError):
    """falcon::error (error.hpp:8-10)."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status, self.message = status, message


class CorruptError(FalconError):
    """falcon::corrupt_error (error.hpp:13-15)."""


class CudaError(FalconError):
    pass


STAGE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.c_uint, C.c_uint64)
READ_FN = C.CFUNCTYPE(C.c_int64, C.c_void_p, C.c_void_p, C.c_uint64)
STORE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64)
PUT_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64)


class PipelineOptions(C.Structure):
    """falcon_pipeline_options == pipeline_options (pipeline.hpp:70-79)."""
    _fields_ = [("chunk_n", C.c_uint32), ("batch_values", C.c_uint64), ("n_streams", C.c_uint32),
                ("workers", C.c_uint32), ("stage_delay", STAGE_FN), ("stage_delay_user", C.c_void_p)]


class PipelineStats(C.Structure):
    _fields_ = [("batches", C.c_uint64), ("values", C.c_uint64), ("blocking_waits", C.c_uint64)]


class ArchiveInfo(C.Structure):
    _fields_ = [("precision", C.c_uint8), ("chunk_n", C.c_uint32), ("batch_values", C.c_uint64),
                ("total_values", C.c_uint64), ("batch_count", C.c_uint64)]


class SynthSpec(C.Structure):
    _fields_ = [("kind", C.c_int), ("decimal_places", C.c_int), ("seed", C.c_uint64),
                ("max_step_units", C.c_int), ("outlier_period", C.c_uint64),
                ("outlier_units", C.c_int64), ("block", C.c_uint32)]


_lib = None


def load() -> C.CDLL:
    """Load libfalcon_b200.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    # FALCON_B200_LIB selects an alternative in-tree build (A/B kernel experiments,
    # scripts/ab.sh); the default is the package's own library
    path = os.environ.get("FALCON_B200_LIB", LIB)
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(path)
    vp, u64, u32, i32 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
    L.falcon_last_error.restype = C.c_char_p
    L.falcon_ctx_create.argtypes = [i32, C.POINTER(vp)]
    L.falcon_ctx_destroy.argtypes = [vp]
    L.falcon_max_encoded_chunk_size.restype = u64
    L.falcon_max_encoded_chunk_size.argtypes = [i32, u32]
    L.falcon_compress_bound.restype = u64
    L.falcon_compress_bound.argtypes = [i32, u64, u32, u64]
    L.falcon_write_header.argtypes = [C.POINTER(ArchiveInfo), vp]
    L.falcon_read_header.argtypes = [vp, u64, C.POINTER(ArchiveInfo)]
    L.falcon_compress_device.argtypes = [vp, i32, vp, u64, u32, u64, vp, u64, C.POINTER(u64), vp]
    L.falcon_compress_device_async.argtypes = [vp, i32, vp, u64, u32, u64, vp, u64, vp, vp]
    L.falcon_decompress_device.argtypes = [vp, i32, vp, u64, vp, u64, C.POINTER(u64), vp]
    L.falcon_decompress_device_async.argtypes = [vp, i32, vp, u64, C.POINTER(ArchiveInfo), vp, u64, vp]
    L.falcon_decompress_device_chained.argtypes = [vp, i32, vp, vp, C.POINTER(ArchiveInfo), vp, u64, vp]
    L.falcon_archive_index.argtypes = [vp, vp, u64, C.POINTER(ArchiveInfo), vp, vp]
    L.falcon_decompress_device_range.argtypes = [vp, i32, vp, C.POINTER(ArchiveInfo), C.POINTER(u64), u64, u64,
                                                 vp, u64, C.POINTER(u64), vp]
    L.falcon_ctx_sync.argtypes = [vp, vp]
    L.falcon_ctx_set_kernel_events.argtypes = [vp, vp, vp, vp, vp]
    L.falcon_selftest_dp.argtypes = [vp, i32, vp, u64, i32, vp, vp, vp, vp, vp]
    L.falcon_selftest_div.argtypes = [vp, i32, vp, u64, i32, vp, vp]
    L.falcon_compress_stream.argtypes = [vp, i32, READ_FN, vp, STORE_FN, vp,
                                         C.POINTER(PipelineOptions), C.POINTER(PipelineStats)]
    L.falcon_decompress_stream.argtypes = [vp, i32, vp, u64, PUT_FN, vp, C.POINTER(PipelineOptions),
                                           C.POINTER(PipelineStats)]
    L.falcon_compress_host.argtypes = [vp, i32, vp, u64, C.POINTER(PipelineOptions), vp, u64,
                                       C.POINTER(u64), C.POINTER(PipelineStats)]
    L.falcon_decompress_host.argtypes = [vp, i32, vp, u64, vp, u64, C.POINTER(u64),
                                         C.POINTER(PipelineOptions), C.POINTER(PipelineStats)]
    L.falcon_compress_chunk.argtypes = [vp, i32, vp, u32, vp, u64, C.POINTER(u64)]
    L.falcon_decompress_chunk.argtypes = [vp, i32, vp, u64, u32, u32, vp]
    L.falcon_synth_fill.argtypes = [i32, C.POINTER(SynthSpec), vp, u64]
    L.falcon_compress_host_multi.argtypes = [C.POINTER(vp), u32, i32, vp, u64, C.POINTER(PipelineOptions), vp, u64,
                                             C.POINTER(u64), C.POINTER(PipelineStats)]
    L.falcon_decompress_host_multi.argtypes = [C.POINTER(vp), u32, i32, vp, u64, vp, u64, C.POINTER(u64),
                                               C.POINTER(PipelineOptions), C.POINTER(PipelineStats)]
    L.falcon_compress_device_frames.argtypes = [vp, i32, vp, u64, u32, u64, vp, u64, vp, vp]
    L.falcon_compress_file.argtypes = [vp, i32, C.c_char_p, C.c_char_p, C.POINTER(PipelineOptions),
                                       C.POINTER(u64), C.POINTER(i32)]
    L.falcon_decompress_file.argtypes = [vp, i32, C.c_char_p, C.c_char_p, C.POINTER(PipelineOptions),
                                         C.POINTER(u64), C.POINTER(i32)]
    L.falcon_synth_fill_at.argtypes = [i32, C.POINTER(SynthSpec), u64, vp, u64]
    L.falcon_synth_device.argtypes = [vp, i32, C.POINTER(SynthSpec), u64, vp, u64, vp]
    L.falcon_default_options.argtypes = [C.POINTER(PipelineOptions)]
    _lib = L
    return L


def _check(status: int) -> None:
    if status == OK:
        return
    msg = load().falcon_last_error().decode()
    if status == ERR_CORRUPT:
        raise CorruptError(status, msg)
    if status == ERR_CUDA:
        raise CudaError(status, msg)
    raise FalconError(status, msg)


def _np_ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def prec_of(dtype) -> int:
    if dtype in (np.float64, "float64") or str(dtype) in ("float64", "torch.float64"):
        return F64
    if dtype in (np.float32, "float32") or str(dtype) in ("float32", "torch.float32"):
        return F32
    raise TypeError(f"unsupported value type {dtype}")


def options(chunk_n=DEFAULT_CHUNK_N, batch_values=DEFAULT_BATCH_VALUES, n_streams=16, workers=0,
            stage_delay=None) -> PipelineOptions:
    o = PipelineOptions()
    o.chunk_n, o.batch_values, o.n_streams, o.workers = chunk_n, batch_values, n_streams, workers
    if stage_delay is not None:
        o.stage_delay = STAGE_FN(lambda _u, stage, slot, seq: stage_delay(stage, slot, seq))
    return o


def compress_bound(prec: int, n: int, chunk_n=DEFAULT_CHUNK_N, batch_values=DEFAULT_BATCH_VALUES) -> int:
    return load().falcon_compress_bound(prec, n, chunk_n, batch_values)


def max_encoded_chunk_size(prec: int, chunk_n: int) -> int:
    return load().falcon_max_encoded_chunk_size(prec, chunk_n)


def read_header(archive) -> ArchiveInfo:
    buf = np.frombuffer(bytes(archive[:47]), np.uint8).copy()
    info = ArchiveInfo()
    _check(load().falcon_read_header(_np_ptr(buf), len(archive), C.byref(info)))
    return info


def synth(kind: str, count: int, prec: int = F64, dp: int = 2, seed: int = 1, step: int = 127,
          period: int = 1025, units: int = 3575, block: int = DEFAULT_CHUNK_N, out=None,
          first: int = 0) -> np.ndarray:
    """Synthetic inputs (synthetic.hpp:36-115; kind 'mixed' = pinned cfg3 generator,
    'field' = counter-based field of the sharded configs, any `first`)."""
    s = SynthSpec(KINDS[kind], dp, seed, step, period, units, block)
    if out is None:
        out = np.empty(count, np.float64 if prec == F64 else np.float32)
    _check(load().falcon_synth_fill_at(prec, C.byref(s), first, _np_ptr(out), count))
    return out


def compress_host_multi(codecs, values: np.ndarray, opt: PipelineOptions | None = None,
                        stats: PipelineStats | None = None) -> np.ndarray:
    """Host-resident compress across several GPUs (one Codec per GPU), batch-range shards
    (falcon_compress_host_multi): bytes equal a single-GPU compress_host."""
    prec = prec_of(values.dtype)
    opt = opt or options()
    v = np.ascontiguousarray(values)
    out = np.empty(compress_bound(prec, len(v), opt.chunk_n, opt.batch_values), np.uint8)
    arr = (C.c_void_p * len(codecs))(*[c.ctx.value for c in codecs])
    nb = C.c_uint64()
    _check(load().falcon_compress_host_multi(arr, len(codecs), prec, _np_ptr(v), len(v), C.byref(opt), _np_ptr(out),
                                             len(out), C.byref(nb), C.byref(stats) if stats else None))
    return out[: nb.value]


def decompress_host_multi(codecs, archive, prec: int = F64, opt: PipelineOptions | None = None,
                          out: np.ndarray | None = None) -> np.ndarray:
    a = np.frombuffer(archive, np.uint8) if isinstance(archive, (bytes, bytearray)) else archive
    total = int.from_bytes(bytes(a[23:31]), "little") if len(a) >= 47 else 0
    if out is None:
        out = np.empty(max(total, 1), np.float64 if prec == F64 else np.float32)
    arr = (C.c_void_p * len(codecs))(*[c.ctx.value for c in codecs])
    nv = C.c_uint64()
    _check(load().falcon_decompress_host_multi(arr, len(codecs), prec, _np_ptr(a), len(a), _np_ptr(out), len(out),
                                               C.byref(nv), C.byref(opt or options()), None))
    return out[: nv.value]


class Codec:
    """One falcon_ctx on one GPU."""

    def __init__(self, device: int = 0):
        self.lib = load()
        self.ctx = C.c_void_p()
        _check(self.lib.falcon_ctx_create(device, C.byref(self.ctx)))
        self.device = device

    def close(self):
        if self.ctx:
            self.lib.falcon_ctx_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- device-resident (torch tensors on this codec's GPU) ----
    def compress_device(self, values, chunk_n=DEFAULT_CHUNK_N, batch_values=DEFAULT_BATCH_VALUES,
                        out=None, stream=None):
        """values: 1-D contiguous float64/float32 CUDA tensor.  Returns (archive u8 tensor, nbytes)."""
        import torch
        prec = prec_of(values.dtype)
        n = values.numel()
        cap = compress_bound(prec, n, chunk_n, batch_values)
        if out is None:
            out = torch.empty(cap, dtype=torch.uint8, device=values.device)
        nb = C.c_uint64()
        st = C.c_void_p(stream if stream is not None else torch.cuda.current_stream(values.device).cuda_stream)
        _check(self.lib.falcon_compress_device(self.ctx, prec, C.c_void_p(values.data_ptr()), n, chunk_n,
                                               batch_values, C.c_void_p(out.data_ptr()), out.numel(),
                                               C.byref(nb), st))
        return out, nb.value

    def compress_device_async(self, values, out, out_bytes, chunk_n=DEFAULT_CHUNK_N,
                              batch_values=DEFAULT_BATCH_VALUES, stream=None):
        import torch
        st = C.c_void_p(stream if stream is not None else torch.cuda.current_stream(values.device).cuda_stream)
        _check(self.lib.falcon_compress_device_async(
            self.ctx, prec_of(values.dtype), C.c_void_p(values.data_ptr()), values.numel(), chunk_n,
            batch_values, C.c_void_p(out.data_ptr()), out.numel(), C.c_void_p(out_bytes.data_ptr()), st))

    def decompress_device(self, archive, nbytes: int, dtype=None, out=None, stream=None):
        import torch
        info = read_header(archive[:47].cpu().numpy().tobytes() if nbytes >= 47 else b"\0" * 0)
        if dtype is None:
            dtype = torch.float64 if info.precision == F64 else torch.float32
        prec = prec_of(dtype)
        if out is None:
            out = torch.empty(max(info.total_values, 1), dtype=dtype, device=archive.device)
        nv = C.c_uint64()
        st = C.c_void_p(stream if stream is not None else torch.cuda.current_stream(archive.device).cuda_stream)
        _check(self.lib.falcon_decompress_device(self.ctx, prec, C.c_void_p(archive.data_ptr()), nbytes,
                                                 C.c_void_p(out.data_ptr()), out.numel(), C.byref(nv), st))
        return out[: nv.value]

    def decompress_device_chained(self, archive, nbytes_dev, info: ArchiveInfo, out, stream=None):
        """Decode with the archive length read on the device (nbytes_dev: a CUDA uint64/int64
        tensor, e.g. the out_bytes of compress_device_async): no host round trip."""
        import torch
        st = C.c_void_p(stream if stream is not None else torch.cuda.current_stream(archive.device).cuda_stream)
        _check(self.lib.falcon_decompress_device_chained(
            self.ctx, prec_of(out.dtype), C.c_void_p(archive.data_ptr()), C.c_void_p(nbytes_dev.data_ptr()),
            C.byref(info), C.c_void_p(out.data_ptr()), out.numel(), st))
        return out

    def archive_index(self, archive, nbytes: int, stream=None):
        """Batch-offset index of a device archive: numpy uint64[batch_count + 1]."""
        import torch
        info = read_header(archive[:47].cpu().numpy().tobytes())
        idx = torch.empty(info.batch_count + 1, dtype=torch.int64, device=archive.device)
        st = C.c_void_p(stream if stream is not None else torch.cuda.current_stream(archive.device).cuda_stream)
        _check(self.lib.falcon_archive_index(self.ctx, C.c_void_p(archive.data_ptr()), nbytes, C.byref(info),
                                             C.c_void_p(idx.data_ptr()), st))
        return idx.cpu().numpy().view(np.uint64)

    def decompress_range(self, archive, index, first_batch: int, n_batches: int, out=None, stream=None):
        """Random-access decode of batches [first_batch, first_batch + n_batches)."""
        import torch
        info = read_header(archive[:47].cpu().numpy().tobytes())
        dtype = torch.float64 if info.precision == F64 else torch.float32
        if out is None:
            out = torch.empty(max(n_batches * info.batch_values, 1), dtype=dtype, device=archive.device)
        idx = np.ascontiguousarray(index, dtype=np.uint64)
        nv = C.c_uint64()
        st = C.c_void_p(stream if stream is not None else torch.cuda.current_stream(archive.device).cuda_stream)
        _check(self.lib.falcon_decompress_device_range(
            self.ctx, info.precision, C.c_void_p(archive.data_ptr()), C.byref(info),
            idx.ctypes.data_as(C.POINTER(C.c_uint64)), first_batch, n_batches, C.c_void_p(out.data_ptr()),
            out.numel(), C.byref(nv), st))
        return out[: nv.value]

    def decompress_device_async(self, archive, nbytes: int, info: ArchiveInfo, out, stream=None):
        import torch
        st = C.c_void_p(stream if stream is not None else torch.cuda.current_stream(archive.device).cuda_stream)
        _check(self.lib.falcon_decompress_device_async(
            self.ctx, prec_of(out.dtype), C.c_void_p(archive.data_ptr()), nbytes, C.byref(info),
            C.c_void_p(out.data_ptr()), out.numel(), st))

    def synth_device(self, out, kind: str = "field", first: int = 0, dp: int = 2, seed: int = 1):
        """Fill the CUDA tensor `out` with values [first, first + out.numel()) of a
        counter-based kind, on the device (asynchronous on the current stream)."""
        import torch
        s = SynthSpec(KINDS[kind], dp, seed, 127, 1025, 3575, DEFAULT_CHUNK_N)
        st = C.c_void_p(torch.cuda.current_stream(out.device).cuda_stream)
        _check(self.lib.falcon_synth_device(self.ctx, prec_of(out.dtype), C.byref(s), first,
                                            C.c_void_p(out.data_ptr()), out.numel(), st))
        return out

    # ---- files through GPU-direct storage ----
    def compress_file(self, raw_path: str, archive_path: str, prec: int = F64, opt: PipelineOptions | None = None):
        """raw value file -> .fln archive; returns (archive bytes, io path: 1 cuFile / 0 bounce)."""
        nb, io = C.c_uint64(), C.c_int32()
        _check(self.lib.falcon_compress_file(self.ctx, prec, raw_path.encode(), archive_path.encode(),
                                             C.byref(opt) if opt else None, C.byref(nb), C.byref(io)))
        return nb.value, io.value

    def decompress_file(self, archive_path: str, raw_path: str, prec: int = F64):
        nv, io = C.c_uint64(), C.c_int32()
        _check(self.lib.falcon_decompress_file(self.ctx, prec, archive_path.encode(), raw_path.encode(), None,
                                               C.byref(nv), C.byref(io)))
        return nv.value, io.value

    def set_kernel_events(self, enc=None, dec=None):
        """enc/dec: (start, stop) torch.cuda.Event pairs recorded around the main kernels."""
        h = lambda e: C.c_void_p(e.cuda_event) if e is not None else None  # noqa: E731
        e0, e1 = enc if enc else (None, None)
        d0, d1 = dec if dec else (None, None)
        _check(self.lib.falcon_ctx_set_kernel_events(self.ctx, h(e0), h(e1), h(d0), h(d1)))

    def selftest_dp(self, values, candidate_alpha: int):
        """values: CUDA tensor.  Returns (full, literal, cert, g) CPU numpy arrays."""
        import torch
        n = values.numel()
        dev_ = values.device
        f = torch.empty(n, dtype=torch.int8, device=dev_)
        lit = torch.empty(n, dtype=torch.int8, device=dev_)
        c = torch.empty(n, dtype=torch.int8, device=dev_)
        g = torch.empty(n, dtype=torch.int64, device=dev_)
        st = C.c_void_p(torch.cuda.current_stream(dev_).cuda_stream)
        _check(self.lib.falcon_selftest_dp(self.ctx, prec_of(values.dtype), C.c_void_p(values.data_ptr()), n,
                                           candidate_alpha, C.c_void_p(f.data_ptr()), C.c_void_p(lit.data_ptr()),
                                           C.c_void_p(c.data_ptr()), C.c_void_p(g.data_ptr()), st))
        return f.cpu().numpy(), lit.cpu().numpy(), c.cpu().numpy(), g.cpu().numpy()

    def selftest_div(self, g, alpha: int, precision: int):
        """g: int64 CUDA tensor.  Returns the decoder's inverse scale of g at alpha (numpy)."""
        import torch
        out = torch.empty(g.numel(), dtype=torch.float64 if precision == 0 else torch.float32, device=g.device)
        st = C.c_void_p(torch.cuda.current_stream(g.device).cuda_stream)
        _check(self.lib.falcon_selftest_div(self.ctx, precision, C.c_void_p(g.data_ptr()), g.numel(), alpha,
                                            C.c_void_p(out.data_ptr()), st))
        return out.cpu().numpy()

    def sync(self, stream=None):
        import torch
        st = C.c_void_p(stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream)
        _check(self.lib.falcon_ctx_sync(self.ctx, st))

    # ---- host-resident pipeline ----
    def compress_host(self, values: np.ndarray, opt: PipelineOptions | None = None, out: np.ndarray | None = None,
                      stats: PipelineStats | None = None):
        prec = prec_of(values.dtype)
        opt = opt or options()
        v = np.ascontiguousarray(values)
        cap = compress_bound(prec, len(v), opt.chunk_n, opt.batch_values)
        if out is None:
            out = np.empty(cap, np.uint8)
        nb = C.c_uint64()
        _check(self.lib.falcon_compress_host(self.ctx, prec, _np_ptr(v), len(v), C.byref(opt), _np_ptr(out),
                                             len(out), C.byref(nb), C.byref(stats) if stats else None))
        return out[: nb.value]

    def decompress_host(self, archive, prec: int = F64, opt: PipelineOptions | None = None,
                        out: np.ndarray | None = None, stats: PipelineStats | None = None) -> np.ndarray:
        a = np.frombuffer(archive, np.uint8) if isinstance(archive, (bytes, bytearray)) else archive
        total = int.from_bytes(bytes(a[23:31]), "little") if len(a) >= 47 else 0
        if out is None:
            out = np.empty(max(total, 1), np.float64 if prec == F64 else np.float32)
        nv = C.c_uint64()
        _check(self.lib.falcon_decompress_host(self.ctx, prec, _np_ptr(a), len(a), _np_ptr(out), len(out),
                                               C.byref(nv), C.byref(opt or options()),
                                               C.byref(stats) if stats else None))
        return out[: nv.value]

    def compress_stream(self, read, store, prec: int, opt: PipelineOptions | None = None,
                        stats: PipelineStats | None = None):
        """read(max_values) -> np.ndarray (empty = EOF); store(offset, bytes)."""
        dt = np.float64 if prec == F64 else np.float32
        esz = np.dtype(dt).itemsize
        err = []

        def _read(_u, dst, maxv):
            try:
                chunk = np.ascontiguousarray(read(maxv), dtype=dt)
                k = min(len(chunk), maxv)
                C.memmove(dst, chunk.ctypes.data, k * esz)
                return k
            except Exception as e:  # noqa: BLE001
                err.append(e)
                return -1

        def _store(_u, off, ptr, ln):
            try:
                store(off, C.string_at(ptr, ln))
                return 0
            except Exception as e:  # noqa: BLE001
                err.append(e)
                return 1

        rf, sf = READ_FN(_read), STORE_FN(_store)
        st = self.lib.falcon_compress_stream(self.ctx, prec, rf, None, sf, None, C.byref(opt or options()),
                                             C.byref(stats) if stats else None)
        if err:
            raise err[0]
        _check(st)

    def decompress_stream(self, archive, put, prec: int, opt: PipelineOptions | None = None,
                          stats: PipelineStats | None = None):
        """put(first_value_index, np.ndarray) -- may be called from several threads."""
        dt = np.float64 if prec == F64 else np.float32
        a = np.frombuffer(archive, np.uint8) if isinstance(archive, (bytes, bytearray)) else archive
        err = []

        def _put(_u, first, ptr, count):
            try:
                arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), (count * np.dtype(dt).itemsize,))
                put(first, arr.view(dt).copy())
                return 0
            except Exception as e:  # noqa: BLE001
                err.append(e)
                return 1

        pf = PUT_FN(_put)
        st = self.lib.falcon_decompress_stream(self.ctx, prec, _np_ptr(a), len(a), pf, None,
                                               C.byref(opt or options()), C.byref(stats) if stats else None)
        if err:
            raise err[0]
        _check(st)

    # ---- per-chunk operators ----
    def compress_chunk(self, values: np.ndarray) -> bytes:
        prec = prec_of(values.dtype)
        v = np.ascontiguousarray(values)
        cap = max_encoded_chunk_size(prec, len(v))
        out = np.empty(cap, np.uint8)
        nb = C.c_uint64()
        _check(self.lib.falcon_compress_chunk(self.ctx, prec, _np_ptr(v), len(v), _np_ptr(out), cap, C.byref(nb)))
        return out[: nb.value].tobytes()

    def decompress_chunk(self, enc: bytes, n: int, count: int, prec: int = F64) -> np.ndarray:
        buf = np.frombuffer(enc, np.uint8).copy() if enc else np.zeros(1, np.uint8)
        out = np.empty(max(count, 1), np.float64 if prec == F64 else np.float32)
        _check(self.lib.falcon_decompress_chunk(self.ctx, prec, _np_ptr(buf), len(enc), n, count, _np_ptr(out)))
        return out[:count]
