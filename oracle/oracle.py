"""ctypes bindings for the parity checkers.  TEST INFRASTRUCTURE ONLY.

* ``Oracle``  -- oracle/liboracle.so, the C restatement (falcon_oracle.c).
* ``Ref``     -- oracle/_ref/libfalcon_ref.so, the unmodified reference library
                 (built from /root/reference by oracle/Makefile; optional).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfalcon_ref.so")

KINDS = {"walk": 0, "decimal": 1, "signflip": 2, "outlier": 3, "bits": 4, "mixed": 5, "field": 6}
F64, F32 = 0, 1


def dtype_of(prec: int):
    return np.float64 if prec == F64 else np.float32


def build(ref: bool = True) -> None:
    """Build liboracle.so (always) and _ref (when /root/reference is present)."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/include"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


class _Spec(C.Structure):
    _fields_ = [("kind", C.c_int), ("decimal_places", C.c_int), ("seed", C.c_uint64),
                ("max_step_units", C.c_int), ("outlier_period", C.c_uint64),
                ("outlier_units", C.c_int64), ("block", C.c_uint32)]


class OracleError(Exception):
    def __init__(self, code: int, message: str, corrupt: bool, batch: int | None = None):
        super().__init__(message)
        self.code, self.message, self.corrupt, self.batch = code, message, corrupt, batch


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.or_error_message.restype = C.c_char_p
        L.or_dp_ds_f64.argtypes = [C.c_double, C.POINTER(C.c_uint8), C.POINTER(C.c_uint8)]
        L.or_dp_ds_f32.argtypes = [C.c_float, C.POINTER(C.c_uint8), C.POINTER(C.c_uint8)]
        L.or_floor_log10_f64.argtypes = [C.c_double]
        L.or_floor_log10_f32.argtypes = [C.c_float]
        L.or_max_encoded_chunk_size.restype = C.c_size_t
        L.or_max_encoded_chunk_size.argtypes = [C.c_int, C.c_size_t]
        for s in ("f64", "f32"):
            f = getattr(L, f"or_compress_chunk_{s}")
            f.restype = C.c_size_t
            f.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p]
            g = getattr(L, f"or_decompress_chunk_{s}")
            g.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_void_p]
        L.or_compress_bound.restype = C.c_uint64
        L.or_compress_bound.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_uint64]
        L.or_compress_archive.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64,
                                          C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        L.or_decompress_archive.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_void_p,
                                            C.c_uint64, C.POINTER(C.c_uint64),
                                            C.POINTER(C.c_uint64)]
        L.or_synth_fill.argtypes = [C.c_int, C.POINTER(_Spec), C.c_void_p, C.c_uint64]
        L.or_synth_fill_at.argtypes = [C.c_int, C.POINTER(_Spec), C.c_uint64, C.c_void_p, C.c_uint64]
        L.or_dp_alpha_batch.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_void_p]
        L.or_round_scale_f64.argtypes = [C.c_double, C.c_int, C.POINTER(C.c_int64)]
        L.or_round_scale_f32.argtypes = [C.c_float, C.c_int, C.POINTER(C.c_int64)]

    def message(self, code: int) -> str:
        return self.lib.or_error_message(code).decode()

    def _raise(self, code: int, batch: int | None = None):
        msg = self.message(code)
        if batch is not None and batch != (1 << 64) - 1:
            msg = f"{msg} (batch {batch})"
        else:
            batch = None
        raise OracleError(code, msg, bool(self.lib.or_error_is_corrupt(code)), batch)

    def dp_ds(self, v: float, prec: int = F64):
        a, b = C.c_uint8(), C.c_uint8()
        f = self.lib.or_dp_ds_f64 if prec == F64 else self.lib.or_dp_ds_f32
        it = f(v, C.byref(a), C.byref(b))
        return a.value, b.value, it

    def dp_alpha_batch(self, values: np.ndarray) -> np.ndarray:
        prec = F64 if values.dtype == np.float64 else F32
        v = np.ascontiguousarray(values)
        out = np.empty(len(v), np.int8)
        self.lib.or_dp_alpha_batch(prec, _ptr(v), len(v), _ptr(out))
        return out

    def round_scale(self, v: float, alpha: int, prec: int = F64):
        g = C.c_int64()
        f = self.lib.or_round_scale_f64 if prec == F64 else self.lib.or_round_scale_f32
        rc = f(v, alpha, C.byref(g))
        return None if rc else g.value

    def floor_log10(self, v: float, prec: int = F64) -> int:
        f = self.lib.or_floor_log10_f64 if prec == F64 else self.lib.or_floor_log10_f32
        return f(v)

    def max_chunk(self, prec: int, n: int) -> int:
        return self.lib.or_max_encoded_chunk_size(prec, n)

    def compress_chunk(self, values: np.ndarray) -> bytes:
        prec = F64 if values.dtype == np.float64 else F32
        v = np.ascontiguousarray(values)
        out = np.zeros(self.max_chunk(prec, len(v)), np.uint8)
        f = self.lib.or_compress_chunk_f64 if prec == F64 else self.lib.or_compress_chunk_f32
        n = f(_ptr(v), len(v), _ptr(out))
        return out[:n].tobytes()

    def decompress_chunk(self, enc: bytes, n: int, count: int, prec: int = F64) -> np.ndarray:
        buf = np.frombuffer(enc, np.uint8).copy() if enc else np.zeros(1, np.uint8)
        out = np.zeros(max(count, 1), dtype_of(prec))
        f = self.lib.or_decompress_chunk_f64 if prec == F64 else self.lib.or_decompress_chunk_f32
        rc = f(_ptr(buf), len(enc), n, count, _ptr(out))
        if rc:
            self._raise(rc)
        return out[:count]

    def compress_bound(self, prec, count, chunk_n=1025, batch_values=1025 * 1024 * 4) -> int:
        return self.lib.or_compress_bound(prec, count, chunk_n, batch_values)

    def compress_archive(self, values: np.ndarray, chunk_n=1025, batch_values=1025 * 1024 * 4) -> bytes:
        prec = F64 if values.dtype == np.float64 else F32
        v = np.ascontiguousarray(values)
        cap = self.compress_bound(prec, len(v), chunk_n, batch_values)
        out = np.zeros(cap, np.uint8)
        n = C.c_uint64()
        rc = self.lib.or_compress_archive(prec, _ptr(v), len(v), chunk_n, batch_values,
                                          _ptr(out), cap, C.byref(n))
        if rc:
            self._raise(rc)
        return out[: n.value].tobytes()

    def decompress_archive(self, archive: bytes, prec: int = F64, cap: int | None = None) -> np.ndarray:
        buf = np.frombuffer(archive, np.uint8).copy() if archive else np.zeros(1, np.uint8)
        if cap is None:
            cap = int.from_bytes(archive[23:31], "little") if len(archive) >= 47 else 0
        out = np.zeros(max(cap, 1), dtype_of(prec))
        n, bad = C.c_uint64(), C.c_uint64()
        rc = self.lib.or_decompress_archive(prec, _ptr(buf), len(archive), _ptr(out), cap,
                                            C.byref(n), C.byref(bad))
        if rc:
            self._raise(rc, bad.value)
        return out[: n.value]

    def synth(self, kind: str, count: int, prec: int = F64, dp: int = 2, seed: int = 1,
              step: int = 127, period: int = 1025, units: int = 3575, block: int = 1025,
              first: int = 0, out: np.ndarray | None = None) -> np.ndarray:
        s = _Spec(KINDS[kind], dp, seed, step, period, units, block)
        if out is None:
            out = np.zeros(count, dtype_of(prec))
        if self.lib.or_synth_fill_at(prec, C.byref(s), first, _ptr(out), count):
            raise ValueError("bad generator spec")
        return out


class RefError(Exception):
    def __init__(self, kind: int, message: str):
        super().__init__(message)
        self.kind, self.message = kind, message   # 1 error, 2 corrupt_error

    @property
    def corrupt(self) -> bool:
        return self.kind == 2


class Ref:
    """The unmodified reference (oracle/_ref/libfalcon_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_dp_ds.argtypes = [C.c_int, C.c_double, C.POINTER(C.c_uint8), C.POINTER(C.c_uint8),
                                C.POINTER(C.c_int)]
        L.ref_floor_log10.argtypes = [C.c_int, C.c_double]
        L.ref_compress_chunk.restype = C.c_uint64
        L.ref_compress_chunk.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]
        L.ref_decompress_chunk.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                           C.c_void_p, C.c_char_p, C.c_size_t]
        L.ref_compress_pipeline.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64,
                                            C.c_uint, C.c_uint, C.POINTER(C.c_void_p),
                                            C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]
        L.ref_decompress_pipeline.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                              C.POINTER(C.c_uint64), C.c_uint, C.c_uint, C.c_char_p,
                                              C.c_size_t]
        L.ref_synth_fill.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_uint64,
                                     C.c_int64, C.c_void_p, C.c_uint64]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_hardware_threads.restype = C.c_uint

    def threads(self) -> int:
        return self.lib.ref_hardware_threads()

    def dp_ds(self, v: float, prec: int = F64):
        a, b, it = C.c_uint8(), C.c_uint8(), C.c_int()
        self.lib.ref_dp_ds(prec, v, C.byref(a), C.byref(b), C.byref(it))
        return a.value, b.value, it.value

    def floor_log10(self, v: float, prec: int = F64) -> int:
        return self.lib.ref_floor_log10(prec, v)

    def compress_chunk(self, values: np.ndarray) -> bytes:
        prec = F64 if values.dtype == np.float64 else F32
        v = np.ascontiguousarray(values)
        out = np.zeros(16 * len(v) + 64, np.uint8)
        n = self.lib.ref_compress_chunk(prec, _ptr(v), len(v), _ptr(out), len(out))
        return out[:n].tobytes()

    def decompress_chunk(self, enc: bytes, n: int, count: int, prec: int = F64) -> np.ndarray:
        buf = np.frombuffer(enc, np.uint8).copy() if enc else np.zeros(1, np.uint8)
        out = np.zeros(max(count, 1), dtype_of(prec))
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_decompress_chunk(prec, _ptr(buf), len(enc), n, count, _ptr(out), msg, 256)
        if rc:
            raise RefError(rc, msg.value.decode())
        return out[:count]

    def compress_pipeline(self, values: np.ndarray, chunk_n=1025, batch_values=1025 * 1024 * 4,
                          n_streams=16, workers=0) -> bytes:
        prec = F64 if values.dtype == np.float64 else F32
        v = np.ascontiguousarray(values)
        p, n = C.c_void_p(), C.c_uint64()
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_compress_pipeline(prec, _ptr(v), len(v), chunk_n, batch_values, n_streams,
                                            workers, C.byref(p), C.byref(n), msg, 256)
        if rc:
            raise RefError(rc, msg.value.decode())
        try:
            return C.string_at(p.value, n.value)
        finally:
            self.lib.ref_free(p)

    def decompress_pipeline(self, archive: bytes, prec: int = F64, n_streams=16, workers=0,
                            out: np.ndarray | None = None) -> np.ndarray:
        buf = np.frombuffer(archive, np.uint8)
        total = int.from_bytes(archive[23:31], "little") if len(archive) >= 47 else 0
        if out is None:
            out = np.zeros(max(total, 1), dtype_of(prec))
        n = C.c_uint64()
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_decompress_pipeline(prec, _ptr(buf), len(archive), _ptr(out), len(out),
                                              C.byref(n), n_streams, workers, msg, 256)
        if rc:
            raise RefError(rc, msg.value.decode())
        return out[: n.value]

    def synth(self, kind: str, count: int, prec: int = F64, dp: int = 2, seed: int = 1,
              step: int = 127, period: int = 1025, units: int = 3575) -> np.ndarray:
        out = np.zeros(count, dtype_of(prec))
        if self.lib.ref_synth_fill(prec, KINDS[kind], dp, seed, step, period, units, _ptr(out), count):
            raise ValueError("bad generator spec")
        return out


def ref_available() -> bool:
    return os.path.exists(REF_SO)
