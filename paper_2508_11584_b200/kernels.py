"""Atomic word access and busy-spin — the reference's ``fanpipe.kernels`` / ``fanpipe._kernels``
interface (kernels.py:10-50, _kernels.pyx:56-109) backed by libvpe's C ABI
(``vpe_u32_* / vpe_u64_* / vpe_busy_spin_ns``).

There is one backend: the native one. ``HAVE_COMPILED`` is always True and
``active_backend()`` always "compiled"; a missing library fails the import (no pure fallback).
"""

from __future__ import annotations

import ctypes as C

from ._lib import check, lib

HAVE_COMPILED = True
BACKEND = "compiled"


def active_backend(force_pure: bool | None = None) -> str:
    if force_pure:
        raise RuntimeError("the pure-Python fallback does not exist in the B200 build")
    return "compiled"


def _export(buf):
    """(address, nbytes, keepalive) of a writable buffer-protocol object or a host tensor. The
    keepalive objects pin the buffer export for the AtomicBuffer's lifetime, so the owner cannot
    be resized or unmapped under the atomics (the reference's typed memoryview does the same)."""
    if hasattr(buf, "data_ptr") and hasattr(buf, "untyped_storage"):
        if buf.is_cuda:
            raise ValueError("AtomicBuffer needs host memory")
        return buf.data_ptr(), buf.numel() * buf.element_size(), (buf,)
    mv = memoryview(buf)
    if mv.readonly:
        raise ValueError("buffer must be writable")
    mv = mv.cast("B")
    cbuf = (C.c_char * mv.nbytes).from_buffer(mv)
    return C.addressof(cbuf), mv.nbytes, (mv, cbuf)


class AtomicBuffer:
    """Atomic word access over a writable buffer, by byte offset (_kernels.pyx:56-98).

    Acquire loads, release stores, acq_rel CAS returning the previous value, acq_rel fetch-add.
    ``ValueError`` on misaligned / out-of-range offsets or a base not 8-byte aligned."""

    def __init__(self, buf):
        self._buf = buf  # keep the owner alive
        self._addr, self._size, self._pin = _export(buf)
        if lib.vpe_atomic_check_base(C.c_void_p(self._addr), self._size) != 0:
            raise ValueError("buffer base address must be 8-byte aligned")

    def _call(self, rc):
        if rc == 20:
            raise ValueError("bad offset")
        check(rc)

    def u32_load(self, off: int) -> int:
        out = C.c_uint32()
        self._call(lib.vpe_u32_load(C.c_void_p(self._addr), self._size, off, C.byref(out)))
        return out.value

    def u32_store(self, off: int, value: int) -> None:
        self._call(lib.vpe_u32_store(C.c_void_p(self._addr), self._size, off, value))

    def u32_cas(self, off: int, expected: int, desired: int) -> int:
        out = C.c_uint32()
        self._call(lib.vpe_u32_cas(C.c_void_p(self._addr), self._size, off, expected, desired, C.byref(out)))
        return out.value

    def u64_load(self, off: int) -> int:
        out = C.c_uint64()
        self._call(lib.vpe_u64_load(C.c_void_p(self._addr), self._size, off, C.byref(out)))
        return out.value

    def u64_store(self, off: int, value: int) -> None:
        self._call(lib.vpe_u64_store(C.c_void_p(self._addr), self._size, off, value))

    def u64_add(self, off: int, delta: int) -> int:
        out = C.c_uint64()
        self._call(lib.vpe_u64_add(C.c_void_p(self._addr), self._size, off, delta, C.byref(out)))
        return out.value

    def close(self) -> None:
        self._pin = ()  # drop the buffer export (the owner may be resized / unmapped again)
        self._buf = None
        self._addr, self._size = 0, 0


def make_atomics(buf, region_os_name: str = "", force_pure: bool | None = None) -> AtomicBuffer:
    active_backend(force_pure)
    return AtomicBuffer(buf)


def busy_spin_ns(duration_ns: int, force_pure: bool | None = None) -> None:
    lib.vpe_busy_spin_ns(int(duration_ns))


def now_ns() -> int:
    return int(lib.vpe_now_ns())
