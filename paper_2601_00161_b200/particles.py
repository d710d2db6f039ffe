"""Particle files in the reference's text format (cli.py:57-112; SURVEY §8(f)
f4), parsed and written by the native code in ``libesp_b200.so``
(csrc/esp_io.cu) so that large systems load at C speed.

``read_particles(path) -> ParticleSystem`` and ``write_particles(path, sys)``
keep the reference's names, semantics (positions wrapped into the cell by
``ParticleSystem``; orthorhombic cells written as ``cell``, others as
``cell3`` in column order; ``%.17g``) and ``InputError`` diagnostics
(path:line[:column])."""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .errors import CellError, InputError
from .system import Cell, ParticleSystem


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def read_particles(path) -> ParticleSystem:
    L = _lib.lib()
    h = C.c_void_p()
    _lib.check(L.esp_particles_read(os.fsencode(str(path)), C.byref(h)), "esp_particles_read")
    try:
        n = C.c_int64()
        tri = C.c_int32()
        h9 = np.zeros(9)
        _lib.check(L.esp_particles_info(h, C.byref(n), C.byref(tri), _dp(h9)), "info")
        pos = np.empty((n.value, 3))
        q = np.empty(n.value)
        m = np.empty(n.value)
        _lib.check(L.esp_particles_copy(h, _dp(pos), _dp(q), _dp(m)), "copy")
    finally:
        L.esp_particles_free(h)
    cell = Cell(h9.reshape(3, 3)) if tri.value else Cell.orthorhombic(np.diag(h9.reshape(3, 3)))
    try:
        return ParticleSystem(cell=cell, positions=pos, charges=q, masses=m)
    except CellError as exc:
        raise InputError(f"{path}: {exc}") from exc


def write_particles(path, sys) -> None:
    pos = np.ascontiguousarray(sys.positions, dtype=np.float64)
    q = np.ascontiguousarray(sys.charges, dtype=np.float64)
    m = np.ascontiguousarray(sys.masses if sys.masses is not None else np.ones(q.size),
                             dtype=np.float64)
    h9 = np.ascontiguousarray(np.asarray(sys.cell.h, dtype=np.float64).reshape(9))
    tri = 0 if sys.cell.is_orthorhombic else 1
    _lib.check(_lib.lib().esp_particles_write(os.fsencode(str(path)), pos.shape[0], _dp(h9), tri,
                                              _dp(pos), _dp(q), _dp(m)), "esp_particles_write")
