"""The C-ABI library loads without a GPU and exports every symbol that
include/omb200.h declares; host-side entry points work on CPU."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "omb200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(omb_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    from paper_2107_10987_b200 import _lib

    L = _lib.load()
    names = declared_symbols()
    assert len(names) >= 12
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_lib.EXPORTS)
    assert L.omb_abi_version() == _lib.ABI_VERSION
    assert L.omb_stage_smem_bytes() <= 232448


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors vs the C compiler's view of include/omb200.h (size + every field offset)."""
    import subprocess

    from paper_2107_10987_b200._abi import (LEAF_INFO_DTYPE, OmbAmrDesc, OmbCflDesc, OmbRefluxDesc,
                                             OmbStageDesc)

    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{ROOT}/include/omb200.h"', "int main(void){"]
    checks = []
    for cls, cname in ((OmbStageDesc, "OmbStageDesc"), (OmbCflDesc, "OmbCflDesc"), (OmbAmrDesc, "OmbAmrDesc"),
                       (OmbRefluxDesc, "OmbRefluxDesc")):
        lines.append(f'printf("%zu\\n", sizeof({cname}));')
        checks.append(ctypes.sizeof(cls))
        for fname, _ in cls._fields_:
            lines.append(f'printf("%zu\\n", offsetof({cname}, {fname}));')
            checks.append(getattr(cls, fname).offset)
    lines.append('printf("%zu\\n", sizeof(OmbLeafInfo));')
    checks.append(LEAF_INFO_DTYPE.itemsize)
    for fname in LEAF_INFO_DTYPE.names:
        lines.append(f'printf("%zu\\n", offsetof(OmbLeafInfo, {fname}));')
        checks.append(LEAF_INFO_DTYPE.fields[fname][1])
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got == checks


@pytest.mark.parametrize("n,level", [(8, 2), (16, 1), (32, 1)])
def test_host_pack_roundtrip(n, level):
    """The native host packing (omb_host_pack / unpack: the copies of the e2e path) equals
    the per-leaf numpy copies -- for 16^3 / 32^3 leaves block by block, straight out of the
    leaf's padded array -- and the unpack leaves every ghost cell untouched."""
    import octomini_host as mesh
    from paper_2107_10987_b200 import _lib
    from paper_2107_10987_b200.batch import LeafBatch

    t = mesh.build_uniform_tree(level, n, boundary="periodic")
    rng = np.random.default_rng(0)
    for lf in t.leaves():
        lf.subgrid.u[...] = rng.normal(size=lf.subgrid.u.shape)
    ghosts = [lf.subgrid.u.copy() for lf in t.sorted_leaves()]
    b = LeafBatch(t)
    assert b.host_m == n + 6
    L = _lib.load()
    ref = b.pack()
    fast = b.pack(lib=L)
    assert np.array_equal(ref, fast)
    b.unpack(fast * 3.0, lib=L)
    assert np.array_equal(b.pack(), ref * 3.0)
    for lf, g in zip(t.sorted_leaves(), ghosts):
        g[:, 3:n + 3, 3:n + 3, 3:n + 3] *= 3.0
        assert np.array_equal(lf.subgrid.u, g)
    assert L.omb_host_pack(b._leaf_ptrs(b.L).ctypes.data, b.L, 8, 8, b.fstride, fast.ctypes.data) < 0  # m < n + 6


def test_no_cpu_fallback_without_gpu():
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2107_10987_b200 import NativeError, kernels

    with pytest.raises(NativeError):
        kernels.primitives(np.ones((6, 14, 14, 14)), 1.4, 1e-3)


def test_block_ptrs_follow_replaced_leaf_arrays():
    """The cached block pointer table of 16^3 leaves is revalidated by the identity of the
    leaves' arrays: a leaf array a user replaces is picked up by the next pack."""
    import octomini_host as mesh
    from paper_2107_10987_b200 import _lib
    from paper_2107_10987_b200.batch import LeafBatch

    t = mesh.build_uniform_tree(1, 16, boundary="periodic")
    rng = np.random.default_rng(1)
    for lf in t.leaves():
        lf.subgrid.u[...] = rng.normal(size=lf.subgrid.u.shape)
    b = LeafBatch(t)
    L = _lib.load()
    p0 = b._leaf_ptrs(b.L).copy()
    lf = t.sorted_leaves()[3]
    lf.subgrid._u = lf.subgrid.u * 2.0  # a new array object
    p1 = b._leaf_ptrs(b.L)
    moved = p0 != p1
    assert moved.sum() == 8 and moved[24:32].all()  # exactly that leaf's 8 blocks
    assert np.array_equal(b.pack(lib=L), b.pack())
