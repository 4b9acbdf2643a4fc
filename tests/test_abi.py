"""C-ABI checks that need no GPU: the library loads, exports every symbol include/*.h declares,
and rejects bad arguments synchronously with the documented codes before touching CUDA."""
import ctypes

import pytest

from paper_2508_18572_b200 import _lib
from paper_2508_18572_b200._lib import PoolDesc, Xfer


@pytest.fixture(scope="module")
def lib():
    from paper_2508_18572_b200 import build
    build.build()
    return _lib.lib()


def test_exports_every_declared_symbol(lib):
    names = _lib.declared_symbols()
    assert len(names) >= 13, names
    for n in names:
        assert hasattr(lib, n), f"libstrata.so does not export {n}"
    for n in ("strata_register_host_pool", "strata_load", "strata_offload", "strata_layer_event"):
        assert n in names
    assert lib.strata_version() >= 100


def test_ctypes_structs_match_the_c_compiler(tmp_path):
    """sizeof / offsetof of every field of every struct in include/*.h as gcc lays them out, against
    the ctypes mirrors the binding passes across the ABI."""
    import os
    import subprocess

    from paper_2508_18572_b200 import ctl, disk
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    structs = [("strata_pool_desc", PoolDesc), ("strata_xfer", Xfer), ("strata_counters", _lib.Counters),
               ("strata_ctl_desc", ctl.CtlDesc), ("strata_ctl_match_t", ctl.Match), ("strata_ctl_round", ctl.Round),
               ("strata_ctl_plan", ctl.Plan), ("strata_ctl_stats", ctl.Stats), ("strata_disk_desc", disk.DiskDesc)]
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "strata.h"', '#include "strata_ctl.h"',
             '#include "strata_disk.h"', "int main(void) {"]
    for cname, cls in structs:
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c99", "-I", inc, "-o", str(exe), str(src)])
    got = {}
    for ln in subprocess.check_output([str(exe)], text=True).splitlines():
        c, f, v = ln.split()
        got[(c, f)] = int(v)
    for cname, cls in structs:
        assert got[(cname, "sizeof")] == ctypes.sizeof(cls), cname
        for f, _ in cls._fields_:
            assert got[(cname, f)] == getattr(cls, f).offset, (cname, f)


def test_struct_layouts_match_header(lib):
    # int32 x8 then pointers/int64 (see include/strata.h); 8-byte aligned, no padding surprises
    assert ctypes.sizeof(PoolDesc) == 8 * 4 + 2 * 8 + 4 * 8 + 8 + 8 + 2 * 4   # + host_heads, head_begin
    assert ctypes.sizeof(Xfer) == 6 * 4 + 7 * 8 + 2 * 8 + 8 + 8


def _desc(**kw):
    k = (ctypes.c_void_p * 2)(0x10000, 0x20000)
    v = (ctypes.c_void_p * 2)(0x30000, 0x40000)
    d = dict(device=0, num_layers=2, num_heads=2, head_dim=64, elem_bytes=2, page_size=16, chunk_tokens=64,
             flags=0, k_ptrs=ctypes.cast(k, ctypes.POINTER(ctypes.c_void_p)),
             v_ptrs=ctypes.cast(v, ctypes.POINTER(ctypes.c_void_p)), page_stride=0, token_stride=0,
             head_stride=0, num_pages=256, host_base=None, num_chunks=64)
    d.update(kw)
    return PoolDesc(**d), (k, v)


def _register(lib, desc):
    h = ctypes.c_void_p()
    rc = lib.strata_register_host_pool(ctypes.byref(desc), ctypes.byref(h))
    return rc, h


@pytest.mark.parametrize("field,value,code", [
    ("num_layers", 0, _lib.STRATA_ERR_INVALID_ARG),
    ("page_size", 0, _lib.STRATA_ERR_INVALID_ARG),
    ("num_chunks", 0, _lib.STRATA_ERR_INVALID_ARG),
    ("token_stride", 1 + 256, _lib.STRATA_ERR_ALIGNMENT),   # not a multiple of e = 2 (R29)
    ("page_stride", 25, _lib.STRATA_ERR_ALIGNMENT),
    ("host_base", 0x1001, _lib.STRATA_ERR_ALIGNMENT),
    ("num_pages", 1 << 31, _lib.STRATA_ERR_INVALID_ARG),
])
def test_register_rejects_bad_descriptor(lib, field, value, code):
    desc, keep = _desc(**{field: value})
    rc, h = _register(lib, desc)
    assert rc == code, lib.strata_last_error()
    assert not h.value
    assert lib.strata_last_error()


def test_register_rejects_null_and_misaligned_layer_ptrs(lib):
    assert lib.strata_register_host_pool(None, ctypes.byref(ctypes.c_void_p())) == _lib.STRATA_ERR_INVALID_ARG
    k = (ctypes.c_void_p * 2)(0x10000, 0)
    desc, keep = _desc(k_ptrs=ctypes.cast(k, ctypes.POINTER(ctypes.c_void_p)))
    assert _register(lib, desc)[0] == _lib.STRATA_ERR_INVALID_ARG
    k = (ctypes.c_void_p * 2)(0x10000, 0x10003)   # not a multiple of the 2-byte element
    desc, keep = _desc(k_ptrs=ctypes.cast(k, ctypes.POINTER(ctypes.c_void_p)))
    assert _register(lib, desc)[0] == _lib.STRATA_ERR_ALIGNMENT


@pytest.mark.parametrize("field,value", [("head_dim", 3), ("token_stride", 8 + 256), ("page_stride", 24),
                                         ("host_base", 0x1008)])
def test_rows_and_strides_need_not_be_16_byte_multiples(lib, field, value):
    """R29: 12-byte rows, 8-byte-aligned strides and bases pass the host-side checks (the narrow LDG
    kernel takes them); on a box without a GPU registration then stops at the first CUDA call."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    desc, keep = _desc(**{field: value})
    rc, h = _register(lib, desc)
    assert rc not in (_lib.STRATA_ERR_ALIGNMENT, _lib.STRATA_ERR_INVALID_ARG), lib.strata_last_error()


def test_valid_descriptor_without_gpu_fails_in_cuda(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    desc, keep = _desc()
    rc, h = _register(lib, desc)
    assert rc == _lib.STRATA_ERR_CUDA
    assert "cuda" in lib.strata_last_error().decode().lower()


def test_null_pool_calls(lib):
    x = Xfer()
    assert lib.strata_load(None, ctypes.byref(x), None, None) == _lib.STRATA_ERR_INVALID_ARG
    assert lib.strata_offload(None, ctypes.byref(x), None, None) == _lib.STRATA_ERR_INVALID_ARG
    ev = ctypes.c_void_p()
    assert lib.strata_layer_event(None, 0, 0, ctypes.byref(ev)) == _lib.STRATA_ERR_INVALID_ARG
    assert lib.strata_unregister_host_pool(None) == _lib.STRATA_OK
    assert lib.strata_host_pool_ptr(None, None, None) == _lib.STRATA_ERR_INVALID_ARG


def test_product_has_no_oracle_dependency():
    """The product package never imports the oracle (which is test infrastructure)."""
    import os
    import re
    root = os.path.join(os.path.dirname(os.path.dirname(__file__)), "paper_2508_18572_b200")
    for dirpath, _, files in os.walk(root):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"\boracle\b", re.sub(r"(#|//).*", "", text)), f
