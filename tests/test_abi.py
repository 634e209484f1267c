"""C-ABI library: loads, exports every symbol include/cm.h declares, validates
graphs before touching the device, key packing helpers.  CPU only (no compute
calls without a GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1910_02653_b200 import _abi
    return _abi.load()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "cm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(cm_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_exports_every_declared_symbol(lib):
    from paper_1910_02653_b200 import _abi
    names = declared_functions()
    assert set(names) == set(_abi.EXPORTS)
    for name in names:
        assert hasattr(lib, name), name


def test_no_torch_in_header():
    src = open(os.path.join(ROOT, "include", "cm.h")).read()
    assert "torch" not in src.lower().replace("pytorch", "")
    assert 'extern "C"' in src


def create(lib, n, edges, cost=None, mem=None, ovh=0):
    ptr = np.zeros(n + 1, np.int32)
    for (_, j) in edges:
        ptr[j + 1] += 1
    ptr = np.cumsum(ptr).astype(np.int32)
    idx = np.zeros(max(len(edges), 1), np.int32)
    fill = ptr[:-1].copy()
    for (i, j) in sorted(edges, key=lambda e: (e[1], e[0])):
        idx[fill[j]] = i
        fill[j] += 1
    c = np.ones(n, np.int64) if cost is None else np.asarray(cost, np.int64)
    m = np.ones(n, np.int64) if mem is None else np.asarray(mem, np.int64)
    h = ctypes.c_void_p()
    st = lib.cm_graph_create(n, ptr.ctypes.data, idx.ctypes.data, c.ctypes.data, m.ctypes.data,
                             ovh, ctypes.byref(h))
    return st, h


def test_graph_validation_codes(lib):
    from paper_1910_02653_b200 import _abi
    assert create(lib, 3, [(1, 0)])[0] == _abi.CM_ETOPO          # i > j
    assert create(lib, 3, [(1, 1)])[0] == _abi.CM_ETOPO          # self loop
    assert create(lib, 3, [(0, 1), (0, 1)])[0] == _abi.CM_EDUP   # E is a set
    assert create(lib, 0, [])[0] == _abi.CM_EINVAL
    assert create(lib, 1025, [])[0] == _abi.CM_ERANGE
    assert create(lib, 3, [(0, 1)], cost=[1, -1, 1])[0] == _abi.CM_EINVAL
    assert create(lib, 3, [(0, 1)], mem=[1 << 61, 1 << 61, 1 << 61])[0] == _abi.CM_ERANGE
    assert create(lib, 3, [(0, 1)], cost=[1 << 61, 1, 1])[0] == _abi.CM_ERANGE
    h = ctypes.c_void_p()
    assert lib.cm_graph_create(3, None, None, None, None, 0, ctypes.byref(h)) == _abi.CM_EINVAL
    assert lib.cm_graph_create(3, None, None, None, None, 0, None) == _abi.CM_EINVAL
    assert b"duplicate" in (create(lib, 3, [(0, 2), (0, 2)]) and lib.cm_last_error())


def test_null_args(lib):
    from paper_1910_02653_b200 import _abi
    assert lib.cm_round_and_evaluate(None, None, None) == _abi.CM_EINVAL
    lib.cm_graph_destroy(None)
    assert lib.cm_graph_n(None) == -1


def test_key_helpers(lib):
    assert lib.cm_key_idx_bits(0) == 0 and lib.cm_key_idx_bits(1) == 0
    assert lib.cm_key_idx_bits(2) == 1 and lib.cm_key_idx_bits(1 << 20) == 20
    assert lib.cm_key_idx_bits((1 << 20) + 1) == 21 and lib.cm_key_idx_bits(10 ** 6) == 20
    c, i = ctypes.c_int64(), ctypes.c_int64()
    lib.cm_decode_key((12345 << 20) | 777, 20, ctypes.byref(c), ctypes.byref(i))
    assert (c.value, i.value) == (12345, 777)
    lib.cm_decode_key((1 << 63) - 1, 20, ctypes.byref(c), ctypes.byref(i))
    assert (c.value, i.value) == (-1, -1)
    lib.cm_decode_key(99, 0, ctypes.byref(c), ctypes.byref(i))
    assert (c.value, i.value) == (99, 0)
    for s in range(7):
        assert lib.cm_status_string(s).startswith(b"CM_")


def test_binding_imports_and_fails_loudly(tmp_path):
    from paper_1910_02653_b200 import _abi
    with pytest.raises(ImportError):
        _abi.load(str(tmp_path / "missing.so"))


def test_eval_args_layout_matches_binding(tmp_path):
    """The ctypes mirror of cm_eval_args has the header's fields, offsets and size (a C
    program compiled against include/cm.h prints them), and the #define constants agree."""
    import shutil
    import subprocess
    from paper_1910_02653_b200 import _abi
    src = open(os.path.join(ROOT, "include", "cm.h")).read()
    body = re.search(r"typedef struct \{(.*?)\} cm_eval_args;", src, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"([A-Za-z_][A-Za-z0-9_]*)\s*;", body)
    assert fields == [f for f, _ in _abi.EvalArgs._fields_]
    for name in ("CM_LAYOUT_DENSE", "CM_LAYOUT_TRI4", "CM_ROUND_THRESHOLD", "CM_ROUND_RANDOMIZED",
                 "CM_EVAL_INIT_KEYS", "CM_EVAL_OVERLAP"):
        m = re.search(r"#define\s+%s\s+(\d+)" % name, src)
        assert m and int(m.group(1)) == getattr(_abi, name), name
    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    prog = tmp_path / "layout.c"
    prog.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "cm.h"\nint main(void) {\n'
                    + "".join(f'  printf("%zu\\n", offsetof(cm_eval_args, {f}));\n' for f in fields)
                    + '  printf("%zu\\n", sizeof(cm_eval_args));\n  return 0;\n}\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [getattr(_abi.EvalArgs, f).offset for f in fields] + [ctypes.sizeof(_abi.EvalArgs)]
    assert got == want
