"""CPU-side checks of the C-ABI library: it loads and exports every symbol
include/pirrt.h declares, and the Python binding's struct layouts match the
header (no compute calls: there is no GPU here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pirrt.h")
HEADERS = [os.path.join(ROOT, "include", f) for f in sorted(os.listdir(os.path.join(ROOT, "include")))
           if f.endswith(".h")]


def declared_functions(headers=None):
    names = set()
    for h in headers or HEADERS:
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(pirrt_[a-z_]+)\s*\(", src))
    return sorted(names)


def test_header_declares_expected_calls():
    names = declared_functions([HEADER])
    # SURVEY.md section 8(b) boundary calls
    for must in ("pirrt_graph_append_batch", "pirrt_exploit", "pirrt_get_policy",
                 "pirrt_get_costs", "pirrt_best_path"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2003_04920_b200 import pirrt
    lib = C.CDLL(pirrt.LIB_PATH)
    names = declared_functions()
    assert sorted(pirrt.EXPORTS) == names
    for name in names:
        assert hasattr(lib, name), name


def test_struct_layouts_match_header(tmp_path):
    # compile the C header with gcc and compare every field offset and the
    # struct sizes with the ctypes mirrors of the binding
    import subprocess
    from paper_2003_04920_b200 import pirrt
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "pirrt.h"', 'int main(void) {']
    for st in (pirrt.pirrt_config, pirrt.pirrt_exploit_stats, pirrt.pirrt_step_result):
        lines.append(f'printf("{st.__name__} size %zu\\n", sizeof({st.__name__}));')
        for f, _ in st._fields_:
            lines.append(f'printf("{st.__name__} {f} %zu\\n", offsetof({st.__name__}, {f}));')
    lines += ['return 0;', '}']
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for st in (pirrt.pirrt_config, pirrt.pirrt_exploit_stats, pirrt.pirrt_step_result):
        assert got[(st.__name__, "size")] == C.sizeof(st)
        for f, _ in st._fields_:
            assert got[(st.__name__, f)] == getattr(st, f).offset, (st.__name__, f)
    cfg = pirrt.pirrt_config()
    pirrt.pirrt_config_init(C.byref(cfg))
    assert cfg.nranks == 1 and cfg.epsilon == 0.0 and cfg.flags == 0 and cfg.n_goals == 0
    assert cfg.root == 0 and cfg.goal == 1          # SURVEY.md 8(b) defaults


@pytest.mark.parametrize("root,goal", [(1, 0), (0, 2), (5, 1), (-1, 1)])
def test_root_goal_fields_validated_without_gpu(root, goal):
    # reading R15: x_init / x_goal are the first two vertices, so
    # only 0 / 1 are valid; checked before any CUDA call (runs on CPU)
    from paper_2003_04920_b200 import pirrt
    cfg = pirrt.pirrt_config()
    pirrt.pirrt_config_init(C.byref(cfg))
    cfg.root, cfg.goal = root, goal
    h = C.c_void_p()
    rc = pirrt.pirrt_create(C.byref(cfg), C.byref(h))
    assert rc == pirrt.PIRRT_E_INVAL
    assert b"R15" in pirrt.pirrt_last_error()


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    # a fresh import with the library path pointing at nothing must raise,
    # never fall back to anything
    import importlib.util
    import sys
    monkeypatch.setenv("PIRRT_LIB", str(tmp_path / "libpirrt.so"))
    spec = importlib.util.spec_from_file_location(
        "pirrt_missing_copy", os.path.join(ROOT, "paper_2003_04920_b200", "pirrt.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["pirrt_missing_copy"] = mod
    try:
        with pytest.raises(ImportError):
            spec.loader.exec_module(mod)
    finally:
        sys.modules.pop("pirrt_missing_copy", None)


def test_so_is_sm100a():
    from paper_2003_04920_b200 import pirrt
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pirrt.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("case", ["nbr_sharded", "nbr_group", "nbr_nranks", "group_with_id",
                                  "nranks_without_id"])
def test_config_combinations_refused_without_gpu(case):
    # configuration errors are reported before any CUDA call (runs on CPU)
    from paper_2003_04920_b200 import pirrt
    cfg = pirrt.pirrt_config()
    pirrt.pirrt_config_init(C.byref(cfg))
    uid = C.create_string_buffer(128)
    if case == "nbr_sharded":
        cfg.flags = pirrt.PIRRT_F_NEIGHBOURS | pirrt.PIRRT_F_SHARDED
    elif case == "nbr_group":
        cfg.flags = pirrt.PIRRT_F_NEIGHBOURS | pirrt.PIRRT_F_LOCAL_GROUP
    elif case == "nbr_nranks":
        cfg.flags = pirrt.PIRRT_F_NEIGHBOURS
        cfg.nranks, cfg.rank, cfg.nccl_unique_id = 2, 0, C.cast(uid, C.c_void_p)
    elif case == "group_with_id":
        cfg.flags = pirrt.PIRRT_F_LOCAL_GROUP
        cfg.nranks, cfg.rank, cfg.nccl_unique_id = 2, 1, C.cast(uid, C.c_void_p)
    else:
        cfg.nranks, cfg.rank = 2, 0
    h = C.c_void_p()
    assert pirrt.pirrt_create(C.byref(cfg), C.byref(h)) == pirrt.PIRRT_E_INVAL
