"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
entry point include/exactz.h declares (no compute calls: CPU-only check)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "exactz.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(exactz_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from __graft_entry__ import _load_builder
    _build = _load_builder()
    lib_path = _build.build()
    lib = ctypes.CDLL(lib_path)
    names = declared_functions()
    assert "exactz_correct" in names and "exactz_correct_sharded" in names
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib_path], text=True)
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(names) <= exported


def test_cubin_is_sm100a():
    from __graft_entry__ import _load_builder
    _build = _load_builder()
    lib_path = _build.build()
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path],
                                  text=True)
    assert "sm_100a" in out


def test_package_imports_and_reports_version():
    import paper_2604_01397_b200 as E
    assert E.version().startswith("exactz sm_100a")
    assert E.lib().exactz_strerror(E.EBOUND) == b"input violates the error bound"


def test_oracle_is_not_used_by_the_product():
    """The product path never imports, links or executes oracle/ (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2604_01397_b200")
    bad = re.compile(r"(from\s+oracle|import\s+oracle|liboracle|exactz_oracle|oracle\.)")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert not bad.search(txt), fn
    out = subprocess.check_output(["ldd", os.path.join(pkg, "libexactz.so")], text=True)
    assert "oracle" not in out
