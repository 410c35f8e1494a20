"""CPU-side checks of the boundary (no GPU compute): the C-ABI library loads, exports every
symbol include/lra.h declares, the ctypes structs match the header's layout, and every
entry point fails loudly (LRA_ECUDA) when no device is present — there is no CPU fallback."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    import paper_1710_07946_b200._build as B
    B.build()
    from paper_1710_07946_b200 import lra
    return lra


def _header_functions():
    src = open(os.path.join(ROOT, "include", "lra.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lra_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    fns = _header_functions()
    for f in ("lra_preprocess", "lra_cross_approx", "lra_cur_residual", "lra_batch"):
        assert f in fns


def test_library_exports_every_declared_symbol(L):
    lib = L.lib()
    for f in _header_functions():
        assert hasattr(lib, f), f"liblra.so does not export {f}"
    assert set(L.EXPORTED) == set(_header_functions())


def test_struct_layouts(L, tmp_path):
    """The ctypes mirrors of the C structs match include/lra.h field by field: a C program
    compiled against the header prints every size and offset (gcc, no CUDA needed)."""
    import subprocess
    fields = {"lra_operand": [f for f, _ in L.lra_operand._fields_],
              "lra_multiplier": [f for f, _ in L.lra_multiplier._fields_],
              "lra_ca_stats": list(L.STATS_DTYPE.names)}
    src = ["#include <stdio.h>", "#include <stddef.h>", '#include "lra.h"', "int main(void) {"]
    for st, fs in fields.items():
        src.append(f'printf("{st} %zu\\n", sizeof({st}));')
        for f in fs:
            src.append(f'printf("{st}.{f} %zu\\n", offsetof({st}, {f}));')
    src.append("return 0; }")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.splitlines())
    for st, cls in (("lra_operand", L.lra_operand), ("lra_multiplier", L.lra_multiplier)):
        assert int(got[st]) == ctypes.sizeof(cls), st
        for f, _ in cls._fields_:
            assert int(got[f"{st}.{f}"]) == getattr(cls, f).offset, (st, f)
    assert int(got["lra_ca_stats"]) == L.STATS_DTYPE.itemsize
    for f in L.STATS_DTYPE.names:
        assert int(got[f"lra_ca_stats.{f}"]) == L.STATS_DTYPE.fields[f][1], f"lra_ca_stats.{f}"


def test_no_cpu_fallback(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(L.LraError) as e:
        L.Handle(0)
    assert e.value.status == L.LRA_ECUDA


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_1710_07946_b200 import lra
    monkeypatch.setattr(lra, "_SO", str(tmp_path / "nope.so"))
    monkeypatch.setattr(lra, "_lib", None)
    with pytest.raises(lra.LibraryMissing):
        lra.lib()


def test_product_path_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1710_07946_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", txt, re.M), f


def test_variance_bound_matches_chi_square(L):
    """lra_variance_bound (host C, Wilson-Hilferty) vs scipy's exact chi-square quantile."""
    from scipy.stats import chi2
    for K in (100, 1000, 10000, 1000000):
        for alpha in (0.01, 0.05, 0.2):
            ref = K * 2.5e-7 / chi2.ppf(alpha, K - 1)
            assert L.lra_variance_bound(2.5e-7, K, alpha) == pytest.approx(ref, rel=2e-3 if K == 100 else 2e-4)
    with pytest.raises(L.LraError):
        L.lra_variance_bound(1.0, 1, 0.05)
