"""The C-ABI library loads and exports every symbol include/fmm.h declares (no GPU needed).
Also: the product package never imports the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = "".join(open(os.path.join(ROOT, "include", h)).read() for h in sorted(os.listdir(os.path.join(ROOT, "include")))
                  if h.endswith(".h"))
    return sorted(set(re.findall(r"FMM_API\s+[\w\s\*]+?\b(fmm_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def libfmm():
    from paper_1602_02244_b200 import build

    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("fmm_setup", "fmm_matvec", "fmm_direct", "fmm_matvec_host", "fmm_destroy", "fmm_last_error",
              "fmm_stencil_apply", "fmm_precond_setup", "fmm_precond_apply", "fmm_pcg_solve"):
        assert s in syms


def test_library_exports_every_declared_symbol(libfmm):
    for s in declared_symbols():
        assert hasattr(libfmm, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_1602_02244_b200", "libfmm.so")],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (fmm_\w+)", out))
    assert exported == set(declared_symbols())


def test_python_binding_names_match(libfmm):
    from paper_1602_02244_b200 import _native

    assert set(_native.EXPORTED) == set(declared_symbols())
    assert _native.lib().fmm_version().decode().startswith("fmm-b200")


def test_library_is_sm100a_cubin():
    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(ROOT, "paper_1602_02244_b200", "libfmm.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_usage_errors_need_no_gpu(libfmm):
    """Argument validation happens before any device work (fmm.h error table)."""
    from paper_1602_02244_b200 import _native as N

    L = N.lib()
    h = ctypes.c_void_p()
    ex = N.FmmExec(0, None, 0, 1)
    assert L.fmm_setup(ctypes.byref(h), None, 10, 4, 8, 0.4, ctypes.byref(ex)) == N.FMM_ERR_USAGE
    assert b"NULL" in L.fmm_last_error()
    dummy = ctypes.c_void_p(1)
    for args in ((0, 4, 8, 0.4), (10, -1, 8, 0.4), (10, 17, 8, 0.4), (10, 4, 0, 0.4), (10, 4, 8, 0.0),
                 (10, 4, 8, 0.58)):
        assert L.fmm_setup(ctypes.byref(h), dummy, *args, ctypes.byref(ex)) == N.FMM_ERR_USAGE
    assert L.fmm_matvec(None, None, 0, None, None) == N.FMM_ERR_USAGE


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1602_02244_b200")
    pat = re.compile(r"(import\s+oracle|from\s+oracle|liboracle|fmm_oracle|oracle\.oracle)")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                assert not pat.search(open(os.path.join(dp, f)).read()), f


def test_m2l_v4_constants_stay_uniform():
    """M2L v4 (csrc/m2l_v4.cu) reads its fixed operator as warp-uniform constant-bank loads at immediate
    addresses (LDCU.128 into uniform registers, DFMA operands) once per use: no per-thread LDC (the ADU
    pipe throttled an earlier build to 5 TFLOP/s), one copy of the pair code in a called function
    (FMM_V4_CIMM: the compiler cannot hoist its constants out of the chunk loop), no spills inside it.
    A compiler-level property of the built library, checked in its SASS."""
    out = subprocess.run(["cuobjdump", "-sass", os.path.join(ROOT, "paper_1602_02244_b200", "libfmm.so")],
                         capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", out)
    body = [f for f in funcs if f.startswith("_ZN3fmm") and "m2l_v4_kernelILi10E" in f.split("\n")[0]]
    assert len(body) == 1
    sass = body[0]
    assert len(re.findall(r"\bLDC(?:\.64)?\s+R\d+, c\[0x3\]", sass)) == 0
    assert len(re.findall(r"\bLDCU\.128\s+UR\d+, c\[0x3\]\[0x[0-9a-f]+\]", sass)) > 800  # immediate, paired
    assert len(re.findall(r"\bDFMA\b[^;]*UR\d+", sass)) >= 1804  # F, G, F^T, G^T: 4 x 451 at p = 10
    assert len(re.findall(r"\bDFMA\b", sass)) < 4000  # one copy of the ~3.2K-FMA pair code
    # the pair function: from the CALL target to its RET, free of local-memory traffic
    ins = re.findall(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", sass)
    targets = {int(t, 16) for t in re.findall(r"CALL\.REL\.NOINC (0x[0-9a-f]+)", sass)}
    assert targets
    t0 = min(targets)
    fn = []
    for a, txt in ins:
        if int(a, 16) >= t0:
            fn.append(txt)
            if txt.strip().startswith("RET"):
                break
    assert sum("DFMA" in t for t in fn) > 3000
    assert not any(re.match(r"\s*(STL|LDL)", t) for t in fn)  # no register spills in the pair code
