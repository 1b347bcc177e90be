"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports
every symbol include/sscg.h declares, and its host-only entry points
(partition, NCCL id) behave -- no compute call is made without a GPU."""
import ctypes as C
import os
import re

import pytest

import paper_2512_09642_b200 as sscg
from paper_2512_09642_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return sscg.load()


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "sscg.h")).read()
    return sorted(set(re.findall(r"SSCG_API\s+[\w\s\*]+?\b(sscg_\w+)\s*\(", hdr)))


def test_header_declares_boundary():
    syms = declared_symbols()
    for name in ("sscg_setup", "sscg_solve", "sscg_stats", "sscg_inspect", "sscg_destroy"):
        assert name in syms
    assert set(syms) == set(sscg.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    # exported dynamic symbols are exactly the C ABI (-fvisibility=hidden)
    out = os.popen(f"nm -D --defined-only {sscg.LIB_PATH}").read()
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(declared_symbols()) <= exported
    assert not [s for s in exported if s.startswith("_ZN4sscg")]


def test_sass_targets_sm100a(lib):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump -lelf {sscg.LIB_PATH}").read()
    assert "sm_100a" in out
    sass = os.popen(f"/usr/local/cuda/bin/cuobjdump -sass {sscg.LIB_PATH}").read()
    assert "UTMALDG" in sass          # K2 streams P and W with TMA tensor loads
    assert "UTMALDG.4D" in sass       # K1T / K1F stage basis planes as 4-D boxes
    assert "SYNCS.PHASECHK" in sass   # mbarrier rings
    assert "DMMA" in sass             # K2D: Gram on FP64 tensor cores (s > 16)
    assert "DFMA" in sass


def test_version_and_error(lib):
    assert b"sm_100a" in lib.sscg_version()
    assert isinstance(lib.sscg_last_error(), bytes)


def test_partition_host_logic(lib):
    for nz, P, spr in ((448 * 8, 8, 1), (384, 8, 1), (33, 2, 3), (7, 7, 1), (100, 3, 2)):
        planes = []
        for r in range(P):
            z0, nzl = sscg.partition(nz, P, spr, r)
            assert nzl >= spr
            planes.append((z0, nzl))
        assert planes[0][0] == 0
        for (a0, an), (b0, _) in zip(planes, planes[1:]):
            assert a0 + an == b0
        assert planes[-1][0] + planes[-1][1] == nz
    with pytest.raises(sscg.SSCGError) as e:
        sscg.partition(3, 4, 1, 0)
    assert e.value.code == sscg.ERR_INVALID


def test_setup_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(sscg.SSCGError) as e:
        sscg.Solver(sscg.Stencil("7pt", 8, 8, 8), 0.1, 1.9, 4, 4)
    assert e.value.code == sscg.ERR_CUDA


def _build_example(tmp_path):
    import os
    import shutil
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2512_09642_b200", "libsscg.so")
    if not os.path.exists(lib) or not shutil.which("gcc"):
        pytest.skip("libsscg.so or gcc missing")
    exe = str(tmp_path / "solve_poisson")
    subprocess.run(["gcc", "-O2", "-Wall", "-Werror", os.path.join(root, "examples", "solve_poisson.c"),
                    "-I", os.path.join(root, "include"), "-L", os.path.dirname(lib), "-l:libsscg.so",
                    "-Wl,-rpath," + os.path.dirname(lib), "-lm", "-o", exe], check=True)
    return exe


def test_c_example_builds(tmp_path):
    """examples/solve_poisson.c uses the C ABI alone (no Python, no CUDA calls in
    the caller) and links against the in-tree library."""
    _build_example(tmp_path)


@pytest.mark.gpu
def test_c_example_solves(tmp_path):
    """The C example on a B200: 48^3 7-point Poisson, host b and x through
    sscg_solve_host, true residual checked on the host (exit code 0)."""
    import subprocess
    exe = _build_example(tmp_path)
    r = subprocess.run([exe, "48", "16", "25"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "converged=1" in r.stdout


def test_coarse_create_validates_before_touching_the_device(lib):
    """sscg_coarse_create (R25) rejects unsupported operators, bad
    aggregate sizes and coarse levels beyond one CTA's shared memory on the
    host, before any CUDA call (so these paths run without a GPU)."""
    def create(kind, dims, b, mode=0):
        op = sscg._Operator(kind, *dims, None, None, None, 0, None, None, None)
        h = C.c_void_p()
        return lib.sscg_coarse_create(C.byref(op), *b, mode, C.byref(h))
    assert create(sscg.OP_STENCIL27, (8, 8, 8), (2, 2, 2)) == sscg.ERR_UNSUPPORTED
    assert create(sscg.OP_CSR, (0, 0, 0), (1, 1, 1)) == sscg.ERR_UNSUPPORTED
    assert create(sscg.OP_STENCIL7, (64, 64, 64), (2, 2, 2)) == sscg.ERR_UNSUPPORTED   # n_c = 32768
    assert b"n_c" in lib.sscg_last_error()
    assert create(sscg.OP_STENCIL7, (8, 8, 8), (0, 2, 2)) == sscg.ERR_INVALID
    assert create(sscg.OP_STENCIL5_2D, (16, 16, 1), (2, 2, 2)) == sscg.ERR_INVALID     # 2D needs bz = 1
    assert create(sscg.OP_VARCOEF7, (8, 8, 8), (2, 2, 2)) == sscg.ERR_INVALID          # faces missing
    assert create(sscg.OP_STENCIL7, (8, 8, 8), (2, 2, 2), mode=2) == sscg.ERR_INVALID
    assert lib.sscg_coarse_fgs(None, None, None, 1, None) == sscg.ERR_INVALID
