"""CPU-side checks of the C-ABI boundary: the library builds, loads and exports
every symbol include/psfs.h declares; argument validation that needs no GPU."""
import ctypes as C
import os
import re

import pytest

from paper_1311_6811_b200 import build as pbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "psfs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(psfs_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    pbuild.build()
    from paper_1311_6811_b200 import psfs
    return psfs.lib()


def test_header_declares_the_five_contract_calls():
    names = _declared_functions()
    for n in ("psfs_create", "psfs_set_cameras", "psfs_set_background", "psfs_reconstruct",
              "psfs_destroy"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    from paper_1311_6811_b200 import psfs
    names = _declared_functions()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(psfs.EXPORTS) == names


def test_built_for_sm100a():
    so = pbuild.build()
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_defaults(lib):
    from paper_1311_6811_b200 import psfs
    assert lib.psfs_status_string(0) == b"PSFS_OK"
    assert b"EINVAL" in lib.psfs_status_string(1)
    assert psfs.default_params() == dict(occlusion_prior=0.5, voxel_prior=0.5, threshold=0.5,
                                         sigma_floor=1.0)


def test_create_rejects_bad_arguments_without_gpu(lib):
    """Validation that happens before any CUDA call."""
    from paper_1311_6811_b200 import psfs
    h = C.c_void_p()
    g = psfs.Grid((C.c_double * 3)(0, 0, 0), 1.0, 8, 8, 8)
    p = psfs.Params(0.5, 0.5, 0.5, 1.0)
    assert lib.psfs_create(None, C.byref(p), None, C.byref(h)) == 1
    bad = psfs.Grid((C.c_double * 3)(0, 0, 0), -1.0, 8, 8, 8)
    assert lib.psfs_create(C.byref(bad), C.byref(p), None, C.byref(h)) == 1
    badp = psfs.Params(1.0, 0.5, 0.5, 1.0)  # p_O not in (0,1)
    assert lib.psfs_create(C.byref(g), C.byref(badp), None, C.byref(h)) == 1
    badp = psfs.Params(0.5, 0.0, 0.5, 1.0)
    assert lib.psfs_create(C.byref(g), C.byref(badp), None, C.byref(h)) == 1
    d = psfs.Dist(0, 2, 2)  # rank out of range
    assert lib.psfs_create(C.byref(g), C.byref(p), C.byref(d), C.byref(h)) == 1
    d = psfs.Dist(0, 0, 3)  # zlen 8 not divisible by 3
    assert lib.psfs_create(C.byref(g), C.byref(p), C.byref(d), C.byref(h)) == 1
    assert lib.psfs_set_cameras(None, 1, None, None, None) == 1


def test_product_package_does_not_import_oracle():
    """The product path never imports oracle/ (test infrastructure only)."""
    import subprocess
    import sys
    code = ("import sys; import paper_1311_6811_b200, paper_1311_6811_b200.parallel; "
            "print(any(m == 'oracle' or m.startswith('oracle.') for m in sys.modules))")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() == "False"
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_1311_6811_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "psfs_oracle" not in txt, f
