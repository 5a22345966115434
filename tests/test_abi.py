"""C-ABI checks that need no GPU: the library builds for sm_100a, loads, exports every symbol
include/srsb.h declares, and validates arguments before touching a device."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def srsb():
    from paper_2003_12693_b200 import build
    build.build()
    from paper_2003_12693_b200 import srsb as S
    return S


def declared_functions():
    hdr = open(os.path.join(ROOT, "include", "srsb.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(sr_sb3?_\w+)\s*\(", hdr)))


def test_every_declared_symbol_is_exported(srsb):
    L = srsb.lib()
    names = declared_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(L, n), n
    assert sorted(srsb.EXPORTS) == names
    assert L.sr_sb_abi_version() == 3


def test_library_is_sm100a_only(srsb):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", srsb.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_params_struct_matches_header(srsb):
    """Field order of the ctypes mirror == sr_sb_params in include/srsb.h."""
    hdr = open(os.path.join(ROOT, "include", "srsb.h")).read()
    body = re.search(r"typedef struct \{(.*?)\} sr_sb_params;", hdr, flags=re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        typ, names = decl.split(None, 1)
        for nm in names.split(","):
            fields.append((nm.strip(), typ))
    mirror = [(n, "int" if t is C.c_int else "float") for n, t in srsb.Params._fields_]
    assert mirror == fields


def test_kernel_classes_match_header(srsb):
    hdr = open(os.path.join(ROOT, "include", "srsb.h")).read()
    body = re.search(r"typedef enum \{\s*(SR_K_RHS.*?)\} sr_kernel_class;", hdr, re.S).group(1)
    names = re.findall(r"SR_K_(\w+) = (\d+)", body)
    classes = [n.lower() for n, v in names if n != "NCLASSES"]
    assert classes == srsb.KERNEL_CLASSES
    assert dict(names)["NCLASSES"] == str(len(classes))


def test_default_params_are_the_design_readings(srsb):
    p = srsb.default_params(128, 128, 1, 3)
    assert (p["gamma"], p["alpha"], p["mu"], p["S"]) == (1.0, 4.0, 8.0, 3)
    assert p["beta"] == pytest.approx(0.2370643, rel=1e-5) and p["tau"] == pytest.approx(0.05)
    assert (p["epsilon"], p["l"], p["rho"], p["d"], p["window"]) == (0.5, 0.5, 30.0, 3.0, 3)
    assert (p["phi_clip"], p["w_proj"], p["window_shape"]) == (1.0, 0, 0)
    from synth import paper_params
    q = paper_params(3)
    for k in ("gamma", "alpha", "beta", "mu", "epsilon", "l", "d", "window", "window_shape", "tau", "S",
              "rho", "sigma", "s", "phi_clip", "w_proj", "w_mode", "w_iters"):
        assert p[k] == pytest.approx(q[k]), k


@pytest.mark.parametrize("field,value,status", [
    ("M", 100, -2), ("N", 16384, -2), ("M", 4, -2), ("batch", 0, -2), ("S", 0, -1), ("s", 3, -1),
    ("window", 9, -1), ("window", -1, -1), ("mu", 0.0, -1), ("epsilon", 0.0, -1), ("window_shape", 2, -1),
    ("w_proj", 3, -1), ("w_mode", 2, -1), ("sigma", 3.0, -1), ("phi_clip", -1.0, -1),
    ("phi_solver", 2, -1), ("phi_solver", -1, -1)])
def test_create_validates_before_device(srsb, field, value, status):
    p = srsb.Params()
    srsb.lib().sr_sb_default_params(C.byref(p), 64, 64, 1, 3)
    setattr(p, field, value)
    ctx = C.c_void_p()
    assert srsb.lib().sr_sb_create(C.byref(p), 0, None, C.byref(ctx)) == status
    assert not ctx.value
    assert srsb.lib().sr_sb_last_error(None)


def test_null_context_calls_are_rejected(srsb):
    L = srsb.lib()
    assert L.sr_sb_iterate(None, 1) == -1
    assert L.sr_sb_get_phi(None, None) == -1
    assert L.sr_sb_set_image(None, None, None) == -1
    assert L.sr_sb_iteration(None) == -1
    L.sr_sb_destroy(None)


def test_product_path_never_imports_the_oracle():
    """The binding and kernels share nothing with oracle/ (DESIGN.md §5)."""
    pkg = os.path.join(ROOT, "paper_2003_12693_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"import\s+oracle|from\s+oracle|liboracle|sr_oracle|orc_", txt), \
                    os.path.join(dirpath, f)


@pytest.mark.parametrize("D,field,value,status", [(3, "M", 64, -2), (8, "batch", 2, -2), (8, "window", 5, -1),
                                                  (2048, "M", 64, -2), (8, "phi_solver", 1, -1), (0, "M", 64, -2)])
def test_create3_validates_before_device(srsb, D, field, value, status):
    p = srsb.Params()
    srsb.lib().sr_sb_default_params(C.byref(p), 64, 64, 1, 3)
    setattr(p, field, value)
    ctx = C.c_void_p()
    assert srsb.lib().sr_sb3_create(C.byref(p), D, 0, None, C.byref(ctx)) == status
    assert not ctx.value
    assert srsb.lib().sr_sb3_last_error(None)
