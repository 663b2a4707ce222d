"""C-ABI checks that need no GPU: libfdsdf.so builds for sm_100a, loads, exports every function
include/fdsdf.h declares, and its host-only entry points (spec validation, flat parameter
layout, status strings) agree with the documented contract.  No compute call is made."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from harness import layer_shapes, make_config, mlp_spec, num_params

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fdsdf.h")


@pytest.fixture(scope="module")
def L():
    from paper_2511_08980_b200._build import build
    build()
    from paper_2511_08980_b200 import fdsdf as F
    return F


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fdsdf_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = declared_functions()
    for must in ("fdsdf_create", "fdsdf_destroy", "fdsdf_eval", "fdsdf_step", "fdsdf_comm_init",
                 "fdsdf_allreduce", "fdsdf_num_params"):
        assert must in names


def test_library_exports_every_declared_symbol(L):
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(fdsdf_\w+)$", out, flags=re.M))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    lib = L.lib()
    for n in declared_functions():
        assert hasattr(lib, n)


def test_library_is_sm100a_code(L):
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_version(L):
    lib = L.lib()
    assert lib.fdsdf_status_string(0) == b"ok"
    assert lib.fdsdf_status_string(2) == b"empty input"
    assert b"sm_100a" in lib.fdsdf_version()


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_num_params_and_offsets_match_layout(L, name):
    from harness.gen import SIREN_256x4, SP512x8  # noqa: F401
    spec = {"c1": mlp_spec([3, 64, 64, 1], "softplus"), "c2": mlp_spec(**SIREN_256x4),
            "c3": mlp_spec(**SP512x8)}[name]
    s = L.make_spec(spec)
    lib = L.lib()
    assert lib.fdsdf_spec_num_params(C.byref(s)) == num_params(spec)
    off = 0
    for l, (o, i) in enumerate(layer_shapes(spec)):
        assert lib.fdsdf_spec_param_offset(C.byref(s), l, 0) == off
        assert lib.fdsdf_spec_param_offset(C.byref(s), l, 1) == off + o * i
        off += o * i + o
    assert lib.fdsdf_spec_param_offset(C.byref(s), len(layer_shapes(spec)), 0) == -1


def test_validate_spec_rejects_bad_specs(L):
    lib = L.lib()
    ok = mlp_spec([3, 64, 64, 1], "softplus")
    assert lib.fdsdf_validate_spec(C.byref(L.make_spec(ok))) == 0
    bad = [
        mlp_spec([3, 1], "softplus"),                          # < 2 linear layers
        mlp_spec([2, 64, 1], "softplus"),                      # width[0] != 3
        mlp_spec([3, 64, 2], "softplus"),                      # width[L] != 1
        mlp_spec([3, 0, 1], "softplus"),                       # width < 1
        mlp_spec([3, 1024, 1], "softplus"),                    # width > 512
        mlp_spec([3, 64, 64, 1], "softplus", beta=0.0),        # beta <= 0
        mlp_spec([3, 64, 64, 1], "sine", omega0_first=0.0),    # omega <= 0
        mlp_spec([3, 64, 64, 1], "softplus", skip_at=2),       # skip at the last layer
        mlp_spec([3, 64, 64, 1], "softplus", skip_at=0),       # skip at the first layer
        mlp_spec([3, 64, 510, 1], "softplus", skip_at=2),      # skip fan-in > 512 (also last)
    ]
    for sp in bad:
        assert lib.fdsdf_validate_spec(C.byref(L.make_spec(sp))) == 1, sp
    assert lib.fdsdf_spec_num_params(C.byref(L.make_spec(bad[0]))) == -1


def test_create_without_gpu_fails_cleanly(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    spec = mlp_spec([3, 64, 64, 1], "softplus")
    with pytest.raises(L.FdsdfError) as e:
        L.fdsdf_create(spec, 0, 128)
    assert e.value.code == "E_UNSUPPORTED"
    # invalid spec is rejected before any device query
    with pytest.raises(L.FdsdfError) as e:
        L.fdsdf_create(mlp_spec([3, 64, 2], "softplus"), 0, 128)
    assert e.value.code == "E_INVALID"


def test_binding_marshalling_matches_header_structs(L):
    """Field order / sizes of the ctypes mirrors against the C structs (x86-64 SysV layout)."""
    assert C.sizeof(L.MlpSpec) == 4 * (1 + 17 + 1) + 4 * 3 + 4
    assert L.Stencil.frame_seed.offset == 8 and L.Stencil.n_surface.offset == C.sizeof(L.Stencil) - 8
    assert C.sizeof(L.EvalOut) == 7 * 8
    c = make_config("c1", 4, 4)
    ls = L.make_loss(c["loss"], (4, 4, 8))
    assert (ls.n_surface_global, ls.n_uniform_global, ls.n_global) == (4, 4, 8)
    st = L.make_stencil(1e-2, 4, frame_seed=(1 << 64) - 1, index_offset=7)
    assert st.frame_seed == (1 << 64) - 1 and st.index_offset == 7 and st.frame_mode == 0
    assert np.float32(st.h) == np.float32(1e-2)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2511_08980_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b|#include.*oracle", txt, flags=re.M), f


def test_header_constants_match_binding():
    """Every enum value and flag the binding hard-codes equals the header's (include/fdsdf.h),
    parsed from the header text (no compiler, no GPU)."""
    import re
    from paper_2511_08980_b200 import fdsdf as F
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "fdsdf.h")).read()
    vals = {k: int(v) for k, v in re.findall(r"\b(FDSDF_[A-Z0-9_]+)\s*=\s*(\d+)u?\b", hdr)}
    mx = re.search(r"#define\s+FDSDF_MAX_LINEAR\s+(\d+)", hdr)
    assert mx and int(mx.group(1)) == F.MAX_LINEAR
    assert {"softplus": vals["FDSDF_ACT_SOFTPLUS"], "sine": vals["FDSDF_ACT_SINE"]} == F.ACT
    assert (vals["FDSDF_FRAME_RANDOM"], vals["FDSDF_FRAME_GIVEN"]) == (F.FRAME_RANDOM, F.FRAME_GIVEN)
    assert {k.lower(): vals["FDSDF_DENOM_" + k] for k in ("PAPER", "ONE", "GRAD")} == F.DENOM
    assert {"ncr": vals["FDSDF_LOSS_NCR"], "nsh": vals["FDSDF_LOSS_NSH"]} == F.KIND
    assert {"abs": vals["FDSDF_FD_ABS"], "square": vals["FDSDF_FD_SQUARE"]} == F.FD_FORM
    assert (vals["FDSDF_STEP_ACCUMULATE"], vals["FDSDF_STEP_ALLREDUCE"]) == (F.STEP_ACCUMULATE, F.STEP_ALLREDUCE)
    assert (vals["FDSDF_CREATE_EVAL_ONLY"], vals["FDSDF_CREATE_FFMA"], vals["FDSDF_CREATE_TENSOR"],
            vals["FDSDF_CREATE_WGRAD_BF16X3"]) == (F.CREATE_EVAL_ONLY, F.CREATE_FFMA, F.CREATE_TENSOR,
                                                   F.CREATE_WGRAD_BF16X3)
    assert {vals["FDSDF_PATH_" + k.upper()]: k for k in F.PATH.values()} == F.PATH
    assert (vals["FDSDF_FLAG_NONFINITE_INPUT"], vals["FDSDF_FLAG_NONFINITE_LOSS"], vals["FDSDF_FLAG_ALL_FD_SKIPPED"],
            vals["FDSDF_FLAG_NONFINITE_GRAD"]) == (F.FLAG_NONFINITE_INPUT, F.FLAG_NONFINITE_LOSS,
                                                   F.FLAG_ALL_FD_SKIPPED, F.FLAG_NONFINITE_GRAD)
    assert {vals["FDSDF_" + v]: v for v in F.STATUS.values()} == F.STATUS
    slots = {k: v for k, v in vals.items() if k.startswith("FDSDF_KSLOT_") and k != "FDSDF_KSLOT_NUM"}
    assert sorted(slots.values()) == list(range(len(F.KSLOTS)))
    assert all(F.KSLOTS[v] == k[len("FDSDF_KSLOT_"):].lower() for k, v in slots.items()), slots
    if "FDSDF_KSLOT_NUM" in vals:
        assert vals["FDSDF_KSLOT_NUM"] == len(F.KSLOTS)
