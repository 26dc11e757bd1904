"""The C-ABI boundary: libsom.so builds, loads and exports every entry point
include/som.h declares; without a GPU it fails loudly (no CPU fallback).
No compute calls here (CPU box)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "som.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(som_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1905_09598_b200 import _build
    _build.build()
    from paper_1905_09598_b200 import som
    return som.lib()


def test_header_declares_the_north_star_calls():
    decl = _declared()
    for name in ["som_create", "som_train_online", "som_map", "som_qerror", "som_umatrix",
                 "som_topographic_error", "som_map_csr", "som_last_error"]:
        assert name in decl


def test_library_exports_every_declared_symbol(lib):
    from paper_1905_09598_b200 import som
    decl = _declared()
    missing = [s for s in decl if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(som.EXPORTS) == decl           # the binding covers the same set


def test_binding_has_same_names():
    from paper_1905_09598_b200 import som
    for s in _declared():
        assert callable(getattr(som, s)), s


def test_schedule_defaults_and_validation_without_gpu(lib):
    from paper_1905_09598_b200 import som
    s = som.som_schedule_default()
    assert s.kind == 0 and abs(s.k - 4.605170185988091) < 1e-15 and s.sigma_min == 1.0 and s.cutoff == 1e-4
    h = ctypes.c_void_p()
    assert lib.som_create(0, 3, 4, 0, 0, ctypes.byref(h)) == som.SOM_EINVAL
    assert lib.som_create(3, 3, 4, 7, 0, ctypes.byref(h)) == som.SOM_EINVAL
    assert lib.som_train_online(None, None, 1, 1, 0.1, 1.0, None, 1, 0, -1, None) == som.SOM_EINVAL
    assert "version" not in som.som_version() and "sm_100a" in som.som_version()


def test_fails_loudly_without_device(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1905_09598_b200 import som
    with pytest.raises(som.SomError) as e:
        som.som_create(2, 2, 4, som.SOM_HEX)
    assert e.value.status == som.SOM_ECUDA


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1905_09598_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "som_oracle" not in txt, f


def test_binding_rejects_mismatched_shapes():
    """the binding checks array sizes against the handle before
    any C call (SOM_EDIM) — a fake handle registered with its
    map shape is enough, nothing reaches the library."""
    import ctypes

    import numpy as np

    from paper_1905_09598_b200 import som
    h = ctypes.c_void_p(0x1234)
    som._dims[0x1234] = (4, 3)
    try:
        bad = [lambda: som.som_map(h, np.zeros((2, 5), np.float32), 2, np.zeros(2, np.int32)),
               lambda: som.som_map(h, np.zeros((2, 3), np.float32), 3, np.zeros(3, np.int32)),
               lambda: som.som_map(h, np.zeros((2, 3), np.float32), 2, np.zeros(1, np.int32)),
               lambda: som.som_get_weights(h, np.zeros((3, 3), np.float32)),
               lambda: som.som_set_weights(h, np.zeros(11, np.float32)),
               lambda: som.som_train_online(h, np.zeros((5, 4), np.float32), 5, 1, 0.1, 1.0, None, 1),
               lambda: som.som_train_online(h, np.zeros((5, 3), np.float32), 5, 2, 0.1, 1.0, None, 1, 0, -1,
                                            np.zeros(9, np.int32)),
               lambda: som.som_umatrix(h, np.zeros(3, np.float32)),
               lambda: som.som_errors_csr(h, np.zeros(2, np.int64), np.zeros(1, np.int32), np.zeros(1, np.float32), 2)]
        for f in bad:
            with pytest.raises(som.SomError) as e:
                f()
            assert e.value.status == som.SOM_EDIM
    finally:
        som._dims.pop(0x1234, None)
