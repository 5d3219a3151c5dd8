"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/voronray_b200.h declares (no compute calls here)."""
import os
import re
import subprocess

import pytest
import torch

from conftest import ROOT


def declared_symbols():
    out = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            src = open(os.path.join(ROOT, "include", fn)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            out |= set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(vr_\w+)\s*\(", src, flags=re.M))
    return out


def test_header_declares_the_entry_points():
    syms = declared_symbols()
    for must in ("vr_raycast_batch", "vr_raycast_recheck", "vr_mc_rays", "vr_mc_reduce",
                 "vr_trav_claim", "vr_pack_generators", "vr_circumcenters"):
        assert must in syms


def test_library_exports_every_declared_symbol(built_library):
    out = subprocess.run(["nm", "-D", "--defined-only", built_library], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (vr_\w+)", out))
    missing = declared_symbols() - exported
    assert not missing, missing


def test_library_is_sm100a(built_library):
    out = subprocess.run(["cuobjdump", "--list-elf", built_library], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_loads_and_reports(built_library):
    from paper_2405_10050_b200 import _lib
    L = _lib.load_library()
    assert L.vr_abi_version() == _lib.ABI_VERSION == 7
    assert [L.vr_record_stride(d) for d in range(2, 9)] == [4, 4, 6, 6, 8, 8, 10]
    assert L.vr_record_stride(9) == 10 and L.vr_record_stride(16) == 18
    assert L.vr_record_stride(17) < 0
    assert L.vr_record_rows(1) == 512 and L.vr_record_rows(512) == 512
    assert L.vr_record_rows(513) == 1024
    assert L.vr_status_string(-2).startswith(b"dimension outside the supported range")
    for name in _lib.EXPORTED:
        getattr(L, name)
    assert set(_lib.EXPORTED) <= declared_symbols()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback(built_library):
    import numpy as np
    import paper_2405_10050_b200 as vb
    from paper_2405_10050_b200.errors import DeviceUnavailable
    ns = vb.build_node_set([(0.0, 0.0), (1.0, 0.0), (0.0, 1.0)])
    with pytest.raises(DeviceUnavailable):
        vb.raycast_batch(ns, np.zeros((1, 2)), np.array([[0.0, 1.0]]), np.zeros((1, 1), int))
    with pytest.raises(DeviceUnavailable):
        vb.mc_areas_only(ns, 0, 10, np.random.default_rng(0))


@pytest.mark.gpu
def test_integration_md_binding_runs():
    """The ctypes binding printed in INTEGRATION.md (what a reference
    maintainer would paste) runs as written and matches raycast_batch."""
    import numpy as np
    import paper_2405_10050_b200 as vb
    from paper_2405_10050_b200._build import LIB_PATH
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# pkg/src/voronray/_b200.py.*?)```", text, re.S).group(1)
    code = code.replace("/path/to/paper_2405_10050_b200/_voronray_b200.so", LIB_PATH)
    env = {}
    exec(compile(code, "INTEGRATION.md", "exec"), env)
    for n, d in ((700, 4), (5000, 6), (3000, 8)):
        pts = np.random.default_rng(4 + d).random((n, d))
        ns = vb.NodeSet(pts)
        dn = env["DeviceNodes"](ns)
        rng = np.random.default_rng(5 + d)
        g = rng.integers(0, n, 3000).astype(np.int32)
        u = rng.standard_normal((3000, d))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        idx, t, rp, fl = env["raycast_many"](dn, pts[g], u, g[:, None])
        ref = vb.raycast_batch(ns, pts[g], u, g[:, None], mode="exhaustive", screen="fp64")
        assert np.array_equal(idx, ref.idx.cpu().numpy())
        assert np.array_equal(fl, ref.flag.cpu().numpy())
        assert np.array_equal(t, ref.t.cpu().numpy(), equal_nan=True)
