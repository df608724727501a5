"""CPU-only checks of the host layer: the C-ABI library loads and exports
every symbol the header declares, input generators, argument validation that
happens before any device work, bench plumbing."""

import ctypes
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "spamm_b200.h")


def _declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(spamm_\w+)\(", src, flags=re.M)))


def test_library_built_and_exports_header_symbols():
    from paper_1403_7458_b200 import _native as nat
    assert os.path.exists(nat.LIB_PATH), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(nat.LIB_PATH)  # loading does not touch the GPU
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/spamm_b200.h but not exported"
    assert set(nat.EXPORTED) == set(declared), "ctypes signature table out of sync with header"


def test_abi_version_and_error_string_without_gpu():
    from paper_1403_7458_b200 import _native as nat
    lib = nat.load()
    assert lib.spamm_abi_version() == nat.ABI_VERSION == 2
    assert lib.spamm_set_near_tau_ulps(-1) == nat.SPAMM_EINVAL
    # argument errors are reported before any CUDA call
    out = ctypes.c_void_p()
    rc = lib.spamm_mat_identity(0, 4, 4, None, ctypes.byref(out))
    assert rc == nat.SPAMM_EINVAL
    assert b"n >= 1" in lib.spamm_last_error()
    rc = lib.spamm_mat_from_dense(None, 4, 4, 3, 4, None, ctypes.byref(out))
    assert rc == nat.SPAMM_EINVAL and b"power of two" in lib.spamm_last_error()
    with pytest.raises(ValueError):
        nat.check(nat.SPAMM_EINVAL)


def test_ctypes_struct_layouts_match_header(tmp_path):
    """sizeof / offsetof of the ABI structs, compiled from include/spamm_b200.h
    with gcc, equal the ctypes mirrors in _native.py."""
    from paper_1403_7458_b200 import _native as nat
    structs = {"spamm_stats": nat.Stats, "spamm_sp2_report": nat.SP2Report,
               "spamm_mat_info": nat.MatInfo}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"',
             "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    try:
        subprocess.run(["gcc", "-o", str(exe), str(src)], check=True, capture_output=True)
    except (OSError, subprocess.CalledProcessError) as e:
        pytest.skip(f"gcc unavailable: {e}")
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True,
                                                         text=True).stdout.splitlines())
    for cname, cls in structs.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, (cname, fname)


def test_sass_contains_tensor_and_tma_instructions():
    from paper_1403_7458_b200 import _native as nat
    try:
        sass = subprocess.run(["cuobjdump", "-sass", nat.LIB_PATH], capture_output=True,
                              text=True, timeout=120).stdout
    except (OSError, subprocess.TimeoutExpired):
        pytest.skip("cuobjdump unavailable")
    assert "DMMA.8x8x4" in sass          # FP64 tensor-core leaf products
    assert "UTMALDG.2D" in sass          # TMA tiled loads in the leaf kernel
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", nat.LIB_PATH], capture_output=True,
                                       text=True).stdout


def test_build_validation_matches_reference_messages():
    import paper_1403_7458_b200 as sp
    with pytest.raises(ValueError, match="square"):
        sp.build_from_dense(np.zeros((3, 4)))
    with pytest.raises(ValueError, match="power of two"):
        sp.build_from_dense(np.zeros((4, 4)), block_size=3)
    with pytest.raises(ValueError, match="smaller than block size"):
        sp.build_from_dense(np.zeros((16, 16)), block_size=4, chunk_size=2)
    with pytest.raises(ValueError, match="power of two"):
        sp.build_from_dense(np.zeros((16, 16)), block_size=4, chunk_size=6)
    with pytest.raises(ValueError, match="exceeds padded size"):
        sp.build_from_dense(np.zeros((16, 16)), block_size=4, chunk_size=32)
    with pytest.raises(ValueError, match="n >= 1"):
        sp.identity(0, 4)


def test_compute_entry_points_fail_loudly_without_cuda():
    import torch

    import paper_1403_7458_b200 as sp
    if torch.cuda.is_available():
        pytest.skip("this host has a GPU")
    with pytest.raises(RuntimeError, match="CUDA device"):
        sp.build_from_dense(np.eye(8), 4)


def test_padded_geometry_matches_reference():
    from paper_1403_7458_b200.quadtree import _default_chunk_size, _padded_geometry
    assert _padded_geometry(2250, 16) == (4096, 8)
    assert _padded_geometry(3750, 64) == (4096, 6)
    assert _padded_geometry(750, 32) == (1024, 5)
    assert _padded_geometry(1, 1) == (1, 0)
    assert _default_chunk_size(4096, 64) == 512


def test_synthetic_generators():
    from paper_1403_7458_b200.synth import CONFIGS, decay_pair, water_cluster
    a, b = decay_pair(64, 0.1, (0, 1))
    assert np.array_equal(a, a.T) and np.array_equal(b, b.T) and not np.array_equal(a, b)
    a2, _ = decay_pair(64, 0.1, (0, 1))
    assert np.array_equal(a, a2)
    h, n_occ = water_cluster(6, seed=2)
    assert h.shape == (150, 150) and n_occ == 30
    assert np.array_equal(h, h.T)
    d = np.diag(h)
    assert np.sum(d < 0) == 30  # 5 occupied sites per molecule sit near -1
    h2, _ = water_cluster(6, seed=2)
    assert np.array_equal(h, h2)
    assert CONFIGS[4].n == 3750 and CONFIGS[4].block_size == 64


def test_fp64_peak_file_and_bench_help():
    sys.path.insert(0, ROOT)
    import bench
    peak, src = bench.fp64_peak()
    assert 30.0 < peak < 45.0 and "measured" in src
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"],
                         capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "--impl" in out.stdout


def test_profiles_committed():
    prof = os.path.join(ROOT, "profiles")
    names = os.listdir(prof)
    assert any(n.startswith("fp64_peak") for n in names)
    with open(os.path.join(prof, "fp64_peak_r01.json")) as f:
        assert json.load(f)["sms"] == 148
