"""librig.so loads and exports every symbol include/rig.h declares; host-side
argument validation (no compute calls, no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rig():
    from paper_1710_07769_b200 import build

    build.build()
    from paper_1710_07769_b200 import rig as r

    return r


def test_header_symbols_exported(rig):
    names = rig.header_symbols()
    expected = {"rig_build", "rig_build_rows", "rig_build_cut", "rig_graph_free", "rig_plan_create", "rig_plan_query",
                "rig_plan_execute", "rig_plan_destroy", "rig_row_split", "rig_cutsize", "rig_build_host",
                "rig_last_error", "rig_launch_count", "rig_version", "rig_profile_enable", "rig_profile_read", "rig_trim",
                "rig_pass_name", "rig_partition_ip", "rig_partition_ip_finalize", "rig_sparsify",
                "rig_csr_free", "rig_int_weights", "rig_hem_match", "rig_coarsen", "rig_coarse_free",
                "rig_last_path", "rig_gather_probe", "rig_mem_stats"}
    assert set(names) == expected
    so = ctypes.CDLL(rig.LIB_PATH)
    for n in names:
        assert hasattr(so, n), n


def test_status_codes_match_header(rig):
    txt = open(os.path.join(ROOT, "include", "rig.h")).read()
    for name in ["RIG_OK", "RIG_ERR_INVALID", "RIG_ERR_NONCANONICAL", "RIG_ERR_ZERO_ROW", "RIG_ERR_NONFINITE",
                 "RIG_ERR_NOMEM", "RIG_ERR_CUDA"]:
        m = re.search(rf"#define {name} \(?(-?\d+)\)?", txt)
        assert m and int(m.group(1)) == getattr(rig, name)
    for name in ["RIG_FLAG_VALIDATE", "RIG_FLAG_DIAG"]:
        m = re.search(rf"#define {name} (0x[0-9a-f]+)u", txt)
        assert m and int(m.group(1), 16) == getattr(rig, name)


def test_sm100a_only_cubin(rig):
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", rig.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_null_arguments_rejected_on_host(rig):
    L = rig.lib
    assert L.rig_build(None, 1, 0.0, 0, None, None) == rig.RIG_ERR_INVALID
    assert b"NULL" in L.rig_last_error()
    assert L.rig_plan_query(None, None, None, None) == rig.RIG_ERR_INVALID
    assert L.rig_cutsize(None, 0, 0, None, 1, None, None) == rig.RIG_ERR_INVALID
    A = rig.rig_csr_t(-1, 3, 0, 1, 1, 1)
    assert L.rig_build(ctypes.byref(A), 1, 0.0, 0, ctypes.byref(rig.rig_graph_t()), None) == rig.RIG_ERR_INVALID
    A = rig.rig_csr_t(3, 3, 0, 1, 1, 1)
    assert L.rig_build(ctypes.byref(A), 1, -1.0, 0, ctypes.byref(rig.rig_graph_t()), None) == rig.RIG_ERR_INVALID
    assert L.rig_build(ctypes.byref(A), 1, float("nan"), 0, ctypes.byref(rig.rig_graph_t()), None) == rig.RIG_ERR_INVALID
    assert L.rig_row_split(ctypes.byref(A), 0, None, None) == rig.RIG_ERR_INVALID
    assert rig.lib.rig_version().startswith(b"librig")


def test_partition_ip_finalize_host(rig):
    """The host conversion of the f2 fixed-point limbs (no GPU needed): each
    cell holds four 64-bit sums of 32-bit limbs of trunc(w * 2^64)."""
    import torch

    def limbs(w):
        hi = int(w)
        lo = int((w - hi) * 2**64)
        return [lo & 0xFFFFFFFF, lo >> 32, hi & 0xFFFFFFFF, hi >> 32]

    K = 2
    vals = {1: [1.5, 0.25, 3.0], 2: [2.0**-40, 7.0]}  # cells (0,1) and (1,0)
    acc = [0] * (4 * K * K + 1)
    for cell, ws in vals.items():
        for w in ws:
            for t, x in enumerate(limbs(w)):
                acc[4 * cell + t] += x
    ip = rig.rig_partition_ip_finalize(torch.tensor(acc, dtype=torch.int64), K)
    assert ip[0, 0] == 0 and ip[1, 1] == 0
    assert ip[0, 1] == 4.75 and ip[1, 0] == 7.0 + 2.0**-40
    acc[-1] = 1  # error flag: bad part id / weight
    with pytest.raises(rig.RigError):
        rig.rig_partition_ip_finalize(torch.tensor(acc, dtype=torch.int64), K)
