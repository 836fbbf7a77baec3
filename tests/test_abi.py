"""CPU: the C-ABI library loads and exports every symbol include/*.h declares
(no compute calls — there is no GPU here)."""
import ctypes
import glob
import os
import re

from conftest import REPO


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(REPO, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(strait_\w+)\s*\(", text))
    return names


def test_header_declares_entry_points():
    names = declared_symbols()
    for must in ("strait_predict", "strait_estimate_latency", "strait_sweep", "strait_refit", "strait_round",
                 "strait_twa", "strait_abi_version", "strait_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2604_28175_b200 import _abi

    lib = _abi.lib()
    missing = [n for n in sorted(declared_symbols()) if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.strait_abi_version() == _abi.ABI_VERSION
    assert isinstance(lib.strait_last_error(), bytes)


def test_ctypes_mirrors_match_the_header_structs():
    """Every ctypes Structure the host passes through the C-ABI has the size of
    its C struct (strait_struct_size), so no field is misplaced."""
    import ctypes as C

    from paper_2604_28175_b200 import _abi, _node_abi as N, _replay_abi as R, devgen, ground_truth

    lib = _abi.lib()
    mirrors = [_abi.SweepArgs, _abi.SweepExpandArgs, _abi.RefitArgs, R.ReplayModels, R.ReplayConfig,
               R.ReplayArgs, None, R.MetricsArgs, devgen.StreamSpec, ground_truth.GroundTruth, N.GpuHdr,
               N.NodeEntry, N.ProposeArgs, N.ProposeOut]
    for i, m in enumerate(mirrors):
        want = lib.strait_struct_size(i)
        got = R.TRACE_DTYPE.itemsize if m is None else C.sizeof(m)
        assert got == want, (i, m, got, want)
    assert lib.strait_struct_size(99) == -1


def test_library_is_sm100a():
    import subprocess

    from paper_2604_28175_b200 import _abi

    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
