"""The C ABI: libpaste.so builds for sm_100a, loads without a GPU and exports
every entry point include/paste.h declares, with the ctypes struct mirrors
matching the header's layouts."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2603_18897_b200 import _native
from paper_2603_18897_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "paste.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(paste_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    build()
    return _native.load_library()


def test_header_declares_entry_points():
    fns = declared_functions()
    assert "paste_predict_batch" in fns and "paste_last_error" in fns
    assert set(fns) == set(_native.EXPORTS), "ctypes EXPORTS out of sync with include/paste.h"


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.paste_abi_version() == 1
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def _c_sizeof(struct_name: str) -> int:
    src = f'#include "paste.h"\n#include <stdio.h>\nint main(){{printf("%zu", sizeof({struct_name}));}}'
    exe = os.path.join("/tmp", f"sz_{struct_name}")
    subprocess.run(["gcc", "-x", "c", "-I", os.path.join(ROOT, "include"), "-o", exe, "-"],
                   input=src, text=True, check=True)
    return int(subprocess.run([exe], capture_output=True, text=True).stdout)


@pytest.mark.parametrize("cname,pyname", [
    ("paste_pool_desc", "PoolDesc"), ("paste_admit_desc", "AdmitDesc"),
    ("paste_windows", "WindowsDesc"), ("paste_predict_out", "PredictOut"),
    ("paste_admit_lists_desc", "AdmitListsDesc"), ("paste_mine_desc", "MineDesc"),
    ("paste_select_desc", "SelectDesc"), ("paste_columnar_desc", "ColumnarDesc"),
    ("paste_leaf_scan_desc", "LeafScanDesc"), ("paste_resolve_desc", "ResolveDesc"),
    ("paste_compact_desc", "CompactDesc"), ("paste_holds_desc", "HoldsDesc"),
    ("paste_hash_desc", "HashDesc"), ("paste_action_keys_desc", "ActionKeysDesc"),
    ("paste_ingest_desc", "IngestDesc"), ("paste_actions_desc", "ActionsDesc"),
    ("paste_jobs_out", "JobsOut"), ("paste_live_actions_desc", "LiveActionsDesc"),
    ("paste_live_plan", "LivePlan"), ("paste_order_desc", "OrderDesc"),
    ("paste_occ_desc", "OccDesc"), ("paste_key_lookup_desc", "KeyLookupDesc"),
    ("paste_jsonl_sizes", "JsonlSizes"), ("paste_jsonl_out", "JsonlOut"),
])
def test_struct_layouts_match_header(cname, pyname):
    assert ctypes.sizeof(getattr(_native, pyname)) == _c_sizeof(cname)


def test_element_dtypes_match_header():
    assert _native.PATTERN_DTYPE.itemsize == _c_sizeof("paste_pattern")
    assert _native.BINDING_DTYPE.itemsize == _c_sizeof("paste_binding")
    from paper_2603_18897_b200.tape import NODE_DTYPE
    assert NODE_DTYPE.itemsize == _c_sizeof("paste_tape_node")


def test_hot_path_refuses_to_run_without_a_device(monkeypatch):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_2603_18897_b200 import Predictor, PredictionWindow
    from paper_2603_18897_b200.mining import MiningConfig, PatternPool
    with pytest.raises(_native.NativeUnavailable):
        Predictor(PatternPool(MiningConfig(), ())).predict(PredictionWindow())
