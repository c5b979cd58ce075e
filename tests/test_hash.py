"""canonical_arg_hash (events.py:94-122): the host mirror and the device
kernel (hash.cu) against the reference's hashes (tests/golden/hash_golden.json,
made by make_golden.py hash)."""

import json
import os

import pytest

from paper_2603_18897_b200.events import canonical_arg_hash

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "hash_golden.json"), encoding="utf-8") as fh:
    CASES = json.load(fh)["cases"]


def _host(v):
    try:
        return canonical_arg_hash(v)
    except (UnicodeEncodeError, ValueError):
        return "error"


def test_host_mirror_matches_reference_hashes():
    assert [_host(c["value"]) for c in CASES] == [c["hash"] for c in CASES]


@pytest.mark.gpu
def test_device_hash_matches_reference_hashes():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2603_18897_b200 import hashing

    ok = [c for c in CASES if c["hash"] != "error"]
    got = hashing.canonical_arg_hash_batch([c["value"] for c in ok])
    assert got == [c["hash"] for c in ok]
    for c in CASES:
        if c["hash"] == "error":
            with pytest.raises(UnicodeEncodeError):
                hashing.canonical_arg_hash_batch([c["value"]])


@pytest.mark.gpu
def test_device_hash_decides_almost_every_value():
    """Only the documented corner cases go back to the host."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import ctypes

    import numpy as np

    from paper_2603_18897_b200 import _native, hashing
    from paper_2603_18897_b200.tape import KeyTable, TapeArena

    values = [c["value"] for c in CASES]
    keys = KeyTable()
    arena = TapeArena(keys, keep_objects=False)
    for v in values:
        arena.add(v)
    nodes, data, refs = arena.arrays()
    kb, ko, kr = hashing.key_tables(keys)
    dev = [torch.from_numpy(np.ascontiguousarray(a)).cuda()
           for a in (nodes.view(np.uint8), data, refs.reshape(-1), kb, ko, kr)]
    n = len(values)
    digest = torch.empty(16 * n, dtype=torch.uint8, device="cuda")
    unsure = torch.empty(n, dtype=torch.uint8, device="cuda")
    d = _native.HashDesc(n, *[_native.ptr(t) for t in dev], _native.ptr(digest),
                         _native.ptr(unsure))
    lib = _native.lib()
    _native.check(lib.paste_canonical_hash(ctypes.byref(d), 0), lib)
    torch.cuda.synchronize()
    expect = [_hard(v) for v in values]
    assert unsure.cpu().numpy().astype(bool).tolist() == expect
    assert sum(expect) < 0.05 * n


def _hard(v, depth=0):
    """The documented host cases: lone surrogates, two keys of one dict with
    one NFC form, nesting deeper than 32, dicts wider than 256 keys."""
    import unicodedata

    if isinstance(v, str):
        return any(0xD800 <= ord(ch) <= 0xDFFF for ch in v)
    if isinstance(v, list):
        return depth >= 32 or any(_hard(x, depth + 1) for x in v)
    if isinstance(v, dict):
        nfc = [unicodedata.normalize("NFC", k) for k in v]
        return (depth >= 32 or len(v) > 256 or len(set(nfc)) < len(nfc)
                or any(_hard(k) or _hard(x, depth + 1) for k, x in v.items()))
    return False
