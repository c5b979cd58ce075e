"""canonical_arg_hash on the device (events.py:94-122).

``canonical_arg_hash_batch(values)`` returns, for many JSON-like values, the
reference's ``canonical_arg_hash`` -- blake2b-128 of the canonical JSON
(NFC keys sorted by code point, integral floats as ints, NFC strings,
``json.dumps(sort_keys=True, separators=(",", ":"), ensure_ascii=False)``).
The values are packed as payload tapes and hashed by ``paste_canonical_hash``
(hash.cu), one thread per value.  Values the kernel flags as unsure (two keys
of one dict with one NFC form, lone surrogates, nesting deeper than 32,
dicts wider than 256 keys) are hashed by the host with the reference
semantics -- for lone surrogates that raises like the reference does.
"""

from __future__ import annotations

import ctypes
import unicodedata
from typing import Any, Sequence

import numpy as np

from . import _native
from ._native import HashDesc, check, ptr
from .events import canonical_arg_hash
from .tape import KeyTable, TapeArena


def key_tables(keys: KeyTable) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(NFC key bytes, offsets, code-point ranks; equal NFC forms share a rank)."""
    nfc = [unicodedata.normalize("NFC", k) for k in keys.names]
    rank = {s: r for r, s in enumerate(sorted(set(nfc)))}
    enc = [s.encode("utf-8", "surrogatepass") for s in nfc]
    off = np.zeros(len(enc) + 1, np.int64)
    off[1:] = np.cumsum([len(b) for b in enc])
    data = np.frombuffer(b"".join(enc) or b"\0", np.uint8).copy()
    ranks = np.array([rank[s] for s in nfc] or [0], np.int32)
    return data, off, ranks


def canonical_arg_hash_batch(values: Sequence[Any]) -> list[str]:
    import torch

    lib = _native.lib()
    if not values:
        return []
    keys = KeyTable()
    arena = TapeArena(keys, keep_objects=False)
    arena.add_many(values)
    nodes, data, refs = arena.arrays()
    kb, ko, kr = key_tables(keys)
    dev = {name: torch.from_numpy(np.ascontiguousarray(a)).cuda()
           for name, a in (("nodes", nodes.view(np.uint8)), ("bytes", data),
                           ("refs", refs.reshape(-1)), ("kb", kb), ("ko", ko), ("kr", kr))}
    n = len(values)
    digest = torch.empty(16 * n, dtype=torch.uint8, device="cuda")
    unsure = torch.empty(n, dtype=torch.uint8, device="cuda")
    d = HashDesc(n, ptr(dev["nodes"]), ptr(dev["bytes"]), ptr(dev["refs"]), ptr(dev["kb"]),
                 ptr(dev["ko"]), ptr(dev["kr"]), ptr(digest), ptr(unsure))
    from .device_ops import stream_handle

    check(lib.paste_canonical_hash(ctypes.byref(d), stream_handle()), lib)
    dg = digest.cpu().numpy().reshape(n, 16)
    us = unsure.cpu().numpy()
    return [canonical_arg_hash(values[i]) if us[i] else dg[i].tobytes().hex() for i in range(n)]
