"""Payload tapes: the HBM layout of tool-call results and arguments.

Every JSON-like payload is flattened into a pre-order *tape* of 16-byte nodes
(dict insertion order, list order -- the traversal order of the reference's
``candidate_paths``/``_scalar_leaves``, mappings.py:237-266,420-428) plus a
byte arena holding the scalar bytes:

=========  ==========================================================
field      meaning
=========  ==========================================================
type  u8   NULL FALSE TRUE INT FLOAT STR LIST DICT
flags u8   NFC (str whose NFC form differs), FLOATSRC (integral float
           stored as INT), NAN
pad   u16  unused
key   i32  interned key of this node inside its parent dict, else -1
a     u32  containers: number of direct children; scalars: byte offset
           relative to the event's byte base
b     u32  containers: subtree size in nodes (next sibling = i + b);
           scalars: byte length
=========  ==========================================================

Scalar bytes are the *canonical* bytes of the reference's equality
(events.py:94-130): decimal digits for ints and integral floats, ``repr`` for
other floats, UTF-8 for strings.  Two scalars are ``values_equal`` iff their
type class and canonical bytes match and neither is NaN; strings whose NFC
form differs from the raw text carry the NFC bytes right after the raw bytes
(``[raw][u32 nfc_len][nfc]``) so the raw leaf can still be returned as the
extracted argument (mappings.py:197-204).
"""

from __future__ import annotations

import struct
import unicodedata
from typing import Any

import numpy as np

NODE_DTYPE = np.dtype([("type", "u1"), ("flags", "u1"), ("pad", "u2"),
                       ("key", "i4"), ("a", "u4"), ("b", "u4")])
assert NODE_DTYPE.itemsize == 16

T_NULL, T_FALSE, T_TRUE, T_INT, T_FLOAT, T_STR, T_LIST, T_DICT = range(8)
F_NFC, F_FLOATSRC, F_NAN, F_ASCII = 1, 2, 4, 8


class KeyTable:
    """Interns dict keys (and mapping path keys) to dense ids shared by the
    pool image and every payload tape of one engine."""

    def __init__(self) -> None:
        self.ids: dict[str, int] = {}
        self.names: list[str] = []

    def intern(self, key: str) -> int:
        kid = self.ids.get(key)
        if kid is None:
            kid = len(self.names)
            self.ids[key] = kid
            self.names.append(key)
        return kid

    def __len__(self) -> int:
        return len(self.names)


def scalar_bytes(value: Any) -> tuple[int, int, bytes]:
    """(type, flags, canonical bytes) of a scalar leaf."""
    if value is None:
        return T_NULL, 0, b""
    if value is True:
        return T_TRUE, 0, b""
    if value is False:
        return T_FALSE, 0, b""
    if isinstance(value, bool):  # numpy bools etc.
        return (T_TRUE if value else T_FALSE), 0, b""
    if isinstance(value, int):
        return T_INT, F_ASCII, str(int(value)).encode()
    if isinstance(value, float):
        if value.is_integer():
            return T_INT, F_FLOATSRC | F_ASCII, str(int(value)).encode()
        return T_FLOAT, (F_NAN if value != value else 0) | F_ASCII, repr(value).encode()
    if isinstance(value, str):
        if value.isascii():
            return T_STR, F_ASCII, value.encode()
        raw = value.encode("utf-8", "surrogatepass")
        nfc = unicodedata.normalize("NFC", value)
        if nfc != value:
            nb = nfc.encode("utf-8", "surrogatepass")
            return T_STR, F_NFC, raw + struct.pack("<I", len(nb)) + nb
        return T_STR, 0, raw
    raise TypeError(f"payload leaf of type {type(value).__name__} is not JSON-like")


_NODE = struct.Struct("<BBHiII")
try:  # the native encoder (csrc/tapes_py.cpp): exact JSON types, ~20x faster
    from . import _tapes as _native_tapes
except ImportError:  # pragma: no cover - built by build(); the Python path is exact
    _native_tapes = None


class TapeArena:
    """Append-only arena of payload tapes (one tape per event payload).

    ``keep_objects`` keeps the Python object of every node so that values the
    device resolves can be handed back by identity (the reference returns the
    payload's own leaf object from ``_walk``).  Nodes are kept packed
    (NODE_DTYPE bytes); ``add_many`` encodes a batch natively."""

    def __init__(self, keys: KeyTable | None = None, keep_objects: bool = True) -> None:
        self.keys = KeyTable() if keys is None else keys
        self.keep_objects = keep_objects
        self._nodes = bytearray()
        self._data = bytearray()
        self._refs: list[tuple[int, int]] = []
        self._objs: list[Any] = []
        self._frozen: tuple[np.ndarray, np.ndarray, np.ndarray] | None = None

    @property
    def n_nodes(self) -> int:
        return len(self._nodes) // 16

    # -- building -----------------------------------------------------------

    def add(self, payload: Any) -> int:
        """Encode one payload; returns its event-tape index."""
        node_base = self.n_nodes
        byte_base = len(self._data)
        self._emit(payload, -1, node_base, byte_base)
        self._refs.append((node_base, byte_base))
        self._frozen = None
        return len(self._refs) - 1

    def add_many(self, payloads) -> list[int]:
        """Encode a batch of payloads (native encoder for the exact JSON
        types; any payload it does not take goes through ``add``)."""
        payloads = list(payloads)
        if _native_tapes is None:
            return [self.add(p) for p in payloads]
        first = len(self._refs)
        i = 0
        while i < len(payloads):
            nodes, data, refs = _native_tapes.encode(
                payloads[i:] if i else payloads, self.keys.ids, self.keys.names, self.n_nodes,
                len(self._data), self._objs if self.keep_objects else None)
            self._nodes += nodes
            self._data += data
            self._refs.extend(refs)
            i += len(refs)
            if i < len(payloads):  # outside the native subset: the exact Python encoder
                self.add(payloads[i])
                i += 1
        self._frozen = None
        return list(range(first, len(self._refs)))

    def _emit(self, value: Any, key: int, node_base: int, byte_base: int) -> None:
        idx = self.n_nodes
        if isinstance(value, dict):
            self._nodes += _NODE.pack(T_DICT, 0, 0, key, len(value), 0)
            if self.keep_objects:
                self._objs.append(value)
            for k, v in value.items():
                if not isinstance(k, str):
                    raise TypeError("payload dict keys must be strings (JSON objects)")
                self._emit(v, self.keys.intern(k), node_base, byte_base)
            _NODE.pack_into(self._nodes, 16 * idx, T_DICT, 0, 0, key, len(value),
                            self.n_nodes - idx)
        elif isinstance(value, list):
            self._nodes += _NODE.pack(T_LIST, 0, 0, key, len(value), 0)
            if self.keep_objects:
                self._objs.append(value)
            for v in value:
                self._emit(v, -1, node_base, byte_base)
            _NODE.pack_into(self._nodes, 16 * idx, T_LIST, 0, 0, key, len(value),
                            self.n_nodes - idx)
        else:
            typ, flags, data = scalar_bytes(value)
            off = len(self._data) - byte_base
            self._data += data
            nbytes = len(data) if not flags & F_NFC else len(value.encode("utf-8", "surrogatepass"))
            self._nodes += _NODE.pack(typ, flags, 0, key, off, nbytes)
            if self.keep_objects:
                self._objs.append(value)

    # -- device view ----------------------------------------------------------

    def arrays(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(nodes[N] NODE_DTYPE, data u8[B], refs i64[E,2] = (node_base, byte_base))."""
        if self._frozen is None:
            nodes = np.frombuffer(bytes(self._nodes), dtype=NODE_DTYPE).copy() if self._nodes \
                else np.zeros(1, NODE_DTYPE)
            data = np.frombuffer(bytes(self._data) or b"\0", dtype=np.uint8).copy()
            refs = np.array(self._refs, dtype=np.int64).reshape(-1, 2)
            self._frozen = (nodes, data, refs)
        return self._frozen

    def __len__(self) -> int:
        return len(self._refs)

    # -- host decode ------------------------------------------------------------

    def node_object(self, event: int, node: int) -> Any:
        base = self._refs[event][0]
        if self.keep_objects:
            return self._objs[base + node]
        nodes, data, refs = self.arrays()
        return decode_node(nodes, data, int(refs[event, 0]), int(refs[event, 1]), node, self.keys)

    def node_type(self, event: int, node: int) -> int:
        return self._nodes[16 * (self._refs[event][0] + node)]

    def path_of(self, event: int, node: int) -> tuple:
        nodes, _, refs = self.arrays()
        return path_to_node(nodes, int(refs[event, 0]), node, self.keys)


def decode_node(nodes: np.ndarray, data: np.ndarray, node_base: int, byte_base: int,
                node: int, keys: KeyTable) -> Any:
    """Rebuild the raw Python value of a tape node (arrays-only tapes)."""
    i = node_base + node
    typ, flags = int(nodes["type"][i]), int(nodes["flags"][i])
    a, b = int(nodes["a"][i]), int(nodes["b"][i])
    if typ == T_NULL:
        return None
    if typ == T_TRUE:
        return True
    if typ == T_FALSE:
        return False
    if typ in (T_INT, T_FLOAT, T_STR):
        raw = bytes(data[byte_base + a: byte_base + a + b])
        if typ == T_STR:
            return raw.decode("utf-8", "surrogatepass")
        if typ == T_INT:
            return float(int(raw)) if flags & F_FLOATSRC else int(raw)
        return float(raw)
    child = node + 1
    if typ == T_LIST:
        out = []
        for _ in range(a):
            out.append(decode_node(nodes, data, node_base, byte_base, child, keys))
            child += _size(nodes, node_base + child)
        return out
    out_d = {}
    for _ in range(a):
        out_d[keys.names[int(nodes["key"][node_base + child])]] = \
            decode_node(nodes, data, node_base, byte_base, child, keys)
        child += _size(nodes, node_base + child)
    return out_d


def _size(nodes: np.ndarray, i: int) -> int:
    return int(nodes["b"][i]) if nodes["type"][i] >= T_LIST else 1


def path_to_node(nodes: np.ndarray, node_base: int, node: int, keys: KeyTable) -> tuple:
    """The key/index path from the payload root to ``node`` (pre-order index)."""
    path: list = []
    cur = 0
    while cur != node:
        i = node_base + cur
        typ, n = int(nodes["type"][i]), int(nodes["a"][i])
        child = cur + 1
        for ordinal in range(n):
            size = _size(nodes, node_base + child)
            if child <= node < child + size:
                path.append(keys.names[int(nodes["key"][node_base + child])]
                            if typ == T_DICT else ordinal)
                cur = child
                break
            child += size
        else:  # pragma: no cover - corrupt tape
            raise ValueError("node is not inside the tape")
    return tuple(path)


def leaf_str_of(value: Any) -> str | None:
    """``_leaf_str`` (mappings.py:197-204): text of a number or string leaf."""
    if isinstance(value, str):
        return value
    if isinstance(value, bool) or not isinstance(value, (int, float)):
        return None
    if isinstance(value, float) and value.is_integer():
        return str(int(value))
    return str(value)


class ArrayTapes:
    """Read-only arena view over (nodes, data, refs) arrays, for decoding."""

    def __init__(self, nodes: np.ndarray, data: np.ndarray, refs: np.ndarray, keys: KeyTable):
        self.nodes, self.data, self.refs, self.keys = nodes, data, refs, keys

    def arrays(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        return self.nodes, self.data, self.refs

    def node_object(self, event: int, node: int) -> Any:
        return decode_node(self.nodes, self.data, int(self.refs[event, 0]),
                           int(self.refs[event, 1]), node, self.keys)
