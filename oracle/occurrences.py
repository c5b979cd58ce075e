"""CPU restatement of Phase II occurrence collection (TEST INFRASTRUCTURE
ONLY: the checker of paste_mine_occurrences in tests/, never imported by the
product package).

Follows /root/reference/pkg/src/spectool/mining.py:
  * :119-156  match_at -- the last context signature equals the anchor's;
              anchored: the rest embeds (rightmost, greedily from the anchor
              backwards) inside the k events ending at the anchor; contiguous
              suffix: the slice ending at the anchor equals the context;
  * :215-227  _collect_occurrences over every anchor of every stream, and
  * :277-279  mine()'s filter to the followed occurrences whose next event
              has the target tool.
Streams are the flagged token form (bit 31 = first event of a stream, token
= 2 * tool + success); positions are indices into the concatenated stream.
"""

from __future__ import annotations

import numpy as np


def occurrences(tok: np.ndarray, context: tuple, target_tool: int, k: int, contiguous: bool):
    """[(anchor, matched positions)] in stream order."""
    tok = np.asarray(tok, np.int64)
    start = tok < 0
    sig = tok & 0x7FFFFFFF
    n = len(tok)
    seg_start = np.zeros(n, np.int64)
    cur = 0
    for i in range(n):
        if start[i]:
            cur = i
        seg_start[i] = cur
    L = len(context)
    out = []
    for a in range(n - 1):
        if start[a + 1] or (sig[a + 1] >> 1) != target_tool or sig[a] != context[-1]:
            continue
        lo_stream = seg_start[a]
        if contiguous:
            s0 = a - L + 1
            if s0 < lo_stream or any(sig[s0 + i] != context[i] for i in range(L)):
                continue
            out.append((a, tuple(range(s0, a + 1))))
            continue
        lo = max(lo_stream, a - k + 1)
        picked = [a]
        j, p = L - 2, a - 1
        while j >= 0 and p >= lo:
            if sig[p] == context[j]:
                picked.append(p)
                j -= 1
            p -= 1
        if j < 0:
            out.append((a, tuple(reversed(picked))))
    return out
