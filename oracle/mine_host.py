"""CPU mine() with Phase II (TEST INFRASTRUCTURE / CPU BASELINE ONLY: used by
bench.py's cpu_baseline of the Phase II mining object, never by the product
package).

Follows /root/reference/pkg/src/spectool/mining.py:248-292: Phase I counts
from the C oracle (oracle_mine_counts, the restatement pinned by
tests/test_mine_oracle.py), then for every (context, target) that clears
sigma and tau on counts, the reference's Phase II on the host -- every
stream rescanned for the context's followed occurrences of the target
(_collect_occurrences, :215-227), infer_mapping (mappings.py:276-417) and
mapping_holds (:202-212) in their Python restatement (phase2.py) -- then
the reference order (:105-111).  One core.
"""

from __future__ import annotations

import numpy as np

from . import bridge


def mine_host(sessions, cfg) -> list:
    from paper_2603_18897_b200 import phase2
    from paper_2603_18897_b200.events import signature_of
    from paper_2603_18897_b200.mine_engine import (SEG_START, decode_context, match_events)
    from paper_2603_18897_b200.mining import MatchRelation, PatternTuple, pattern_sort_key
    from paper_2603_18897_b200.packing import SigTable

    streams = [s.tool_events() for s in sessions]
    sigs = SigTable(sorted({e.tool_type for st in streams for e in st}))
    tok = []
    for st in streams:
        for i, e in enumerate(st):
            t = sigs.sig(e.tool_type, e.status)
            tok.append(int(np.int32(t | SEG_START)) if i == 0 else t)
    S = max(sigs.n_sigs, 2)
    rel = 0 if cfg.match_relation is MatchRelation.ANCHORED_SUBSEQUENCE else 1
    tables = bridge.mine_counts(np.array(tok, np.int32), S, cfg.k, rel)
    cands = bridge.select_candidates(*tables, S, cfg.k, cfg.sigma, cfg.tau)
    sig_streams = [[signature_of(e) for e in st] for st in streams]
    out = []
    for tool, cidx, support, n_match, follow in cands:
        context = tuple(sigs.signature(x) for x in decode_context(cidx, S, cfg.k))
        target = sigs.tools[tool]
        hits, mapping = follow, None
        if follow >= 2:
            occ = []
            for st, sg in zip(streams, sig_streams):
                for a in range(len(st) - 1):
                    if st[a + 1].tool_type != target:
                        continue
                    m = match_events(st, sg, a, context, cfg.k, cfg.match_relation)
                    if m is not None:
                        occ.append((m, st[a + 1]))
            mapping = phase2.infer_mapping(occ, cfg.validation_fraction)
            if mapping is not None:
                hits = sum(1 for m, nxt in occ if phase2.mapping_holds(mapping, m, nxt))
        p = hits / n_match
        if p >= cfg.tau:
            out.append(PatternTuple(context=context, target=target, mapping=mapping, p=p,
                                    support=support))
    out.sort(key=pattern_sort_key)
    return out
