"""torchrun worker for test_sharded_mining_equals_single_device: each rank
mines whole-session shards of one columnar corpus with mine_columnar(group=)
(gloo, ranks sharing GPU 0) and writes its pattern list for the test."""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_18897_b200.mine_engine import mine_columnar  # noqa: E402
from paper_2603_18897_b200.mining import MiningConfig  # noqa: E402
from paper_2603_18897_b200.packing import SigTable  # noqa: E402
from paper_2603_18897_b200.synth import C4_TOOLS, columnar_corpus  # noqa: E402


def main_sessions(out_path):
    """mine() with payload mappings over session shards (mine_golden's
    mapped corpora)."""
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import golden_io as G
    from paper_2603_18897_b200.mappings import mapping_to_json
    from paper_2603_18897_b200.mining import MatchRelation, mine

    dist.init_process_group("gloo")
    rank = dist.get_rank()
    torch.cuda.set_device(0)
    results = []
    for corpus in G.golden("mine_golden.json")["mapped"]:
        sessions = [G.session(s) for s in corpus["sessions"]]
        c = corpus["config"]
        cfg = MiningConfig(k=c["k"], sigma=c["sigma"], tau=c["tau"],
                           match_relation=MatchRelation(c["match_relation"]))
        cut = len(sessions) // 3
        shard = sessions[:cut] if rank == 0 else sessions[cut:]
        pats = mine(shard, cfg, group=dist.group.WORLD)
        results.append([[[[s.tool_type, s.status.value] for s in p.context], p.target,
                         mapping_to_json(p.mapping) if p.mapping else None, p.p, p.support]
                        for p in pats])
    gathered = [None, None]
    dist.all_gather_object(gathered, results)
    if rank == 0:
        with open(out_path, "w") as fh:
            json.dump({"0": gathered[0], "1": gathered[1]}, fh)
    dist.barrier()
    dist.destroy_process_group()


def main(out_path):
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    torch.cuda.set_device(0)
    c = columnar_corpus(400_000, seed=31)
    bounds = np.flatnonzero(c["session"][1:] != c["session"][:-1]) + 1
    cut = int(bounds[len(bounds) // 3])  # a session boundary
    lo, hi = (0, cut) if rank == 0 else (cut, len(c["session"]))
    shard = {k: torch.from_numpy(np.ascontiguousarray(v[lo:hi])).cuda() for k, v in c.items()}
    cfg = MiningConfig(k=3, sigma=5, tau=0.3)
    pats = mine_columnar(shard, SigTable(C4_TOOLS), cfg, group=dist.group.WORLD)
    sliced = mine_columnar(shard, SigTable(C4_TOOLS), cfg, group=dist.group.WORLD, tail="sliced")
    assert sliced == pats, "sliced tail differs from the all-reduce tail"
    rows = [[[[s.tool_type, s.status.value] for s in p.context], p.target, p.p, p.support]
            for p in pats]
    gathered = [None, None]
    dist.all_gather_object(gathered, rows)
    if rank == 0:
        with open(out_path, "w") as fh:
            json.dump({"0": gathered[0], "1": gathered[1]}, fh)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "sessions":
        main_sessions(sys.argv[1])
    else:
        main(sys.argv[1])
