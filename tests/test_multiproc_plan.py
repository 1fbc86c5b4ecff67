"""Host-side logic of the N>1 path, on CPU: every process must derive identical
cross-process message layouts (CUDA-IPC inbox/outbox offsets) and NCCL stage groups.
A world_size-2 gloo job exchanges each process's own view and checks agreement; the
full G in {1,2,4,8} matrix is checked in-process."""
import ctypes as C
import json
import os

import pytest

from paper_2107_06925_b200 import _lib
from paper_2107_06925_b200 import pipesim as P

_lib.register("ck_link_plan", C.c_int, [C.c_char_p, C.c_int, C.c_longlong, C.POINTER(C.c_void_p)])


def plan(cfg, per, msg_bytes=8 << 20):
    text = P.generate_json(cfg, None, -1)
    return json.loads(_lib.call_str(_lib.lib().ck_link_plan, text.encode(), per, msg_bytes))


CFGS = [P.PipelineConfig("chimera", 4, 2, 4, 4, 1), P.PipelineConfig("chimera", 8, 1, 8, 1, 1),
        P.PipelineConfig("chimera", 8, 1, 16, 1, 2), P.PipelineConfig("gpipe", 4, 2, 4, 2)]


@pytest.mark.parametrize("cfg", CFGS)
def test_plan_invariants(cfg):
    ranks = cfg.W * cfg.D
    for G in (1, 2, 4, 8):
        if ranks % G:
            continue
        per = ranks // G
        pl = plan(cfg, per)
        assert pl["procs"] == G
        for m in pl["messages"]:
            k = str(m["key"])
            pq, cq = m["producer"] // per, m["consumer"] // per
            assert k in pl["inbox"][cq]["slots"]  # receive slot on the consumer
            assert (k in pl["outbox"][pq]["slots"]) == (pq != cq)  # ack only across processes
            for q in range(G):
                if q != cq:
                    assert k not in pl["inbox"][q]["slots"]
        for q in range(G):  # slots are disjoint and inside the arena
            spans = sorted((v[0], v[0] + (8 << 20)) for v in pl["inbox"][q]["slots"].values())
            assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:]))
            assert all(v[1] + 4 <= pl["inbox"][q]["bytes"] for v in pl["inbox"][q]["slots"].values())
            # the stage-collective rendezvous flags: distinct, 4-byte aligned, past every
            # message buffer and flag, inside the arena
            rf = pl["inbox"][q]["ready_flags"]
            assert len(rf) == cfg.D * G and len(set(rf)) == len(rf) and all(r % 4 == 0 for r in rf)
            used = [v[0] + (8 << 20) for v in pl["inbox"][q]["slots"].values()] + \
                   [v[1] + 4 for v in pl["inbox"][q]["slots"].values()]
            assert min(rf) >= max(used, default=0) and max(rf) + 4 <= pl["inbox"][q]["bytes"]
        # every stage is held by 2f*W ranks (perfmodel::replicas_per_stage)
        if cfg.scheme == "chimera":
            holders = set()
            for g in pl["stage_groups"]:
                holders |= set(g)
            assert holders == set(range(G))


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = CFGS[0]
    per = cfg.W * cfg.D // world
    mine = plan(cfg, per)  # each process computes the plan independently
    views = [None] * world
    dist.all_gather_object(views, mine)
    ok = all(v == views[0] for v in views)
    # process q's own inbox as computed by q equals what every other process assumes
    ok = ok and all(views[q]["inbox"][q] == views[0]["inbox"][q] for q in range(world))
    out.put((rank, ok))
    dist.destroy_process_group()


def test_gloo_world2_agreement():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 200
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]
