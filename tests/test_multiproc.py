"""CPU, world_size 2 (gloo): the N>1 path of SURVEY.md §8 E1.

* prompt sharding keeps GRPO groups on one rank and covers every request once;
* the prompt-sharded KD step -- replicated selection over global indices, rank-local K5
  gradients, torch.distributed all-reduce -- reproduces the compiled reference's kd_update
  (learner.cpp:98-160) on both ranks. The rank-local gradient here is the CPU oracle (no GPU
  in this container); on the B200 the same code path runs rs_kd_grad_tabular
  (tests/test_tabular_gpu.py::test_distributed_kd_step_on_gpu)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_golden

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def gloo_all_reduce(vec):
    """Host-reduce hook of kd_step_distributed (the library's NCCL communicator on GPUs)."""
    import torch
    t = torch.tensor(vec, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.tolist()


def _worker(rank, port, case_idx, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_2510_26475_b200 as rb
        from paper_2510_26475_b200.distributed import kd_step_distributed, shard_requests
        from oracle_client import Oracle

        g = load_golden("kd_update.json")
        c = g["cases"][case_idx]
        buf = g["buffer"]
        mine = shard_requests(list(range(len(buf))), rank, WORLD, group_size=8)
        oracle = Oracle()

        def grad_fn(samples, weights):
            if not samples:
                return [0.0] * len(g["drafter"]["logits"]), 0.0
            out = oracle("kd_grad", drafter=g["drafter"], samples=samples, weights=list(weights))
            return out["grad"], out["loss"]

        p = c["policy"]
        mode = {"reward": rb.WeightMode.Reward, "uniform": rb.WeightMode.Uniform}[p["mode"]]
        pol = rb.KDPolicy(p["interval"], mode, p["clip_lo"], p["clip_hi"], p["lr"])
        res = kd_step_distributed([s["reward"] for s in buf], [len(s["response"]) for s in buf],
                                  [buf[i] for i in mine], mine, pol, rb.SelectionRng(c["selection_seed"]), 0.02,
                                  grad_fn, gloo_all_reduce)
        new = [z + gr * -p["lr"] for z, gr in zip(g["drafter"]["logits"], res.grad)]
        q.put((rank, mine, new, res.loss, res.samples_used, res.sim_time, res.selected))
    finally:
        dist.destroy_process_group()


def test_shard_requests_partition():
    from paper_2510_26475_b200.distributed import shard_requests
    reqs = list(range(32))
    shards = [shard_requests(reqs, r, 4, group_size=8) for r in range(4)]
    assert sorted(x for s in shards for x in s) == reqs
    for s in shards:
        assert all(len({x // 8 for x in s[i:i + 8]}) == 1 for i in range(0, len(s), 8))  # groups intact
    with pytest.raises(ValueError):
        shard_requests(list(range(10)), 0, 2, group_size=8)


@pytest.mark.parametrize("case_idx", [0, 1, 2])
def test_prompt_sharded_kd_step_matches_reference(oracle, case_idx):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, case_idx, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=120) for _ in range(WORLD)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = load_golden("kd_update.json")
    exp = g["cases"][case_idx]["out"]
    # both ranks hold the same updated drafter, equal to the reference's single-process update
    for _, mine, new, loss, used, sim, sel in outs:
        assert used == exp["samples_used"]
        assert loss == pytest.approx(exp["loss"], rel=1e-12)
        assert sim == pytest.approx(exp["sim_time"], rel=1e-12)
        assert max(abs(a - b) for a, b in zip(new, exp["logits"])) < 1e-12
    assert outs[0][2] == outs[1][2]
    assert sorted(outs[0][1] + outs[1][1]) == list(range(len(g["buffer"])))
    # the replicated selection is the reference's (oracle restatement checked against it)
    ref = oracle("kd_update", drafter=g["drafter"], buffer=g["buffer"], policy=g["cases"][case_idx]["policy"],
                 selection_seed=g["cases"][case_idx]["selection_seed"], cost_per_token=0.02)
    assert outs[0][6] == ref["selected"]


def _rdv_worker(rank, port, q):
    from paper_2510_26475_b200.distributed import _rendezvous
    payload = bytes(range(128)) if rank == 0 else None
    q.put((rank, _rendezvous(rank, WORLD, payload, "127.0.0.1", port, 30.0)))


def test_comm_id_rendezvous_two_ranks():
    """Comm.from_env's id hand-off: rank 0 serves the 128-byte NCCL id, rank 1 receives it."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rdv_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=60) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=30)
    assert got[0] == got[1] == bytes(range(128))


def test_bench_relaunches_under_torchrun(monkeypatch):
    """bench.py --gpus N outside a launcher re-runs itself as N ranks (torch.distributed.run)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    assert bench.relaunch(4) == 0
    cmd = calls[0]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "3"]
