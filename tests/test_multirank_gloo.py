"""Multi-process (world_size 2 and 4, gloo, CPU) execution of the planner's
per-stage instruction streams with real asynchronous point-to-point
messaging: each rank walks ITS stage's stream from tpipe_plan_create exactly
like the NCCL runtime does (SEND = isend on the channel, SEND_WAIT = wait on
message j's send, RECV = blocking recv), carrying a scalar "activation"
through F ops and a scalar "gradient" through B ops. Checks: every message
arrives on the channel the plan names, in FIFO order with the (chunk, mb)
the sender produced; the step completes (no deadlock with real async
delivery); the values match a sequential evaluation of the same dataflow.
"""

import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def f_fn(x, s, c):      # stage function used for the forward scalar
    return 2.0 * x + (s + 1) + 100.0 * c


def b_fn(g, s, c):      # and for the backward scalar
    return 0.5 * g + (s + 1) * 10.0 + c


def sequential_reference(p, v, m):
    """Scalar dataflow of the pipeline evaluated in plain order."""
    res = {}
    for i in range(1, m + 1):
        x = float(i)
        for c in range(1, v + 1):
            for s in range(p):
                x = f_fn(x, s, c)
                res[("F", s, c, i)] = x
        g = x                                           # "loss" seeds the backward
        for c in range(v, 0, -1):
            for s in range(p - 1, -1, -1):
                g = b_fn(g, s, c)
                res[("B", s, c, i)] = g
    return res


def _worker(rank, world, port, strategy, m, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import sys
        sys.path.insert(0, ROOT)
        from paper_2503_03182_b200 import plan as P
        L = 2 * world
        plan = P.Plan(P.Model(L, 64, 4, 256, 128, 32, 2), world, m, strategy=strategy)
        v, p, s = plan.v, world, rank
        ops, _bufs = plan.ops(s)
        chan_id = {ch: n for n, ch in enumerate(plan.channels)}
        local_in, local_gin = {}, {}
        inbox_act, inbox_grad = {}, {}
        pending = {}                       # (channel, msg) -> isend work
        vals = {}
        for op in ops:
            k = op["kind"]
            if k == "SEND_WAIT":
                pending.pop((op["channel"], op["msg"])).wait()
            elif k in ("RECV_ACT", "RECV_GRAD"):
                ch = op["channel"]
                buf = torch.zeros(3, dtype=torch.float64)
                dist.recv(buf, src=op["peer"], tag=chan_id[ch])
                c_sent, mb_sent, val = int(buf[0]), int(buf[1]), float(buf[2])
                assert (c_sent, mb_sent) == (op["chunk"], op["mb"]), (s, op, c_sent, mb_sent)
                (inbox_act if k == "RECV_ACT" else inbox_grad)[(op["chunk"], op["mb"])] = val
            elif k == "F":
                c, i = op["chunk"], op["mb"]
                if s == 0 and c == 1:
                    x = float(i)
                elif (c, i) in inbox_act:
                    x = inbox_act.pop((c, i))
                else:
                    x = local_in.pop((c, i))          # p == 1 local hand-off
                y = f_fn(x, s, c)
                vals[("F", s, c, i)] = y
                if s == p - 1 and c == v:
                    local_gin[(c, i)] = y              # loss seeds the backward
                elif s == p - 1 and p == 1:
                    local_in[(c + 1, i)] = y
                else:
                    pending_val = y
                    vals[("out", c, i)] = pending_val
            elif k == "B":
                c, i = op["chunk"], op["mb"]
                g = inbox_grad.pop((c, i)) if (c, i) in inbox_grad else local_gin.pop((c, i))
                gy = b_fn(g, s, c)
                vals[("B", s, c, i)] = gy
                if s == 0 and c > 1 and p == 1:
                    local_gin[(c - 1, i)] = gy
                vals[("gout", c, i)] = gy
            elif k in ("SEND_ACT", "SEND_GRAD"):
                c, i = op["chunk"], op["mb"]
                val = vals[("out", c, i)] if k == "SEND_ACT" else vals[("gout", c, i)]
                cons_c = c
                if k == "SEND_ACT" and s == p - 1:
                    cons_c = c + 1                     # wrap edge p-1 -> 0
                if k == "SEND_GRAD" and s == 0:
                    cons_c = c - 1                     # wrap edge 0 -> p-1
                t = torch.tensor([cons_c, i, val], dtype=torch.float64)
                pending[(op["channel"], op["msg"])] = dist.isend(t, dst=op["peer"],
                                                                tag=chan_id[op["channel"]])
        assert not pending and not inbox_act and not inbox_grad
        ref = sequential_reference(p, v, m)
        for key, val in vals.items():
            if key[0] in ("F", "B"):
                assert abs(val - ref[key]) <= 1e-9 * max(1.0, abs(ref[key])), (key, val, ref[key])
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface to the parent
        import traceback
        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("strategy", ["tpipe", "tpipe_trecomp", "1f1b", "interleave", "interleave_trecomp"])
def test_streams_execute_over_gloo(world, strategy):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, strategy, 8, errq))
             for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=120)
    alive = [pr for pr in procs if pr.is_alive()]
    for pr in alive:
        pr.kill()
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not alive, "deadlock: ranks did not finish"
    assert not errs, "\n".join(errs)
    assert all(pr.exitcode == 0 for pr in procs)
