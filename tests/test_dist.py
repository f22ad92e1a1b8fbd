"""The N>1 path: one process per GPU, NCCL halo exchange.

CPU (gloo, world size 2): every rank derives the same decomposition from the
same domain with no communication (the reference's partition is a pure
function of the domain, decomp.hpp:65-188), and the per-rank views the
engine would build (own sites, neighbour lists, cut-link counts) are
consistent across ranks.

GPU (>= 2 devices): torchrun-style ranks running Simulation.distributed with
NCCL send/recv must reproduce the single-process result bit for bit.
"""
import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest

import cases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_ranks(script, world, env_extra=None, timeout=300):
    """Runs `script` as `world` ranks; a rank still running at the deadline
    (e.g. waiting on a peer that died) is killed with all the others."""
    import time
    deadline = time.time() + timeout
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "tests")]))
        env.update(env_extra or {})
        procs.append(subprocess.Popen([sys.executable, "-c", script], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=max(1.0, deadline - time.time()))
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            out, _ = p.communicate()
            out += "\n[test harness] killed at the deadline"
        outs.append((p.returncode, out))
    return outs


GLOO_SCRIPT = textwrap.dedent("""
    import os, hashlib, json
    import numpy as np
    import torch, torch.distributed as td
    import cases, impls
    td.init_process_group("gloo")
    rank, world = td.get_rank(), td.get_world_size()
    P = impls.product()
    d = P.build_bifurcation(4, 3, 12, 12)
    W = 4
    p = P.partition(d, W)
    dig = json.dumps(cases.partition_digest(p), sort_keys=True)
    # ranks own workers rank, rank+world, ...: their local views
    mine = {w: dict(n=len(p.parts[w].sites), nb=p.parts[w].neighbors) for w in range(rank, W, world)}
    objs = [None] * world
    td.all_gather_object(objs, (dig, mine))
    assert all(o[0] == objs[0][0] for o in objs), "ranks disagree on the decomposition"
    views = {}
    for o in objs:
        views.update(o[1])
    assert sorted(views) == list(range(W))
    assert sum(v["n"] for v in views.values()) == d.n_sites()
    for w, v in views.items():
        for nb in v["nb"]:
            assert w in views[nb]["nb"], "neighbour relation not symmetric"
    td.barrier()
    td.destroy_process_group()
    print("OK", rank, flush=True)
""")


def test_gloo_two_ranks_agree_on_decomposition():
    outs = _run_ranks(GLOO_SCRIPT, 2)
    for rc, out in outs:
        assert rc == 0, out
        assert "OK" in out


NCCL_SCRIPT = textwrap.dedent("""
    import os, types
    import numpy as np
    import torch, torch.distributed as td
    import cases, impls
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    td.init_process_group("gloo")
    P = impls.product()
    uid = P.Simulation.nccl_unique_id() if rank == 0 else bytes(128)
    obj = [uid]
    td.broadcast_object_list(obj, 0)
    run = dict(domain="bif_4_3_12_12", bcs=("bif", "smoke_inlet"), tau=0.8, dt=1e-3, W=world, steps=60,
               noise=(11, 0.01))
    d = cases.make_domain(P, cases.DOMAINS[run["domain"]])
    kw = dict(tau=0.8, dt_s=1e-3, workers=world, capture_period=20, observe_iolets=True)
    # 0 NCCL, 1 fused P2P, 2 AA single buffer (P2P in place); 3/4/5 the same
    # three built slab-locally from a geometry source; 6/7 the pull scheme
    # (update_pull + fill_send_slots) over NCCL / fused P2P
    mode = int(os.environ["HALO"])
    base = mode % 3 if mode < 6 else mode - 6
    prm = P.EngineParams(devices=[rank], halo_mode=min(base, 1), storage=1 if base == 2 else 0,
                         scheme=1 if mode >= 6 else 0, **kw)
    pa = None
    if mode >= 3:
        src = P.Source.bifurcation(4, 3, 12, 12)
        sim = P.Simulation.distributed(src, cases.make_bcs(P, run["bcs"]), prm, rank, world, obj[0])
        assert sim.slab_local() and sim.n_sites() == d.n_sites()
        win = src.window(world, rank)
        parts = [types.SimpleNamespace(sites=np.zeros(0, np.int64)) for _ in range(world)]
        parts[rank] = types.SimpleNamespace(sites=win["global_index"][win["part"].parts[rank].sites])
        pa = types.SimpleNamespace(n_workers=world, parts=parts)
    else:
        sim = P.Simulation.distributed(d, cases.make_bcs(P, run["bcs"]), prm, rank, world, obj[0])
    cases.apply_noise(P, sim, cases.noise_for(d.n_sites(), *run["noise"]), pa)
    sim.run(25)
    sim.run(run["steps"] - 25)
    # snapshot, captures and iolet series are assembled across ranks
    got = (cases.h(sim.snapshot_fields()), [(c.step, cases.h(c.fields)) for c in sim.cache()],
           {k: [cases.h(a) for a in v] for k, v in sim.series().items() if k != "rows"})
    ref = P.Simulation(d, cases.make_bcs(P, run["bcs"]), P.EngineParams(devices=[rank], **kw))
    cases.apply_noise(P, ref, cases.noise_for(d.n_sites(), *run["noise"]))
    ref.run(25)
    ref.run(run["steps"] - 25)
    want = (cases.h(ref.snapshot_fields()), [(c.step, cases.h(c.fields)) for c in ref.cache()],
            {k: [cases.h(a) for a in v] for k, v in ref.series().items() if k != "rows"})
    assert got == want, (got[1], want[1])
    td.barrier()
    print("OK", rank)
""")


@pytest.mark.gpu
@pytest.mark.parametrize("halo", ["0", "1", "2", "3", "4", "5", "6", "7"])
def test_nccl_ranks_match_single_process(halo):
    """halo 0: NCCL send/recv + PostReceive; 1: fused NVLink P2P stores into
    IPC-mapped neighbour buffers, flag-synchronised; 2: AA single buffer.
    3/4/5: the same built slab-locally (each rank classifies only its own
    slices of a geometry source).  6/7: the pull scheme over
    NCCL / fused P2P."""
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = 4 if n >= 4 else 2
    outs = _run_ranks(NCCL_SCRIPT, world, env_extra={"HALO": halo})
    for rc, out in outs:
        assert rc == 0, out
        assert "OK" in out


DEAD_RANK_SCRIPT = textwrap.dedent("""
    import os, time
    import torch, torch.distributed as td
    import cases, impls
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    td.init_process_group("gloo")
    P = impls.product()
    uid = P.Simulation.nccl_unique_id() if rank == 0 else bytes(128)
    obj = [uid]
    td.broadcast_object_list(obj, 0)
    d = P.build_pipe(6, 60)
    bcs = cases.make_bcs(P, ("pressure", 0.34, cases.CS2))
    prm = P.EngineParams(devices=[rank], workers=world, halo_mode=int(os.environ["HALO"]), exchange_timeout_s=5.0)
    sim = P.Simulation.distributed(d, bcs, prm, rank, world, obj[0])
    sim.run(3)
    td.barrier()
    if rank == world - 1:
        # this worker stops stepping: over NCCL it dies; over the fused P2P
        # halo it stays alive but stuck (a dead exporter's IPC memory must not
        # be written by the survivor's already-queued step), then exits
        if os.environ["HALO"] == "0":
            os._exit(0)
        time.sleep(40)
        os._exit(0)
    t0 = time.time()
    print("running", flush=True)
    try:
        sim.run(500)
        print("NO ERROR")
    except P.Error as e:
        print("ERROR after %.1f s: %s" % (time.time() - t0, e), flush=True)
    sim.close()  # teardown must not hang on streams blocked by the dead peer
    print("CLOSED", flush=True)
    os._exit(0)
""")


@pytest.mark.gpu
@pytest.mark.parametrize("halo", ["0", "1"])
def test_dead_rank_fails_within_timeout(halo):
    """A worker that dies (NCCL) or stops stepping (fused P2P) is reported by
    its neighbour within exchange_timeout_s of the last completed step, with
    the reference's message (Mailbox::take, engine.hpp:92-101), and the
    survivor's teardown completes."""
    import re
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    outs = _run_ranks(DEAD_RANK_SCRIPT, 2, env_extra={"HALO": halo}, timeout=120)
    rc, out = outs[0]
    assert rc == 0 and "CLOSED" in out, out
    m = re.search(r"ERROR after ([0-9.]+) s: (.*)", out)
    assert m, out
    assert float(m.group(1)) < 30.0, out
    assert "exchange failure" in m.group(2), out
    if halo == "1":
        assert "timed out waiting for neighbor 1" in m.group(2), out
