"""Native shard communicator (sb_comm_*): the engine's multi-GPU exchange without PyTorch.

CPU: two processes over the TCP star (host exchange only): allgather / barrier / shard
bounds, and the reference oracle's shard protocol driven through the native callbacks must
equal the single-process run bit for bit. GPU: two engine processes on one B200 exchange
their FIFO round counts through CUDA-IPC-mapped count boards and stream memory waits; the
concatenated shards must equal the single engine bit for bit."""
import json
import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_ranks(script: str, world: int, port: int, out_dir: str, timeout: float = 240.0):
    """Launch `world` python processes running `script` with RANK / WORLD / PORT / OUT set;
    kill them all if any exceeds the timeout."""
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD=str(world), PORT=str(port), OUT=out_dir,
                   PYTHONPATH=ROOT)
        procs.append(subprocess.Popen([sys.executable, "-c", textwrap.dedent(script)], env=env,
                                      cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    outs = []
    try:
        for p in procs:
            out, _ = p.communicate(timeout=timeout)
            outs.append(out.decode(errors="replace"))
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-3000:]
    return outs


HOST_SCRIPT = """
import json, os
import paper_2512_16896_b200 as pkg
r, w, port = int(os.environ["RANK"]), int(os.environ["WORLD"]), int(os.environ["PORT"])
c = pkg.Comm(r, w, device=None, host="127.0.0.1", port=port, timeout_s=60)
g = c.allgather([r, 10 * r + 1, 2**63 + r])
c.barrier()
g2 = c.allgather([])
sh = c.shard(1001)
json.dump({"g": [str(v) for v in g], "g2": g2, "b": [sh.begin, sh.end, sh.rank, sh.world_size]},
          open(os.path.join(os.environ["OUT"], f"h{r}.json"), "w"))
c.close()
"""


def test_comm_host_exchange_three_ranks(tmp_path):
    world = 3
    _run_ranks(HOST_SCRIPT, world, _free_port(), str(tmp_path))
    want = [str(v) for r in range(world) for v in (r, 10 * r + 1, 2**63 + r)]
    bounds = [1001 * r // world for r in range(world + 1)]
    for r in range(world):
        d = json.load(open(tmp_path / f"h{r}.json"))
        assert d["g"] == want
        assert d["g2"] == []
        assert d["b"] == [bounds[r], bounds[r + 1], r, world]


def test_comm_rejects_bad_arguments(pkg):
    with pytest.raises(ValueError):  # std::invalid_argument
        pkg.Comm(2, 2, device=None, port=_free_port())
    with pytest.raises(ValueError):
        pkg.Comm(0, 0, device=None, port=_free_port())
    c = pkg.Comm(0, 1, device=None, port=_free_port())  # world 1: no sockets at all
    assert c.allgather([5, 6]) == [5, 6]
    c.barrier()
    sh = c.shard(10)
    assert (sh.begin, sh.end) == (0, 10)


ORACLE_SCRIPT = """
import os
import numpy as np
import paper_2512_16896_b200 as pkg
from oracle import oracle as O
from paper_2512_16896_b200 import scenes
r, w, port = int(os.environ["RANK"]), int(os.environ["WORLD"]), int(os.environ["PORT"])
c = pkg.Comm(r, w, device=None, host="127.0.0.1", port=port, timeout_s=60)
n = 240
scene = scenes.tabletop_mixed(n, n_objects=9)
res = O.generate(scene, 3, threads=1, shard=c.shard(n))
np.savez(os.path.join(os.environ["OUT"], f"r{r}.npz"), accepted=res["accepted"],
         valid=res["valid"], poses=res["poses"])
c.barrier()
"""


def test_native_comm_oracle_shards_equal_single(ref, tmp_path):
    world = 2
    _run_ranks(ORACLE_SCRIPT, world, _free_port(), str(tmp_path))
    from paper_2512_16896_b200 import scenes

    whole = ref.generate(scenes.tabletop_mixed(240, n_objects=9), 3, threads=1)
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    assert np.array_equal(np.concatenate([p["accepted"] for p in parts], axis=1), whole["accepted"])
    assert np.array_equal(np.concatenate([p["valid"] for p in parts]), whole["valid"])
    assert np.array_equal(np.concatenate([p["poses"] for p in parts], axis=1), whole["poses"])


ENGINE_SCRIPT = """
import os, json
import numpy as np
import paper_2512_16896_b200 as pkg
from paper_2512_16896_b200 import scenes
r, w, port = int(os.environ["RANK"]), int(os.environ["WORLD"]), int(os.environ["PORT"])
c = pkg.Comm(r, w, device=0, host="127.0.0.1", port=port, timeout_s=120)
out = {"waits": c.uses_stream_waits()}
for name, make, seed in (("fifo", lambda n: scenes.tabletop_boxes(n_instances=n, n_objects=10, attempts=64), 5),
                         ("mixed", lambda n: scenes.tabletop_mixed(n, n_objects=9), 3)):
    n = int(os.environ.get("N", "3000"))
    eng = pkg.Engine(make(n), shard=c.shard(n), device=0)
    for rep in range(2):  # a second (warm) run reuses the boards' later epochs
        g = eng.generate(run_seed=seed + rep)
        np.savez(os.path.join(os.environ["OUT"], f"{name}{rep}_r{r}.npz"), accepted=g.accepted,
                 valid=g.valid, poses=g.poses)
    eng.close()
json.dump(out, open(os.path.join(os.environ["OUT"], f"e{r}.json"), "w"))
c.barrier()
"""


@pytest.mark.gpu
@pytest.mark.parametrize("spin", [False, True])
def test_native_comm_engine_processes_equal_single(gpu, tmp_path, spin, monkeypatch):
    from paper_2512_16896_b200 import scenes

    monkeypatch.setenv("SB_COMM_SPIN", "1" if spin else "0")
    world, n = 2, 3000
    _run_ranks(ENGINE_SCRIPT, world, _free_port(), str(tmp_path), timeout=300)
    waits = json.load(open(tmp_path / "e0.json"))["waits"]
    assert waits == (not spin)
    for name, make, seed in (("fifo", lambda n: scenes.tabletop_boxes(n_instances=n, n_objects=10, attempts=64), 5),
                             ("mixed", lambda n: scenes.tabletop_mixed(n, n_objects=9), 3)):
        eng = gpu.Engine(make(n), device=0)
        for rep in range(2):
            whole = eng.generate(run_seed=seed + rep)
            parts = [np.load(tmp_path / f"{name}{rep}_r{r}.npz") for r in range(world)]
            assert np.array_equal(np.concatenate([p["accepted"] for p in parts], axis=1), whole.accepted), name
            assert np.array_equal(np.concatenate([p["valid"] for p in parts]), whole.valid), name
            assert np.array_equal(np.concatenate([p["poses"] for p in parts], axis=1), whole.poses), name
        eng.close()
