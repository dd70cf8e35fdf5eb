"""N > 1 plumbing on CPU: two processes over torch.distributed gloo (127.0.0.1) run the
reference oracle on their variation shards with the allgather the bench uses
(paper_2512_16896_b200.dist.torch_allgather); the concatenated shards must equal the
single-process run bit for bit (accepted attempt indices, valid masks, poses)."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out_dir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2512_16896_b200 import scenes
    from paper_2512_16896_b200.dist import shard_bounds, torch_allgather
    from paper_2512_16896_b200.world import Shard

    scene = scenes.tabletop_mixed(n, n_objects=9)
    b = shard_bounds(n, world)
    r = O.generate(scene, 3, threads=1, shard=Shard(b[rank], b[rank + 1], rank, world, torch_allgather(world)))
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), accepted=r["accepted"], valid=r["valid"], poses=r["poses"])
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_equal_single(ref, tmp_path):
    import torch.multiprocessing as mp

    n, world = 240, 2
    mp.start_processes(_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world,
                       start_method="spawn")
    from paper_2512_16896_b200 import scenes

    whole = ref.generate(scenes.tabletop_mixed(n, n_objects=9), 3, threads=1)
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    assert np.array_equal(np.concatenate([p["accepted"] for p in parts], axis=1), whole["accepted"])
    assert np.array_equal(np.concatenate([p["valid"] for p in parts]), whole["valid"])
    assert np.array_equal(np.concatenate([p["poses"] for p in parts], axis=1), whole["poses"])
