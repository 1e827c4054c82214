"""Tensor-parallel host plumbing on CPU: config validation of the
shard split, and the NCCL unique-id hand-off between ranks over torch.distributed
(gloo, world size 2, 127.0.0.1) exactly as bench.py does it under torchrun.
The sharded math itself is checked on the GPU (test_gpu_parity.py::test_tp_*)."""
import os
import socket

import pytest

from paper_2604_23467_b200 import graphrt as g


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("kw,msg", [
    (dict(arch=g.ARCH_LLAMA, n_heads=4, tp_size=3), "n_heads must be divisible"),
    (dict(arch=g.ARCH_LLAMA, n_heads=4, tp_size=2, tp_rank=2), "tp_rank must be in"),
    (dict(arch=g.ARCH_LLAMA, n_heads=4, tp_size=2, vocab_size=255), "vocab_size must be divisible"),
    (dict(arch=g.ARCH_LLAMA, n_heads=4, tp_size=4, d_ff_=72), "d_ff / tp_size"),
    (dict(arch=g.ARCH_REF, n_heads=4, tp_size=2), "LLaMA arch"),
])
def test_tp_config_validation(kw, msg):
    with pytest.raises(g.Error) as ei:
        g.Model(g.ModelConfig(**kw))
    assert msg in str(ei.value)


def _rank_main(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    obj = [g.tp_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    uid = obj[0]
    gathered = [None] * world
    dist.all_gather_object(gathered, uid)
    out[rank] = (len(uid), all(x == gathered[0] for x in gathered))
    dist.destroy_process_group()


def test_tp_unique_id_handoff_gloo():
    import torch.multiprocessing as mp
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rank_main, args=(world, port, out), nprocs=world, join=True)
    assert dict(out) == {0: (128, True), 1: (128, True)}
