"""Real NCCL on the decode path.

* One GPU: a 1-rank NCCL group.  With a communicator attached the plans hold
  the in-graph collectives (allreduce of x after Wo and down, allgather of the
  logits; the prefill's [P, d] allreduces), which on one rank are identities --
  so the NCCL capture path (stream capture into the bucket graphs, the batched
  prefill graph, and the conditional bodies of the device-resident loop) runs
  on real NCCL and must reproduce the plain model bit for bit.
* Two or more GPUs (skipped on a 1-GPU box): one process per GPU, tensor
  parallel over min(device_count, 8) ranks, NCCL unique id handed over a queue,
  compared with the single-GPU model.
"""
import numpy as np
import pytest

from paper_2604_23467_b200 import graphrt as g
from paper_2604_23467_b200.bench_harness import make_prompt

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

KW = dict(arch=g.ARCH_LLAMA, n_layers=2, d_model=4096, n_heads=32, vocab_size=32000, max_seq_len=256, d_ff_=11008,
          weight_dtype=g.BF16, kv_dtype=g.BF16, init=g.INIT_PHILOX, seed=21)


def _cache(**kw):
    return g.CacheConfig(bucket_size=32, warmup_hi=2, batched_prefill=True, **kw)


def test_one_rank_nccl_group_in_graph_matches_plain_model():
    torch.cuda.init()  # NCCL (dlopen'ed by soname) binds to the one torch loaded
    prompt = make_prompt(42, 20, 32000)
    plain = g.Session(g.ModelConfig(**KW), _cache())
    want = plain.run(g.GenerationRequest(prompt=prompt, gen_len=40))
    want_logits = plain.logits()
    m = g.Model(g.ModelConfig(**KW))
    m.attach_nccl(g.tp_unique_id())  # tp_size 1: a 1-rank group
    assert m.tp_info() == (1, 0, True)  # x moved into an NCCL symmetric window
    s = g.Session(m, _cache())
    r1 = s.run(g.GenerationRequest(prompt=prompt, gen_len=40))  # eager misses + inline captures (NCCL nodes)
    r2 = s.run(g.GenerationRequest(prompt=prompt, gen_len=40))  # prefill graph + step graphs replayed
    assert r1.tokens == want.tokens and r2.tokens == want.tokens
    assert r2.prefill_paths == [g.StepPath.BatchedReplayed] * len(prompt)
    assert all(p == g.StepPath.Replayed for p in r2.decode_paths)
    assert np.array_equal(s.logits(), want_logits)
    # the device-resident loop with NCCL nodes inside its conditional bodies
    r3 = s.run(g.GenerationRequest(mode=g.RunMode.DeviceLoop, prompt=prompt, gen_len=40))
    assert r3.tokens == want.tokens
    assert r3.counters.kernel_launches == 0 and r3.counters.graph_replays == 2


def _rank(rank, world, q_id, q_out, prompt, steps):
    import torch as t
    t.cuda.set_device(rank)
    t.cuda.init()
    from paper_2604_23467_b200 import graphrt as gg
    uid = gg.tp_unique_id() if rank == 0 else None
    if rank == 0:
        for _ in range(world - 1):
            q_id.put(uid)
    else:
        uid = q_id.get(timeout=300)
    m = gg.Model(gg.ModelConfig(tp_size=world, tp_rank=rank, device=rank, **KW))
    m.attach_nccl(uid)
    s = gg.Session(m, gg.CacheConfig(bucket_size=32, warmup_hi=2, batched_prefill=True))
    r = s.run(gg.GenerationRequest(prompt=prompt, gen_len=steps))
    q_out.put((rank, r.tokens, s.logits()))


def test_multi_gpu_tensor_parallel_nccl_matches_single_gpu():
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (one process per GPU, real NCCL)")
    world = 8 if n >= 8 else (4 if n >= 4 else 2)
    prompt = make_prompt(42, 20, 32000)
    steps = 16
    ref = g.Session(g.ModelConfig(**KW), _cache())
    want = ref.run(g.GenerationRequest(prompt=prompt, gen_len=steps))
    want_logits = ref.logits()
    ref.close()
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q_id, q_out = ctx.Queue(), ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, world, q_id, q_out, prompt, steps)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q_out.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(60)
    for rank, toks, lg in outs:
        assert float(np.abs(lg - want_logits).max()) <= 2e-3, rank
        agree = sum(a == b for a, b in zip(toks, want.tokens))
        assert agree >= steps - 2, (rank, toks, want.tokens)
