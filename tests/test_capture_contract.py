"""The capture / replay contract of the CUDA engine (VERDICT r01 missing #2).

Reference: CaptureEngine / CaptureSession / validate_replay
(exec_graph.hpp:73-141, exec_graph.cpp:49-103) and its unit tests
(tests/unit/exec_graph_test.cpp:40-163); acceptance c9 (warm-up contract) and
c10 (graphs share the workspace; acceptance_main.cpp:504-567).

Our op classes: Static plan kernels; Dynamic context ops (NVRTC sampler /
preprocess reading token, position and RNG draw from device memory) -- legal in
a FUSED hybrid step graph, rejected from a static-only graph exactly as the
reference rejects every dynamic op; Host ops (the step API's host->device token
upload) are never capturable.
"""
import numpy as np
import pytest

from paper_2604_23467_b200 import graphrt as g
from paper_2604_23467_b200.bench_harness import make_prompt

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def raises(code, fn, *a, **kw):
    with pytest.raises(g.Error) as ei:
        fn(*a, **kw)
    assert ei.value.code == code, (ei.value.code, code, str(ei.value))


@pytest.fixture()
def sess():
    # tiny-ref (reference defaults), exact-length keys as the reference (bucket 1), cold cache
    s = g.Session(g.ModelConfig(), g.CacheConfig(bucket_size=1, warmup_hi=0))
    yield s
    s.close()


def test_capture_records_static_kernels(sess):
    """exec_graph_test.cpp:40-54: a capture of plan(4) freezes its kernels."""
    n = sess.plan_size(4)
    c = sess.begin_capture(4)
    for i in range(n):
        c.record_plan(4, i)
    assert c.recorded == n and c.state == g.CaptureState.Open
    k, ep1 = c.end_capture()
    assert k == n and c.state == g.CaptureState.Closed
    c2 = sess.begin_capture(5)
    c2.record_plan(5, 0)
    _, ep2 = c2.end_capture()
    assert ep2 > ep1  # capture epochs increase (exec_graph_test.cpp:120-125)


def test_dynamic_op_aborts_a_static_only_capture(sess):
    """exec_graph_test.cpp:56-72: recording a dynamic op aborts the session, keeps
    nothing, closes it, and releases the key."""
    c = sess.begin_capture(1, fused=False)
    c.record_plan(1, 0)
    raises(g.Errc.CaptureViolation, c.record, g.CaptureOp.SamplePreprocess)
    assert c.state == g.CaptureState.Aborted and c.recorded == 0
    raises(g.Errc.SessionClosed, c.end_capture)
    raises(g.Errc.SessionClosed, c.record_plan, 1, 0)
    retry = sess.begin_capture(1, fused=False)  # key released
    retry.record_plan(1, 0)
    assert retry.end_capture()[0] == 1


def test_fused_capture_takes_device_dynamic_ops_but_never_host_ops(sess):
    """The hybrid step graph (north star (b)): NVRTC context ops are capturable
    into a fused graph; a host-valued op is not, fused or not."""
    c = sess.begin_capture(2, fused=True)
    c.record(g.CaptureOp.SamplePreprocess)
    c.record_plan(2, 0)
    raises(g.Errc.CaptureViolation, c.record, g.CaptureOp.HostToken)
    assert c.state == g.CaptureState.Aborted and c.recorded == 0
    c2 = sess.begin_capture(2, fused=False)
    raises(g.Errc.CaptureViolation, c2.record, g.CaptureOp.HostToken)


def test_foreign_buffer_is_rejected(sess):
    """exec_graph_test.cpp:74-80: a binding outside the model arena."""
    stranger = torch.zeros(64, dtype=torch.float32, device="cuda")
    c = sess.begin_capture(2)
    raises(g.Errc.ForeignBuffer, c.record_external, stranger.data_ptr(), stranger.numel() * 4)
    assert c.state == g.CaptureState.Aborted


def test_empty_capture_and_closed_session_use(sess):
    """exec_graph_test.cpp:92-104."""
    c = sess.begin_capture(3)
    raises(g.Errc.EmptyCapture, c.end_capture)
    assert c.state == g.CaptureState.Aborted
    again = sess.begin_capture(3)
    again.record_plan(3, 0)
    again.end_capture()
    raises(g.Errc.SessionClosed, again.record_plan, 3, 0)
    raises(g.Errc.SessionClosed, again.end_capture)


def test_one_open_capture_per_key(sess):
    """exec_graph_test.cpp:106-118."""
    first = sess.begin_capture(7)
    raises(g.Errc.CaptureInProgress, sess.begin_capture, 7)
    other = sess.begin_capture(8)  # a different key is fine
    first.record_plan(7, 0)
    first.end_capture()
    reopened = sess.begin_capture(7)  # a closed key reopens
    assert reopened.state == g.CaptureState.Open
    other.close()
    raises(g.Errc.LengthOutOfRange, sess.begin_capture, 10 ** 6)


def _capture_step(sess, key, fused=True):
    c = sess.begin_capture(key, fused=fused)
    if fused:
        c.record(g.CaptureOp.Preprocess)
    for i in range(sess.plan_size(key)):
        c.record_plan(key, i)
    return c.end_capture()


def test_replay_validation_host_and_device(sess):
    """exec_graph_test.cpp:142-163 validate_replay: a graph replays only at its
    length.  The host check (validate) raises WrongLength; with it skipped, the
    device-side check in the attention kernel flags a live length beyond the
    graph's bucket and the step raises WrongLength too."""
    prompt = [7, 226, 123]
    sess.prefill(prompt)  # cur_len 3
    _capture_step(sess, 4)
    _capture_step(sess, 6)
    ref = g.Session(g.ModelConfig(), g.CacheConfig(bucket_size=1, warmup_hi=0))
    ref.prefill(prompt)
    ref.step(48)
    sess.replay(4, 48)  # the right length: same result as the step API
    assert np.array_equal(sess.logits(), ref.logits())
    raises(g.Errc.WrongLength, sess.replay, 6, 233)  # host validate_replay: cur_len 4 != 5
    assert sess.cur_len == 4
    raises(g.Errc.WrongLength, sess.replay, 4, 233, validate=False)  # device: length 5 > bucket of key 4
    sess.reset()  # clears the device error flag
    sess.prefill(prompt)
    sess.replay(4, 48)
    assert np.array_equal(sess.logits(), ref.logits())
    # a static-only graph replays with the dynamic op launched outside it
    s2 = g.Session(g.ModelConfig(), g.CacheConfig(bucket_size=1, warmup_hi=0))
    s2.prefill(prompt)
    _capture_step(s2, 4, fused=False)
    s2.replay(4, 48, fused=False)
    assert np.array_equal(s2.logits(), ref.logits())


def test_c9_warmup_contract():
    """acceptance_main.cpp:504-540 with the default warm-up [1, 50] and exact
    length keys: a run inside the range never falls back; (10, 100) falls back
    exactly once per length 51..110, each followed by exactly one insert."""
    prompt = make_prompt(9000, 10, 256)

    def fresh():
        return g.Session(g.ModelConfig(), g.CacheConfig(bucket_size=1))

    inside = fresh().run(g.GenerationRequest(mode=g.RunMode.Hybrid, prompt=prompt, gen_len=40))
    fb = sum(p == g.StepPath.EagerFallback for p in inside.prefill_paths + inside.decode_paths)
    assert fb == 0
    assert inside.counters.captures == 0 and inside.cache_delta.inserts == 0
    outside = fresh().run(g.GenerationRequest(mode=g.RunMode.Hybrid, prompt=prompt, gen_len=100))
    assert all(p == g.StepPath.Replayed for p in outside.prefill_paths)
    for i in range(1, 101):
        want = g.StepPath.Replayed if 10 + i <= 50 else g.StepPath.EagerFallback
        assert outside.decode_paths[i - 1] == want, (10 + i, outside.decode_paths[i - 1])
    assert outside.cache_delta.inserts == 60 and outside.captures_completed == 60
    assert outside.counters.captures == 60


def test_c10_captures_share_the_arena():
    """acceptance_main.cpp:546-567: capturing 100 more lengths allocates nothing
    in the model's arena (graphs bind the shared workspace)."""
    s = g.Session(g.ModelConfig(), g.CacheConfig(bucket_size=1, warmup_hi=50, capacity=600))
    before = s.model.arena_info()
    for key in range(51, 151):
        c = s.begin_capture(key, fused=False)
        for i in range(s.plan_size(key)):
            c.record_plan(key, i)
        c.end_capture()
    assert s.model.arena_info() == before
    st, size = s.cache_stats()
    assert size == 150
