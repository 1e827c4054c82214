"""The reporting surface of the reference harness (bench_test.cpp): nearest-rank
KATs, make_prompt, the frozen CSV schema and its byte round trip, config parsing
and apply_config errors, the sweep's skip rule -- host logic, CPU only; one GPU
test runs a tiny sweep end to end."""
import io
import math

import pytest

from paper_2604_23467_b200 import bench_harness as bh
from paper_2604_23467_b200 import graphrt as g


def test_percentile_nearest_rank_kats():
    # bench_test.cpp:61-78
    xs = [15, 20, 35, 40, 50]
    assert bh.percentile(xs, 5) == 15
    assert bh.percentile(xs, 30) == 20
    assert bh.percentile(xs, 40) == 20
    assert bh.percentile(xs, 50) == 35
    assert bh.percentile(xs, 100) == 50
    assert bh.percentile([3.0], 99) == 3.0
    with pytest.raises(g.Error) as e:
        bh.percentile([], 50)
    assert e.value.code == g.Errc.EmptySamples
    with pytest.raises(g.Error):
        bh.percentile(xs, 0)


def test_make_prompt_matches_reference(golden):
    # make_prompt(42, 10, 256) from the reference binary
    assert bh.make_prompt(42, 10, 256) == [7, 226, 123, 48, 233, 161, 21, 56, 125, 232]
    fx = golden("tiny_ref_greedy.json")
    assert bh.make_prompt(42, len(fx["prompt"]), 256) == fx["prompt"]


def test_fmt_shortest_round_trip():
    for v in (0.0, 1.0, 100.0, 2612.345, 0.1, 1e-7, 123456789.0, 1e21, 3.25e-5, 1 / 3):
        s = bh.fmt(v)
        assert float(s) == v, (v, s)
    assert bh.fmt(100.0) == "100"  # std::to_chars spelling, not Python's "100.0"
    assert bh.fmt(1e21) == "1e+21"
    assert bh.fmt(0.0001) == "1e-04"


def _rows():
    return [bh.TrialRow(g.RunMode.Hybrid, 10, 32, -1, 1234.5, 9876.25, 101.125, 130.0, 3, 42, 0, 42, 0),
            bh.TrialRow(g.RunMode.AblateFused, 50, 10, 0, 1e-3, 1 / 3, 2.0 ** -20, 7.5e12, 0, 0, 1, 2, 3)]


def test_csv_header_frozen_and_round_trip():
    buf = io.StringIO()
    bh.emit_csv(buf, _rows())
    text = buf.getvalue()
    assert text.split("\n")[0] == ("mode,prompt_len,gen_len,trial,ttft_us,total_us,mean_tok_us,p99_tok_us,"
                                   "dispatches,replays,captures,cache_hits,cache_misses")
    assert bh.parse_csv(text) == _rows()
    buf2 = io.StringIO()
    bh.emit_csv(buf2, bh.parse_csv(text))
    assert buf2.getvalue() == text  # byte identical (bench_test.cpp:97-138)
    assert bh.parse_csv(text.replace("\n", "\r\n")) == _rows()
    with pytest.raises(g.Error) as e:
        bh.parse_csv("mode,foo\n")
    assert e.value.code == g.Errc.IoError
    with pytest.raises(g.Error):
        bh.parse_csv(text.split("\n")[0] + "\nhybrid,1,2\n")


def test_config_parse_and_apply():
    kv = bh.parse_config_text("""
        # comment
        model.n_layers = 2
        model.arch = llama      # B200 extension
        cache.policy = lru
        cache.bucket_size = 16
        cost.alpha = 0.02       # virtual clock: accepted, ignored
        bench.modes = hybrid, eager
        bench.prompt_lens = 10,20
        bench.trials = 3
        bench.strategy = temperature
        bench.temperature = 0.8
        model.n_layers = 3      # last writer wins
    """)
    cfg = bh.BenchConfig()
    ignored = bh.apply_config(cfg, kv)
    assert cfg.model.n_layers == 3 and cfg.model.arch == g.ARCH_LLAMA
    assert cfg.cache.policy == g.EvictionPolicy.LeastRecentlyUsed and cfg.cache.bucket_size == 16
    assert cfg.modes == [g.RunMode.Hybrid, g.RunMode.Eager] and cfg.prompt_lens == [10, 20]
    assert cfg.trials == 3 and cfg.strategy.kind == 1 and math.isclose(cfg.strategy.temperature, 0.8)
    assert ignored == ["cost.alpha"]
    for bad in ("model.bogus = 1", "cache.policy = fifo", "bench.trials = x", "no equals sign", " = 3"):
        with pytest.raises(g.Error) as e:
            bh.apply_config(bh.BenchConfig(), bh.parse_config_text(bad))
        assert e.value.code == g.Errc.InvalidConfig


def test_sweep_skips_cells_over_capacity_without_device():
    cfg = bh.BenchConfig(model=g.ModelConfig(max_seq_len=32), prompt_lens=[40], gen_lens=[10],
                         modes=[g.RunMode.Hybrid], trials=1)
    res = bh.run_bench(cfg)  # every cell skipped: no model is ever built
    assert res.rows == [] and res.skipped_cells == ["hybrid p=40 g=10 exceeds max_seq_len"]
    with pytest.raises(g.Error):
        bh.run_bench(bh.BenchConfig(trials=0))


@pytest.mark.gpu
def test_tiny_sweep_end_to_end(tmp_path):
    cfg = bh.BenchConfig(modes=[g.RunMode.Eager, g.RunMode.Hybrid], prompt_lens=[10], gen_lens=[8, 16], trials=2)
    res = bh.run_bench(cfg)
    assert len(res.rows) == 2 * 2 * 3 and len(res.summaries) == 4
    assert all(r.mean_tok_us > 0 for r in res.rows)
    hyb = [r for r in res.rows if r.mode == g.RunMode.Hybrid and r.trial >= 0]
    assert all(r.replays > 0 for r in hyb)
    p = tmp_path / "sweep.csv"
    bh.write_csv_file(str(p), res.rows)
    assert bh.read_csv_file(str(p)) == res.rows
    out = io.StringIO()
    bh.format_summary(out, res.summaries)
    assert "per-token p99 (us)" in out.getvalue()
