"""The reference's latency-sweep harness (bench.hpp / bench.cpp) on real clocks.

Same surface as graphrt::run_bench & co: a BenchConfig
grid of modes x prompt lengths x generation lengths x trials (one warm trial
-1 first, one fresh Session -- i.e. graph cache -- per cell), TrialRow /
CellSummary, the byte-stable CSV with the frozen header (bench.hpp:91-93),
nearest-rank percentile (bench.cpp:41-49), make_prompt (bench.cpp:34-39), the
fixed-width summary tables (bench.cpp:230-292) and the flat `section.key =
value` config format with apply_config (bench.cpp:333-416).

Differences: timings are real (host wall clock for ttft/total, device
%globaltimer gaps for per-token); the reference's virtual-clock `cost.*` keys
are accepted and ignored (real hardware has no cost model), and `model.*` /
`cache.*` gain the B200 extensions (arch, dims, dtype, bucket_size, ...).
"""
from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, TextIO

from . import graphrt as g

CSV_HEADER = ("mode,prompt_len,gen_len,trial,ttft_us,total_us,mean_tok_us,p99_tok_us,"
              "dispatches,replays,captures,cache_hits,cache_misses")

ALL_MODES = [g.RunMode.Eager, g.RunMode.Hybrid, g.RunMode.GraphOnly, g.RunMode.AblateAsync,
             g.RunMode.AblateFused, g.RunMode.AblateBoth]


# ---------------------------------------------------------------------------
# std::mt19937_64 (the standard fixes its output sequence) for make_prompt

class _MT19937_64:
    N, M = 312, 156
    MATRIX_A, UPPER, LOWER = 0xB5026F5AA96619E9, 0xFFFFFFFF80000000, 0x7FFFFFFF
    MASK = (1 << 64) - 1

    def __init__(self, seed: int):
        self.mt = [0] * self.N
        self.mt[0] = seed & self.MASK
        for i in range(1, self.N):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & self.MASK
        self.i = self.N

    def _twist(self):
        mt, N, M = self.mt, self.N, self.M
        for i in range(N):
            x = (mt[i] & self.UPPER) | (mt[(i + 1) % N] & self.LOWER)
            xa = x >> 1
            if x & 1:
                xa ^= self.MATRIX_A
            mt[i] = mt[(i + M) % N] ^ xa
        self.i = 0

    def __call__(self) -> int:
        if self.i >= self.N:
            self._twist()
        x = self.mt[self.i]
        self.i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & self.MASK


def make_prompt(base_seed: int, prompt_len: int, vocab_size: int) -> List[int]:
    """bench.cpp:34-39: mt19937_64(seed * 1000003 + len) % vocab."""
    eng = _MT19937_64((base_seed * 1000003 + prompt_len) & _MT19937_64.MASK)
    return [eng() % vocab_size for _ in range(prompt_len)]


def percentile(samples: List[float], p: float) -> float:
    """Nearest rank: the ceil(p/100 * n)-th smallest (bench.cpp:41-49)."""
    if not samples:
        raise g.Error(g.Errc.EmptySamples, "percentile of empty sample set")
    if not (p > 0.0) or p > 100.0:
        raise g.Error(g.Errc.InvalidConfig, "percentile p outside (0, 100]")
    s = sorted(samples)
    rank = max(1, int(math.ceil(p / 100.0 * len(s))))
    return s[rank - 1]


def _mean(xs: List[float]) -> float:
    if not xs:
        raise g.Error(g.Errc.EmptySamples, "mean of empty sample set")
    return sum(xs) / len(xs)


# ---------------------------------------------------------------------------

@dataclass
class BenchConfig:
    model: g.ModelConfig = field(default_factory=g.ModelConfig)
    cache: g.CacheConfig = field(default_factory=g.CacheConfig)
    modes: List[g.RunMode] = field(default_factory=lambda: list(ALL_MODES))
    prompt_lens: List[int] = field(default_factory=lambda: [10, 50, 100])
    gen_lens: List[int] = field(default_factory=lambda: [10, 50, 100])
    trials: int = 100
    base_seed: int = 42
    strategy: g.SampleStrategy = field(default_factory=g.SampleStrategy.greedy)


@dataclass
class TrialRow:
    mode: g.RunMode = g.RunMode.Eager
    prompt_len: int = 0
    gen_len: int = 0
    trial: int = 0
    ttft_us: float = 0.0
    total_us: float = 0.0
    mean_tok_us: float = 0.0
    p99_tok_us: float = 0.0
    dispatches: int = 0
    replays: int = 0
    captures: int = 0
    cache_hits: int = 0
    cache_misses: int = 0


@dataclass
class CellSummary:
    mode: g.RunMode = g.RunMode.Eager
    prompt_len: int = 0
    gen_len: int = 0
    kept_trials: int = 0
    ttft_mean_us: float = 0.0
    ttft_p99_us: float = 0.0
    tok_mean_us: float = 0.0
    tok_p50_us: float = 0.0
    tok_p99_us: float = 0.0
    total_mean_us: float = 0.0
    replays_mean: float = 0.0
    captures_mean: float = 0.0


@dataclass
class BenchResult:
    rows: List[TrialRow] = field(default_factory=list)
    summaries: List[CellSummary] = field(default_factory=list)
    skipped_cells: List[str] = field(default_factory=list)


def mode_name(m: g.RunMode) -> str:
    return g.mode_name(m)


def run_bench(cfg: BenchConfig, progress: Optional[TextIO] = None, model: Optional[g.Model] = None) -> BenchResult:
    """bench.cpp:51-138.  The weights are built once (or `model` is reused, its
    config must be cfg.model's); every cell gets a fresh Session (its own graph
    cache), as the reference builds a Session per cell."""
    if cfg.trials < 1:
        raise g.Error(g.Errc.InvalidConfig, "bench trials must be >= 1")
    out = BenchResult()
    for mode in cfg.modes:
        for p in cfg.prompt_lens:
            for gl in cfg.gen_lens:
                if p + gl > cfg.model.max_seq_len:
                    out.skipped_cells.append(f"{mode_name(mode)} p={p} g={gl} exceeds max_seq_len")
                    continue
                if model is None:
                    model = g.Model(cfg.model)
                session = g.Session(model, cfg.cache)
                prompt = make_prompt(cfg.base_seed, p, cfg.model.vocab_size)
                pooled, ttfts, totals = [], [], []
                replay_sum = capture_sum = 0.0
                for trial in range(-1, cfg.trials):
                    r = session.run(g.GenerationRequest(mode=mode, prompt=prompt, gen_len=gl,
                                                        strategy=cfg.strategy, sampler_seed=cfg.base_seed))
                    row = TrialRow(mode, p, gl, trial, r.ttft_us, r.total_us, _mean(r.per_token_us),
                                   percentile(r.per_token_us, 99.0), r.counters.dispatches,
                                   r.counters.graph_replays, r.counters.captures, r.cache_delta.hits,
                                   r.cache_delta.misses)
                    out.rows.append(row)
                    if trial >= 0:
                        pooled += r.per_token_us
                        ttfts.append(r.ttft_us)
                        totals.append(r.total_us)
                        replay_sum += r.counters.graph_replays
                        capture_sum += r.counters.captures
                s = CellSummary(mode, p, gl, cfg.trials, _mean(ttfts), percentile(ttfts, 99.0), _mean(pooled),
                                percentile(pooled, 50.0), percentile(pooled, 99.0), _mean(totals),
                                replay_sum / cfg.trials, capture_sum / cfg.trials)
                out.summaries.append(s)
                session.close()
                if progress is not None:
                    progress.write(f"cell {mode_name(mode)} p={p} g={gl}: ttft_mean={fmt(s.ttft_mean_us)}us "
                                   f"tok_p99={fmt(s.tok_p99_us)}us\n")
    return out


# ---------------------------------------------------------------------------
# CSV (bench.cpp:143-225): fixed header, modes by name, shortest round-trip floats

def fmt(v: float) -> str:
    """std::to_chars(double) shortest form: the shorter of the fixed and
    scientific spellings of the shortest round-trip digits (fixed on a tie)."""
    if v == 0.0:
        return "-0" if math.copysign(1.0, v) < 0 else "0"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    if math.isnan(v):
        return "nan"
    r = repr(float(v))
    sign = "-" if r.startswith("-") else ""
    r = r.lstrip("-")
    if "e" in r:
        mant, exp = r.split("e")
        e = int(exp)
    else:
        mant, e = r, 0
    if "." in mant:
        ip, fp = mant.split(".")
    else:
        ip, fp = mant, ""
    digits = (ip + fp).lstrip("0")
    point = len(ip) + e  # decimal point position relative to the digit string of ip+fp
    lead_zeros = len(ip + fp) - len((ip + fp).lstrip("0"))
    point -= lead_zeros
    digits = digits.rstrip("0") or "0"
    # scientific
    sci_exp = point - 1
    sci = digits[0] + ("." + digits[1:] if len(digits) > 1 else "") + "e" + ("-" if sci_exp < 0 else "+") + \
        f"{abs(sci_exp):02d}"
    # fixed
    if point <= 0:
        fixed = "0." + "0" * (-point) + digits
    elif point >= len(digits):
        fixed = digits + "0" * (point - len(digits))
    else:
        fixed = digits[:point] + "." + digits[point:]
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def emit_csv(os: TextIO, rows: List[TrialRow]) -> None:
    os.write(CSV_HEADER + "\n")
    for r in rows:
        os.write(f"{mode_name(r.mode)},{r.prompt_len},{r.gen_len},{r.trial},{fmt(r.ttft_us)},{fmt(r.total_us)},"
                 f"{fmt(r.mean_tok_us)},{fmt(r.p99_tok_us)},{r.dispatches},{r.replays},{r.captures},"
                 f"{r.cache_hits},{r.cache_misses}\n")


def parse_csv(text: str) -> List[TrialRow]:
    lines = text.split("\n")
    if not lines or not lines[0].rstrip("\r"):
        raise g.Error(g.Errc.IoError, "csv: empty input")
    if lines[0].rstrip("\r") != CSV_HEADER:
        raise g.Error(g.Errc.IoError, f"csv: unexpected header '{lines[0]}'")
    rows = []
    for line in lines[1:]:
        line = line.rstrip("\r")
        if not line:
            continue
        f = line.split(",")
        if len(f) != 13:
            raise g.Error(g.Errc.IoError, f"csv: expected 13 fields, got {len(f)}")
        try:
            rows.append(TrialRow(g.mode_from_name(f[0]), int(f[1]), int(f[2]), int(f[3]), float(f[4]), float(f[5]),
                                 float(f[6]), float(f[7]), int(f[8]), int(f[9]), int(f[10]), int(f[11]), int(f[12])))
        except ValueError as e:
            raise g.Error(g.Errc.IoError, f"csv: bad field in '{line}': {e}")
    return rows


def write_csv_file(path: str, rows: List[TrialRow]) -> None:
    try:
        with open(path, "w", newline="") as f:
            emit_csv(f, rows)
    except OSError as e:
        raise g.Error(g.Errc.IoError, f"cannot write '{path}': {e}")


def read_csv_file(path: str) -> List[TrialRow]:
    try:
        with open(path, newline="") as f:
            return parse_csv(f.read())
    except OSError as e:
        raise g.Error(g.Errc.IoError, f"cannot open '{path}': {e}")


# ---------------------------------------------------------------------------
# summary tables (bench.cpp:230-292)

def format_summary(os: TextIO, summaries: List[CellSummary]) -> None:
    if not summaries:
        os.write("no cells ran\n")
        return
    for title, fld in (("ttft mean", "ttft_mean_us"), ("per-token p50", "tok_p50_us"),
                       ("per-token p99", "tok_p99_us"), ("total mean", "total_mean_us")):
        cells, modes = [], []
        for s in summaries:
            if (s.prompt_len, s.gen_len) not in cells:
                cells.append((s.prompt_len, s.gen_len))
            if s.mode not in modes:
                modes.append(s.mode)
        os.write(f"{title} (us)\n")
        os.write("  prompt    gen" + "".join(f" {mode_name(m):>14s}" for m in modes) + "\n")
        for p, gl in cells:
            line = f"  {p:6d} {gl:6d}"
            for m in modes:
                hit = next((s for s in summaries if s.mode == m and s.prompt_len == p and s.gen_len == gl), None)
                line += f" {('%.3f' % getattr(hit, fld)) if hit else '-':>14s}"
            os.write(line + "\n")
        os.write("\n")


# ---------------------------------------------------------------------------
# config files (bench.cpp:333-416)

def parse_config_text(text: str) -> Dict[str, str]:
    kv = {}
    for lineno, line in enumerate(text.split("\n"), 1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise g.Error(g.Errc.InvalidConfig, f"config line {lineno}: expected key = value")
        key, value = (x.strip() for x in line.split("=", 1))
        if not key:
            raise g.Error(g.Errc.InvalidConfig, f"config line {lineno}: empty key")
        kv[key] = value  # last writer wins
    return kv


def parse_config_file(path: str) -> Dict[str, str]:
    try:
        with open(path) as f:
            return parse_config_text(f.read())
    except OSError:
        raise g.Error(g.Errc.IoError, f"cannot open config '{path}'")


def _num(value: str, key: str, typ):
    try:
        v = typ(value)
    except ValueError:
        raise g.Error(g.Errc.InvalidConfig, f"config: bad number for {key}: '{value}'")
    return v


def _bool(value: str, key: str) -> bool:
    if value in ("true", "1"):
        return True
    if value in ("false", "0"):
        return False
    raise g.Error(g.Errc.InvalidConfig, f"config: bad bool for {key}: '{value}'")


def _int_list(value: str, key: str) -> List[int]:
    out = [_num(x.strip(), key, int) for x in value.split(",") if x.strip()]
    if not out:
        raise g.Error(g.Errc.InvalidConfig, f"config: empty list for {key}")
    return out


_MODEL_INT = ("n_layers", "d_model", "n_heads", "vocab_size", "max_seq_len", "seed", "device")
_CACHE_INT = ("capacity", "warmup_lo", "warmup_hi", "bucket_size", "pass_impl")
_COST_KEYS = ("launch_us", "host_us", "alpha", "capture_us", "jitter", "jitter_sigma")


def apply_config(cfg: BenchConfig, kv: Dict[str, str]) -> List[str]:
    """Applies `kv` to cfg; unknown keys raise InvalidConfig.  Returns the
    accepted-but-ignored reference keys (the virtual clock's cost.*)."""
    ignored = []
    for key, value in kv.items():
        sec, _, name = key.partition(".")
        if sec == "model" and name in _MODEL_INT:
            setattr(cfg.model, name, _num(value, key, int))
        elif key == "model.ln_eps":
            cfg.model.ln_eps = _num(value, key, float)
        elif key == "model.d_ff":
            cfg.model.d_ff_ = _num(value, key, int)
        elif key == "model.rope_theta":
            cfg.model.rope_theta = _num(value, key, float)
        elif key == "model.arch":
            if value not in ("ref", "llama"):
                raise g.Error(g.Errc.InvalidConfig, f"config: unknown model.arch '{value}'")
            cfg.model.arch = g.ARCH_REF if value == "ref" else g.ARCH_LLAMA
        elif key in ("model.weight_dtype", "model.kv_dtype"):
            if value not in ("f32", "bf16"):
                raise g.Error(g.Errc.InvalidConfig, f"config: unknown {key} '{value}'")
            setattr(cfg.model, name, g.F32 if value == "f32" else g.BF16)
        elif key == "model.init":
            inits = {"mt19937": g.INIT_MT19937, "philox": g.INIT_PHILOX}
            if value not in inits:
                raise g.Error(g.Errc.InvalidConfig, f"config: unknown model.init '{value}'")
            cfg.model.init = inits[value]
        elif sec == "cache" and name in _CACHE_INT:
            setattr(cfg.cache, name, _num(value, key, int))
        elif key in ("cache.prefill_uses_graphs", "cache.batched_prefill", "cache.prefill_fuse_norm"):
            setattr(cfg.cache, name, _bool(value, key))
        elif key == "cache.policy":
            if value == "least_used":
                cfg.cache.policy = g.EvictionPolicy.LeastUsed
            elif value == "lru":
                cfg.cache.policy = g.EvictionPolicy.LeastRecentlyUsed
            else:
                raise g.Error(g.Errc.InvalidConfig, f"config: unknown cache.policy '{value}'")
        elif sec == "cost" and name in _COST_KEYS:
            ignored.append(key)  # virtual clock parameters: real hardware
        elif key == "bench.modes":
            cfg.modes = [g.mode_from_name(x.strip()) for x in value.split(",") if x.strip()]
            if not cfg.modes:
                raise g.Error(g.Errc.InvalidConfig, "config: empty bench.modes")
        elif key == "bench.prompt_lens":
            cfg.prompt_lens = _int_list(value, key)
        elif key == "bench.gen_lens":
            cfg.gen_lens = _int_list(value, key)
        elif key == "bench.trials":
            cfg.trials = _num(value, key, int)
        elif key == "bench.seed":
            cfg.base_seed = _num(value, key, int)
        elif key == "bench.strategy":
            if value == "greedy":
                cfg.strategy = dataclasses.replace(cfg.strategy, kind=0)
            elif value == "temperature":
                cfg.strategy = dataclasses.replace(cfg.strategy, kind=1)
            else:
                raise g.Error(g.Errc.InvalidConfig, f"config: unknown bench.strategy '{value}'")
        elif key == "bench.temperature":
            cfg.strategy = dataclasses.replace(cfg.strategy, temperature=_num(value, key, float))
        elif key == "bench.trace":
            _bool(value, key)
            ignored.append(key)  # the virtual device timeline; use ncu / profiles/ here
        else:
            raise g.Error(g.Errc.InvalidConfig, f"config: unknown key '{key}'")
    return ignored
