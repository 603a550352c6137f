"""Benchmark CLI with built-in verification (mirrors coophash/bench.py).

  python -m paper_2009_07914_b200.bench single-sweep|multi-sweep|bucket-sweep|distributed-sweep \
      [--n 2^20] [--densities ...] [--multiplicities ...] [--policies ...] [--shards ...] --out x.csv

Same subcommands, flags, workloads (gen_unique / gen_multiplicity with the reference's RNG
calls), CSV schema and exit codes as the reference (bench.py:88-132, 156-359, 373-452):
every sweep point builds a fresh table, times the bulk insert and the bulk retrieve, checks
the answers against an in-memory oracle and writes one CSV row per (point, operation); a
wrong answer aborts with exit code 2 and no CSV.

B200 differences, all additive:
  * ``--warmup`` (default 1) untimed repetitions before the timed ones;
  * timing: CUDA events around the device bulk op with the inputs already in HBM (the
    reference times its Python call with the inputs materialised in host memory; the
    host -> device copy happens once, before the clock, like its list construction);
  * three extra CSV columns after the reference's: ``gbps`` (algorithmic bytes per op of
    SURVEY.md §8(d) x ops/s), ``roofline_frac`` (gbps / measured HBM peak) and ``gpus``.
    plots/ reads columns by name and ignores them; ``--reference-columns`` writes exactly
    the reference's header for tools that compare it verbatim (its load_csv does);
  * ``--threads`` is accepted and ignored: a bulk op is one kernel pipeline over all SMs.
"""
from __future__ import annotations

import argparse
import csv
import json
import math
import os
import sys
from dataclasses import dataclass, fields
from typing import Sequence

import numpy as np
import torch

from .bucket_list import BucketListHashTable, GrowthPolicy
from .distributed import DistributedTable, ShardMode
from .layout import LayoutKind, LayoutUnsupported
from .multi_table import MultiValueHashTable
from .single_table import SingleValueHashTable
from .workloads import WorkloadSpec, gen_multiplicity, gen_unique

DEFAULT_N = 1 << 20
DEFAULT_DENSITIES = (0.5, 0.6, 0.7, 0.8, 0.9, 0.95)
DEFAULT_MULTIPLICITIES = (1, 16, 256, 4096)
POOL_HEADROOM = 2.5

# algorithmic bytes per op: one 32 B sector per table touch + the op's I/O
INSERT_BYTES = 73
RETRIEVE_BYTES = 41
BUCKET_INSERT_BYTES = 137


class VerificationError(Exception):
    """A benchmark produced results that disagree with the oracle."""


@dataclass
class BenchRecord:
    structure: str
    operation: str
    layout: str
    group_width: int
    n: int
    r: int
    target_density: float
    achieved_density: float
    seconds: float
    mops: float
    probe_attempts_mean: float
    shards: int = 1
    gbps: float = 0.0
    roofline_frac: float = 0.0
    gpus: int = 1


REFERENCE_FIELDS = [f.name for f in fields(BenchRecord)][:12]   # bench.py:103 CSV_FIELDS
CSV_FIELDS = [f.name for f in fields(BenchRecord)]


def emit_csv(records: Sequence[BenchRecord], path: str, reference_columns: bool = False) -> None:
    names = REFERENCE_FIELDS if reference_columns else CSV_FIELDS
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(names)
        for rec in records:
            w.writerow([getattr(rec, name) for name in names])


def load_csv(path: str) -> list[BenchRecord]:
    """Reads this module's CSV or the reference's (GPU columns then take their defaults)."""
    out = []
    casts = {f.name: f.type for f in fields(BenchRecord)}
    with open(path, newline="") as fh:
        reader = csv.DictReader(fh)
        if reader.fieldnames not in (CSV_FIELDS, REFERENCE_FIELDS):
            raise ValueError(f"unexpected CSV header: {reader.fieldnames}")
        for row in reader:
            kw = {}
            for name, val in row.items():
                typ = casts[name]
                kw[name] = int(val) if typ in ("int", int) else float(val) if typ in ("float", float) else val
            out.append(BenchRecord(**kw))
    return out


# ------------------------------------------------------------------ measurement helpers

def _peak_gbs() -> float:
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0   # B200_PROFILING.md fallback


def _timed(fn):
    """Device time of fn() (CUDA events on the current stream), and its result."""
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    out = fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3, out


def _dev(a: np.ndarray, bits: int, device: int = 0) -> torch.Tensor:
    a = np.ascontiguousarray(a.astype(np.uint32 if bits <= 32 else np.uint64))
    return torch.from_numpy(a.view(np.int32 if bits <= 32 else np.int64)).to(f"cuda:{device}")


def _host_u64(t: torch.Tensor) -> np.ndarray:
    a = t.cpu().numpy()
    return (a.view(np.uint32) if a.dtype == np.int32 else a.view(np.uint64)).astype(np.uint64)


def _mean_attempts(table, c0) -> float:
    c = table.probe_counters()
    ops = c.ops - c0.ops
    return (c.attempts - c0.attempts) / ops if ops else 0.0


def _check_inserted(st: torch.Tensor, context: str) -> None:
    bad = int((st != 0).sum().item())
    if bad:
        raise VerificationError(f"{context}: {bad} of {st.numel()} inserts failed")


def _record(structure, op, layout, g, n, r, rho, achieved, secs, attempts, shards=1, bytes_total=0.0,
            gpus=1) -> BenchRecord:
    gbps = bytes_total / secs / 1e9 if secs > 0 else 0.0
    return BenchRecord(structure=structure, operation=op, layout=layout, group_width=g, n=n, r=r,
                       target_density=rho, achieved_density=achieved, seconds=secs, mops=n / secs / 1e6,
                       probe_attempts_mean=attempts, shards=shards, gbps=gbps,
                       roofline_frac=gbps / _peak_gbs(), gpus=gpus)


def _multi_reference(keys: np.ndarray, vals: np.ndarray):
    """Sorted (key, value) pairs: the per-key sorted multisets of bench.py:190-198."""
    order = np.lexsort((vals, keys))
    return keys[order], vals[order]


def _verify_multi(queries: np.ndarray, offsets: np.ndarray, flat: np.ndarray, ref, context: str) -> None:
    """Per-query sorted segments equal the reference multisets (bench.py:201-220)."""
    rk, rv = ref
    if offsets[-1] != len(rk):
        raise VerificationError(f"{context}: retrieved {offsets[-1]} values, expected {len(rk)}")
    counts = np.diff(offsets)
    qk = np.repeat(queries, counts)
    order = np.lexsort((flat, qk))
    if not (np.array_equal(qk[order], rk) and np.array_equal(flat[order], rv)):
        bad = np.nonzero((qk[order] != rk) | (flat[order] != rv))[0]
        raise VerificationError(f"{context}: value mismatch for key {int(rk[bad[0]]) if len(bad) else '?'}")


def _multi_retrieve_bytes(counts: np.ndarray) -> float:
    """sum over queries of 8 + 2*32*max(1, ceil(m/4)) + 24 + 4 m."""
    m = counts.astype(np.float64)
    return float(np.sum(8 + 64 * np.maximum(1, np.ceil(m / 4)) + 24 + 4 * m))


def _bucket_retrieve_bytes(counts: np.ndarray) -> float:
    """SURVEY.md §8(d), buckets approximated by whole 32 B sectors of the values."""
    m = counts.astype(np.float64)
    return float(np.sum(8 + 128 + 24 + 32 * np.ceil(4 * (m + 1) / 32) + 4 * m))


# ------------------------------------------------------------------ sweeps

def run_single_sweep(densities: Sequence[float], spec: WorkloadSpec, *, layout: str = "soa",
                     group_width: int = 32, threads: int = 1, repeats: int = 10,
                     warmup: int = 1) -> list[BenchRecord]:
    keys = gen_unique(spec)
    values = np.arange(1, spec.n + 1, dtype=np.uint64)
    vbits = 32 if layout == "packed" else 64
    dk, dv = _dev(keys, spec.key_bits), _dev(values, vbits)
    records: list[BenchRecord] = []
    for rho in sorted(densities):
        ins_secs = ret_secs = ins_att = ret_att = 0.0
        achieved = 0.0
        for rep in range(repeats + warmup):
            table = SingleValueHashTable(int(np.ceil(spec.n / rho)), layout=layout, key_bits=spec.key_bits,
                                         value_bits=vbits, group_width=group_width, workers=threads)
            c0 = table.probe_counters()
            secs, st = _timed(lambda: table.insert_device(dk, dv))
            _check_inserted(st, f"single-sweep rho={rho}")
            ins_secs += secs if rep >= warmup else 0.0
            ins_att += _mean_attempts(table, c0) if rep >= warmup else 0.0
            achieved = table.load_factor()
            c0 = table.probe_counters()
            secs, (got, found) = _timed(lambda: table.retrieve_device(dk))
            if not (bool(found.bool().all()) and np.array_equal(_host_u64(got), values)):
                raise VerificationError(f"single-sweep rho={rho}: retrieval mismatch")
            ret_secs += secs if rep >= warmup else 0.0
            ret_att += _mean_attempts(table, c0) if rep >= warmup else 0.0
            del table
        for op, secs, att, b in (("insert", ins_secs, ins_att, INSERT_BYTES), ("retrieve", ret_secs, ret_att,
                                                                              RETRIEVE_BYTES)):
            mean = secs / repeats
            records.append(_record("single_value", op, layout, group_width, spec.n, 1, rho, achieved, mean,
                                   att / repeats, bytes_total=b * spec.n))
    return records


def run_multi_sweep(multiplicities: Sequence[int], spec: WorkloadSpec, *, layout: str = "soa",
                    group_width: int = 32, threads: int = 1, repeats: int = 10,
                     warmup: int = 1) -> list[BenchRecord]:
    records: list[BenchRecord] = []
    vbits = 32 if layout == "packed" else 64
    for r in multiplicities:
        wspec = WorkloadSpec(n=spec.n, r=r, key_bits=spec.key_bits, seed=spec.seed,
                             target_density=spec.target_density)
        keys = gen_multiplicity(wspec)
        vals = np.arange(1, wspec.n + 1, dtype=np.uint64)
        queries = np.arange(1, wspec.n + 1, dtype=np.uint64)
        ref = _multi_reference(keys, vals)
        dk, dv, dq = _dev(keys, spec.key_bits), _dev(vals, vbits), _dev(queries, spec.key_bits)
        rho = spec.target_density
        ins_secs = ret_secs = ins_att = ret_att = 0.0
        achieved = 0.0
        rbytes = 0.0
        for rep in range(repeats + warmup):
            table = MultiValueHashTable(int(np.ceil(wspec.n / rho)), layout=layout, key_bits=spec.key_bits,
                                        value_bits=vbits, group_width=group_width, workers=threads)
            c0 = table.probe_counters()
            secs, st = _timed(lambda: table.insert_device(dk, dv))
            _check_inserted(st, f"multi-sweep r={r}")
            ins_secs += secs if rep >= warmup else 0.0
            ins_att += _mean_attempts(table, c0) if rep >= warmup else 0.0
            achieved = table.load_factor()
            c0 = table.probe_counters()
            secs, (off, flat) = _timed(lambda: table.retrieve_device(dq))
            offsets = off.cpu().numpy()
            _verify_multi(queries, offsets, _host_u64(flat), ref, f"multi-sweep r={r}")
            rbytes = _multi_retrieve_bytes(np.diff(offsets))
            del off, flat  # the next repetition's outputs reuse the cached blocks
            ret_secs += secs if rep >= warmup else 0.0
            ret_att += _mean_attempts(table, c0) if rep >= warmup else 0.0
            del table
        for op, secs, att, b in (("insert", ins_secs, ins_att, INSERT_BYTES * wspec.n),
                                 ("retrieve", ret_secs, ret_att, rbytes)):
            mean = secs / repeats
            records.append(_record("multi_value", op, layout, group_width, wspec.n, r, rho, achieved, mean,
                                   att / repeats, bytes_total=b))
    return records


def _parse_policy(name: str, r: int) -> tuple[str, GrowthPolicy]:
    """bench.py:270-277."""
    if name == "default":
        return "bucket_list[s0=1,growth=1.1]", GrowthPolicy(1, "1.1")
    if name == "optimal":
        return f"bucket_list[s0={r},growth=1.0]", GrowthPolicy(max(1, r), "1.0")
    s0, _, lam = name.partition(":")
    return f"bucket_list[s0={s0},growth={lam}]", GrowthPolicy(int(s0), lam)


def run_bucket_sweep(policies: Sequence[str], spec: WorkloadSpec, *, group_width: int = 32,
                     threads: int = 1, repeats: int = 10, warmup: int = 1) -> list[BenchRecord]:
    keys = gen_multiplicity(spec)
    vals = np.arange(1, spec.n + 1, dtype=np.uint64)
    queries = np.arange(1, spec.n + 1, dtype=np.uint64)
    ref = _multi_reference(keys, vals)
    distinct = len(np.unique(keys))
    rho = spec.target_density
    pool_slots = int(spec.n * POOL_HEADROOM) + 64
    dk, dv, dq = _dev(keys, spec.key_bits), _dev(vals, 64), _dev(queries, spec.key_bits)
    records: list[BenchRecord] = []
    for name in policies:
        label, policy = _parse_policy(name, spec.r)
        ins_secs = ret_secs = 0.0
        achieved = 0.0
        rbytes = 0.0
        for rep in range(repeats + warmup):
            table = BucketListHashTable(int(np.ceil(distinct / rho)), pool_slots,
                                        growth=GrowthPolicy(policy.initial_size, policy.factor),
                                        key_bits=spec.key_bits, group_width=group_width, workers=threads)
            secs, st = _timed(lambda: table.insert_device(dk, dv))
            _check_inserted(st, f"bucket-sweep {name}")
            ins_secs += secs if rep >= warmup else 0.0
            achieved = table.key_load_factor()
            secs, (off, flat) = _timed(lambda: table.retrieve_device(dq))
            offsets = off.cpu().numpy()
            _verify_multi(queries, offsets, _host_u64(flat), ref, f"bucket-sweep {name}")
            rbytes = _bucket_retrieve_bytes(np.diff(offsets))
            del off, flat
            ret_secs += secs if rep >= warmup else 0.0
            del table
        for op, secs, b in (("insert", ins_secs, BUCKET_INSERT_BYTES * spec.n), ("retrieve", ret_secs, rbytes)):
            mean = secs / repeats
            records.append(_record(label, op, "soa", group_width, spec.n, spec.r, rho, achieved, mean, 0.0,
                                   bytes_total=b))
    return records


def run_distributed_sweep(shard_counts: Sequence[int], spec: WorkloadSpec, *, layout: str = "soa",
                          group_width: int = 32, threads: int = 1, repeats: int = 10,
                          mode: ShardMode = ShardMode.DISTRIBUTED, warmup: int = 1) -> list[BenchRecord]:
    """Multi-value shards (bench.py:305-359); shard s lives on GPU s mod (visible GPUs)."""
    keys = gen_multiplicity(spec)
    vals = np.arange(1, spec.n + 1, dtype=np.uint64)
    queries = np.arange(1, spec.n + 1, dtype=np.uint64)
    ref = _multi_reference(keys, vals)
    rho = spec.target_density
    vbits = 32 if layout == "packed" else 64
    dk, dv, dq = _dev(keys, spec.key_bits), _dev(vals, vbits), _dev(queries, spec.key_bits)
    ngpu = max(1, torch.cuda.device_count())
    records: list[BenchRecord] = []
    for shards in shard_counts:
        per_shard = int(np.ceil(spec.n / shards / rho))
        ins_secs = ret_secs = 0.0
        achieved = 0.0
        rbytes = 0.0
        for rep in range(repeats + warmup):
            with DistributedTable(shards, lambda s: MultiValueHashTable(
                    per_shard, layout=layout, key_bits=spec.key_bits, value_bits=vbits,
                    group_width=group_width, device=s % ngpu), mode=mode) as table:
                secs, st = _timed(lambda: table.insert_device(dk, dv))
                _check_inserted(st, f"distributed-sweep shards={shards}")
                ins_secs += secs if rep >= warmup else 0.0
                achieved = sum(t.occupied for t in table.shards) / sum(t.capacity for t in table.shards)
                secs, (off, flat) = _timed(lambda: table.retrieve_device(dq))
                offsets = off.cpu().numpy()
                _verify_multi(queries, offsets, _host_u64(flat), ref, f"distributed-sweep shards={shards}")
                rbytes = _multi_retrieve_bytes(np.diff(offsets))
                del off, flat
                ret_secs += secs if rep >= warmup else 0.0
        for op, secs, b in (("insert", ins_secs, INSERT_BYTES * spec.n), ("retrieve", ret_secs, rbytes)):
            mean = secs / repeats
            records.append(_record("distributed_multi", op, layout, group_width, spec.n, spec.r, rho, achieved,
                                   mean, 0.0, shards=shards, bytes_total=b, gpus=min(shards, ngpu)))
    return records


# ------------------------------------------------------------------ CLI (bench.py:363-452)

def _int_list(text: str) -> list[int]:
    return [int(tok) for tok in text.split(",") if tok]


def _float_list(text: str) -> list[float]:
    return [float(tok) for tok in text.split(",") if tok]


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="bench", description="B200 hash table sweep benchmarks with "
                                                               "built-in verification")
    common = argparse.ArgumentParser(add_help=False)
    common.add_argument("--n", type=int, default=DEFAULT_N, help="elements per sweep point (default 2^20)")
    common.add_argument("--r", type=int, default=16, help="mean key multiplicity for multi-value workloads")
    common.add_argument("--density", type=float, default=0.8, help="target storage density for fixed-density sweeps")
    common.add_argument("--densities", type=_float_list, default=list(DEFAULT_DENSITIES),
                        help="comma list of target densities (single-sweep)")
    common.add_argument("--multiplicities", type=_int_list, default=list(DEFAULT_MULTIPLICITIES),
                        help="comma list of r values (multi-sweep)")
    common.add_argument("--group-width", type=int, default=32, choices=(1, 2, 4, 8, 16, 32))
    common.add_argument("--layout", default="soa", choices=[k.value for k in LayoutKind])
    common.add_argument("--threads", type=int, default=1, help="accepted for compatibility; ignored on the GPU")
    common.add_argument("--shards", type=_int_list, default=[1, 2, 4],
                        help="comma list of shard counts (distributed-sweep)")
    common.add_argument("--key-bits", type=int, default=32, choices=(32, 64))
    common.add_argument("--seed", type=int, default=42)
    common.add_argument("--repeats", type=int, default=10, help="timed repetitions averaged per sweep point")
    common.add_argument("--warmup", type=int, default=1,
                        help="untimed repetitions first (allocator pools, module loading)")
    common.add_argument("--policies", default="default,optimal", help="comma list: default, optimal, or s0:growth")
    common.add_argument("--reference-columns", action="store_true",
                        help="write exactly the reference's CSV header (no GPU columns)")
    common.add_argument("--out", required=True, help="output CSV path")
    sub = parser.add_subparsers(dest="command", required=True)
    for name in ("single-sweep", "multi-sweep", "bucket-sweep", "distributed-sweep"):
        sub.add_parser(name, parents=[common])
    return parser


def main(argv: Sequence[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        spec = WorkloadSpec(n=args.n, r=args.r, key_bits=args.key_bits, seed=args.seed,
                            target_density=args.density)
    except ValueError as err:
        print(f"invalid workload: {err}", file=sys.stderr)
        return 2
    try:
        if args.command == "single-sweep":
            records = run_single_sweep(args.densities, spec, layout=args.layout, group_width=args.group_width,
                                       threads=args.threads, repeats=args.repeats, warmup=args.warmup)
        elif args.command == "multi-sweep":
            records = run_multi_sweep(args.multiplicities, spec, layout=args.layout, group_width=args.group_width,
                                      threads=args.threads, repeats=args.repeats, warmup=args.warmup)
        elif args.command == "bucket-sweep":
            records = run_bucket_sweep([p for p in args.policies.split(",") if p], spec,
                                       group_width=args.group_width, threads=args.threads, repeats=args.repeats, warmup=args.warmup)
        else:
            records = run_distributed_sweep(args.shards, spec, layout=args.layout, group_width=args.group_width,
                                            threads=args.threads, repeats=args.repeats, warmup=args.warmup)
    except VerificationError as err:
        print(f"verification failed: {err}", file=sys.stderr)
        return 2
    except (ValueError, LayoutUnsupported) as err:
        print(f"invalid configuration: {err}", file=sys.stderr)
        return 2
    emit_csv(records, args.out, reference_columns=args.reference_columns)
    for rec in records:
        print(f"{rec.structure:>28} {rec.operation:>8} rho={rec.target_density:.2f} r={rec.r} "
              f"shards={rec.shards} {rec.mops:10.1f} Mops {rec.gbps:8.1f} GB/s")
    return 0


if __name__ == "__main__":
    sys.exit(main())
