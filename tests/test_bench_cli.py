"""Bench CLI / CSV parity (reference tests/test_bench.py): workload generators against the
reference's own outputs (tests/golden/workloads.json), the CSV schema, and -- on the GPU --
the four sweeps, the CLI and its exit codes."""
import csv
import os

import pytest

from gold import load

from paper_2009_07914_b200.bench import (CSV_FIELDS, REFERENCE_FIELDS, BenchRecord,  # noqa: E402
                                         VerificationError, emit_csv, load_csv, main)
from paper_2009_07914_b200.workloads import WorkloadSpec, gen_multiplicity, gen_unique  # noqa: E402


# ------------------------------------------------------------------ CPU: generators and schema

def test_generators_match_reference_outputs():
    g = load("workloads.json")
    for n, kb, seed in [(1000, 32, 42), (1 << 16, 32, 10_010), (5000, 64, 12)]:
        got = gen_unique(WorkloadSpec(n=n, key_bits=kb, seed=seed))[:64]
        assert [str(int(k)) for k in got] == g[f"unique_{n}_{kb}_{seed}"]
    for n, r, seed in [(1000, 4, 77), (1 << 14, 16, 42), (1000, 1, 4)]:
        got = gen_multiplicity(WorkloadSpec(n=n, r=r, seed=seed))[:64]
        assert [str(int(k)) for k in got] == g[f"mult_{n}_{r}_{seed}"]


def test_gen_unique_properties():                      # test_bench.py:13-31
    keys = gen_unique(WorkloadSpec(n=8, seed=1)).tolist()
    assert len(keys) == len(set(keys)) == 8 and all(k >= 1 for k in keys)
    keys = gen_unique(WorkloadSpec(n=50_000, key_bits=32, seed=2)).tolist()
    top = (1 << 32) - 1
    assert len(set(keys)) == 50_000 and top not in keys and top - 1 not in keys


def test_gen_multiplicity_properties():                # test_bench.py:49-62
    spec = WorkloadSpec(n=100_000, r=16, seed=3)
    keys = gen_multiplicity(spec)
    assert len(keys) == spec.n and int(keys.max()) <= spec.n // spec.r
    assert abs(spec.n / len(set(keys.tolist())) - 16) / 16 < 0.05
    assert sorted(gen_multiplicity(WorkloadSpec(n=1000, r=1, seed=4)).tolist()) == list(range(1, 1001))


def test_invalid_spec():                               # test_bench.py:65-69
    with pytest.raises(ValueError):
        WorkloadSpec(n=10, r=11)
    with pytest.raises(ValueError):
        WorkloadSpec(n=10, target_density=1.5)


def test_emit_csv_round_trip(tmp_path):                # test_bench.py:72-83
    path = str(tmp_path / "bench.csv")
    records = [
        BenchRecord("single_value", "insert", "soa", 32, 1024, 1, 0.8, 0.79, 0.5, 2.048, 33.5),
        BenchRecord("multi_value", "retrieve", "packed", 8, 2048, 16, 0.9, 0.88, 0.25, 8.192, 40.0, shards=4,
                    gbps=123.5, roofline_frac=0.02, gpus=2),
    ]
    emit_csv(records, path)
    assert load_csv(path) == records
    with open(path) as fh:
        assert fh.readline().strip() == ",".join(CSV_FIELDS)
    # the reference's exact header (its load_csv compares it verbatim) and back
    emit_csv(records, path, reference_columns=True)
    with open(path) as fh:
        header = next(csv.reader(fh))
    assert header == REFERENCE_FIELDS == ["structure", "operation", "layout", "group_width", "n", "r",
                                          "target_density", "achieved_density", "seconds", "mops",
                                          "probe_attempts_mean", "shards"]
    back = load_csv(path)
    assert [b.mops for b in back] == [r.mops for r in records] and back[1].gpus == 1


def test_emit_csv_empty(tmp_path):                     # test_bench.py:86-91
    path = str(tmp_path / "empty.csv")
    emit_csv([], path)
    with open(path) as fh:
        assert fh.read().splitlines() == [",".join(CSV_FIELDS)]


def test_cli_invalid_workload_exits_2(tmp_path):
    out = str(tmp_path / "x.csv")
    assert main(["single-sweep", "--n", "0", "--out", out]) == 2
    assert not os.path.exists(out)


def test_verification_error_type():
    with pytest.raises(VerificationError):
        raise VerificationError("boom")


# ------------------------------------------------------------------ GPU: sweeps and CLI

@pytest.mark.gpu
def test_single_sweep_record_shape():                  # test_bench.py:94-103
    from paper_2009_07914_b200.bench import run_single_sweep
    records = run_single_sweep([0.7, 0.5, 0.9], WorkloadSpec(n=2048, seed=5), repeats=2)
    assert len(records) == 6
    densities = [r.target_density for r in records[::2]]
    assert densities == sorted(densities)
    for rec in records:
        assert rec.mops > 0 and rec.gbps > 0 and 0 < rec.roofline_frac < 1
        assert 0 < rec.achieved_density <= rec.target_density
        assert rec.operation in ("insert", "retrieve")


@pytest.mark.gpu
def test_multi_sweep_conserves_totals():               # test_bench.py:106-110
    from paper_2009_07914_b200.bench import run_multi_sweep
    records = run_multi_sweep([1, 16], WorkloadSpec(n=4096, seed=6, target_density=0.8), repeats=1)
    assert len(records) == 4 and {r.r for r in records} == {1, 16}


@pytest.mark.gpu
def test_bucket_sweep_policies():                      # test_bench.py:113-117
    from paper_2009_07914_b200.bench import run_bucket_sweep
    records = run_bucket_sweep(["default", "optimal"], WorkloadSpec(n=2048, r=8, seed=7, target_density=0.8),
                               repeats=1)
    assert len(records) == 4 and any("s0=8" in r.structure for r in records)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["distributed", "independent"])
def test_distributed_sweep_shards_column(mode):        # test_bench.py:120-124
    from paper_2009_07914_b200 import ShardMode
    from paper_2009_07914_b200.bench import run_distributed_sweep
    records = run_distributed_sweep([1, 2], WorkloadSpec(n=2048, r=4, seed=8, target_density=0.8), repeats=1,
                                    mode=ShardMode(mode))
    assert [r.shards for r in records] == [1, 1, 2, 2]


@pytest.mark.gpu
def test_cli_end_to_end(tmp_path):                     # test_bench.py:127-134
    out = str(tmp_path / "cli.csv")
    assert main(["single-sweep", "--n", "1024", "--densities", "0.5,0.8", "--repeats", "1", "--seed", "1",
                 "--out", out]) == 0
    assert len(load_csv(out)) == 4 and os.path.getsize(out) > 0


@pytest.mark.gpu
def test_cli_group_width_and_layout(tmp_path):         # test_bench.py:137-145
    out = str(tmp_path / "cli2.csv")
    assert main(["multi-sweep", "--n", "1024", "--multiplicities", "1,4", "--layout", "packed",
                 "--group-width", "8", "--repeats", "1", "--out", out]) == 0
    assert all(r.layout == "packed" and r.group_width == 8 for r in load_csv(out))


@pytest.mark.gpu
def test_cli_rejects_bad_layout_combination(tmp_path):  # test_bench.py:34-41
    out = str(tmp_path / "x.csv")
    assert main(["single-sweep", "--n", "512", "--densities", "0.5", "--layout", "packed", "--key-bits", "64",
                 "--repeats", "1", "--out", out]) == 2
    assert not os.path.exists(out)


@pytest.mark.gpu
def test_cli_verification_failure_exits_nonzero(tmp_path, monkeypatch):   # test_bench.py:148-166
    from paper_2009_07914_b200 import multi_table

    original = multi_table.MultiValueHashTable.retrieve_device

    def corrupted(self, keys, stream=None):
        offsets, flat = original(self, keys, stream)
        if flat.numel():
            flat[0] ^= 1
        return offsets, flat

    monkeypatch.setattr(multi_table.MultiValueHashTable, "retrieve_device", corrupted)
    out = str(tmp_path / "bad.csv")
    assert main(["multi-sweep", "--n", "512", "--multiplicities", "4", "--repeats", "1", "--out", out]) == 2
    assert not os.path.exists(out)
