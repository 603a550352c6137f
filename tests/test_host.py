"""CPU-only checks: host utilities vs the reference goldens, the C ABI surface,
and the multi-process exchange plumbing (gloo, world_size 2).  No GPU needed."""
import os
import re
import socket

import numpy as np
import pytest
import torch

from gold import ints, load

from paper_2009_07914_b200 import (CapacityPlan, GrowthPolicy, ProbingConfig, ProbingScheme,  # noqa: E402
                                   choose_capacity, cops_positions, dh_step, exchange, is_prime,
                                   mix64, next_bucket_size, pack_handle, pack_pair, probing,
                                   unpack_handle, unpack_pair, window_starts)
from paper_2009_07914_b200 import _lib  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "coophash_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|uint64_t|const char\*)\s+(ch_\w+)\s*\(", header, re.M))
    assert declared, "no declarations parsed"
    lib = _lib.lib()  # loads without a GPU
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.exported_symbols())
    assert lib.ch_version() == 1


def test_dist_abi_validates_arguments_without_a_gpu():
    import ctypes as C
    lib = _lib.lib()
    h = C.c_void_p()
    assert lib.ch_dist_create(C.byref(h), None, 2, 0) == _lib.CH_EINVAL
    arr = (C.c_void_p * 1)(None)
    assert lib.ch_dist_create(C.byref(h), arr, 0, 0) == _lib.CH_EINVAL      # no shards
    assert lib.ch_dist_create(C.byref(h), arr, 1, 7) == _lib.CH_EINVAL      # bad transport
    assert lib.ch_dist_create(C.byref(h), arr, 1, 0) == _lib.CH_EINVAL      # null shard table
    assert "shard" in _lib.last_error()
    assert lib.ch_dist_insert(None, None, None, None, None, None) == _lib.CH_EINVAL
    assert lib.ch_dist_destroy(None) == 0


def test_probing_matches_golden():
    g = load("probing.json")
    keys = ints(g["keys"])
    assert [mix64(k) for k in keys] == ints(g["mix64"])
    assert probing.mix64_array(keys[:64]).tolist() == ints(g["mix64_array_first"])
    for m, (p, c) in g["plans"].items():
        plan = choose_capacity(int(m))
        assert (plan.p, plan.c) == (p, c)
    for p, steps in g["steps"].items():
        plan = CapacityPlan(p=int(p), c=32 * int(p))
        assert [dh_step(k, plan) for k in keys[:100]] == steps
    assert [is_prime(int(n)) for n in g["primes"]] == g["prime_flags"]
    plan = choose_capacity(1000)
    for scheme in ProbingScheme:
        cfg = ProbingConfig(plan=plan, scheme=scheme)
        for k, starts in g["window_starts"][scheme.value].items():
            assert list(window_starts(int(k), cfg)) == starts
    cfg4 = ProbingConfig(plan=plan, group_width=4, max_outer_attempts=3)
    for k, pos in g["cops_g4"].items():
        assert [cops_positions(int(k), cfg4, i) for i in range(0, 96, 4)] == pos
    for k, order in g["probe_order"].items():
        assert probing.probe_order(int(k), ProbingConfig(plan=plan), limit=100) == order


def test_config_validation():
    plan = choose_capacity(1000)
    with pytest.raises(ValueError):
        ProbingConfig(plan=plan, group_width=3)
    with pytest.raises(ValueError):
        ProbingConfig(plan=plan, max_outer_attempts=plan.p + 1)
    with pytest.raises(ValueError):
        CapacityPlan(p=9, c=288)
    with pytest.raises(ValueError):
        choose_capacity(31)


def test_codecs_and_growth():
    assert unpack_pair(pack_pair(7, 9)) == (7, 9)
    with pytest.raises(ValueError):
        pack_pair(1 << 32, 0)
    g = load("bucket.json")
    for s, c, t, word in g["handles"]:
        assert pack_handle(s, c, t) == int(word) and unpack_handle(int(word)) == (s, c, t)
    for spec, sizes in g["growth"].items():
        s0, lam = spec.split(":")
        pol = GrowthPolicy(int(s0), lam)
        assert [pol.bucket_size(i) for i in range(len(sizes))] == sizes
    assert [GrowthPolicy(1, 2).buckets_for(c) for c in range(40)] == g["buckets_for_doubling"]
    assert next_bucket_size(GrowthPolicy(1, 2), 4) == 8


def test_exchange_host():
    assert exchange([[[1, 2, 3]]]) == [[1, 2, 3]]
    assert exchange([[[1], [2, 3]], [[4, 5], [6]]]) == [[1, 4, 5], [2, 3, 6]]
    with pytest.raises(ValueError):
        exchange([[[1], [2]], [[3]]])


def test_tables_refuse_without_gpu():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2009_07914_b200 import ExtensionMissing, SingleValueHashTable
    with pytest.raises(ExtensionMissing):
        SingleValueHashTable(1000)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _exchange_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2009_07914_b200.distributed import all_to_all_back, all_to_all_segments
    import oracle as orc
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(100 + rank)
        keys = rng.integers(0, 1 << 62, size=5000 + 37 * rank, dtype=np.uint64)
        perm, offsets = orc.multi_split(keys, world)  # test-side plan (the GPU split is tested on GPU)
        send = torch.from_numpy(keys[perm].view(np.int64))
        counts = np.diff(offsets).astype(np.int64).tolist()
        recv, rcounts = all_to_all_segments(send, counts)
        got = recv.numpy().view(np.uint64)
        ok = all(orc.route(int(k), world) == rank for k in got[:2000])
        # answer every received key with key ^ 1 and send it back
        back = all_to_all_back(torch.from_numpy((got ^ np.uint64(1)).view(np.int64)), rcounts, counts)
        ok &= bool((back.numpy().view(np.uint64) == (keys[perm] ^ np.uint64(1))).all())
        total = torch.tensor([len(got)], dtype=torch.int64)
        dist.all_reduce(total)
        q.put((rank, ok, int(total.item())))
    finally:
        dist.destroy_process_group()


def _grouped_worker(rank, world, port, q):
    """exchange_segments (the ShardedTable / bench exchange): keys and values of every
    (rank -> peer) segment in one grouped send/recv, then results back."""
    import torch.distributed as dist
    from paper_2009_07914_b200.distributed import exchange_segments
    import oracle as orc
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(200 + rank)
        n = 3000 + 101 * rank
        keys = rng.integers(0, 1 << 31, size=n, dtype=np.uint64).astype(np.uint32)
        vals = (keys.astype(np.uint64) * 7 % (1 << 32)).astype(np.uint32)
        perm, offsets = orc.multi_split(keys.astype(np.uint64), world)
        send = np.diff(offsets).astype(np.int64).tolist()
        sc = torch.tensor(send, dtype=torch.int64)
        rc = torch.empty(world, dtype=torch.int64)
        dist.all_to_all_single(rc, sc)
        recv = rc.tolist()
        kt = torch.from_numpy(keys[perm].view(np.int32))
        vt = torch.from_numpy(vals[perm].view(np.int32))
        rk, rv = exchange_segments([kt, vt], send, recv)
        gk = rk.numpy().view(np.uint32)
        ok = all(orc.route(int(k), world) == rank for k in gk)
        ok &= bool((rv.numpy().view(np.uint32) == (gk.astype(np.uint64) * 7 % (1 << 32)).astype(np.uint32)).all())
        # answer with (key + 1, key & 1) and send both arrays back in one group
        bv, bf = exchange_segments([rk + 1, (rk & 1).to(torch.uint8)], recv, send)
        ok &= bool((bv.numpy() == kt.numpy() + 1).all()) and bool((bf.numpy() == (kt.numpy() & 1)).all())
        total = torch.tensor([len(gk)], dtype=torch.int64)
        dist.all_reduce(total)
        q.put((rank, ok, int(total.item())))
    except Exception as e:
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_grouped_exchange_gloo(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grouped_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
    assert all(ok for _, ok, _ in res), res
    assert res[0][2] == sum(3000 + 101 * r for r in range(world))


def test_all_to_all_exchange_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert all(ok for _, ok, _ in res)
    assert res[0][2] == 5000 + 5037


def test_sorted_greedy_scan_model():
    """The sorted-greedy region insert's parallel form (csrc/staged.cu k_st_insert_sg: clamped
    additions composed by one scan over the window starts) equals the sequential greedy slot for
    slot on random regions with pre-occupied slots, and keeps far more keys in window 0 than an
    arbitrary claim order (tools/sim_sorted_greedy.py)."""
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("sim_sg", os.path.join(root, "tools", "sim_sorted_greedy.py"))
    sim = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(sim)
    rng = np.random.default_rng(9)
    for _ in range(4):
        pre = rng.uniform(0, 0.5)
        occ = rng.random(sim.R) < pre
        m = int(sim.R * rng.uniform(0.6, 1.05) * (1 - pre))
        lo = np.sort(rng.integers(0, sim.R - sim.W + 1, size=m))
        assert sim.sequential(lo, occ) == sim.clamp_scan(lo, occ)
    m = int(sim.R * 0.95)
    lo = rng.integers(0, sim.R - sim.W + 1, size=m)
    empty = np.zeros(sim.R, bool)
    assert sim.sequential(np.sort(lo), empty).count(-1) * 5 < sim.sequential(lo, empty).count(-1)
