"""GPU parity: distribution layer (K10 split, K11 scatter, DistributedTable)."""
import os
import random
from collections import Counter

import numpy as np
import pytest
import torch

import oracle as orc
from gold import ints, load

pytestmark = pytest.mark.gpu

from paper_2009_07914_b200 import (DistributedTable, InsertStatus, MultiValueHashTable,  # noqa: E402
                                   ShardMode, ShardRouter, SingleValueHashTable, multi_split)
from paper_2009_07914_b200.distributed import ShardedTable, split_device  # noqa: E402

INSERTED = InsertStatus.INSERTED


def test_split_matches_golden_plans():
    g = load("distributed.json")
    keys = ints(g["keys"])
    for s, plan in g["splits"].items():
        p = multi_split(keys, ShardRouter(int(s)))
        assert p.permutation == plan["perm"] and p.offsets == plan["offsets"]


@pytest.mark.parametrize("shards", [1, 2, 3, 8, 37, 256])
def test_large_split_is_stable_and_exact(shards):
    n = (1 << 20) + 123
    rng = np.random.default_rng(shards)
    keys = rng.integers(0, 1 << 63, size=n, dtype=np.uint64)
    vals = rng.integers(0, 1 << 31, size=n, dtype=np.uint64).astype(np.uint32)
    k = torch.from_numpy(keys.view(np.int64)).cuda()
    v = torch.from_numpy(vals.view(np.int32)).cuda()
    perm, offsets, kout, vout = split_device(k, shards, v)
    rperm, roff = orc.multi_split(keys, shards)
    assert (perm.cpu().numpy() == rperm.astype(np.int64)).all()
    assert (offsets.cpu().numpy() == roff.astype(np.int64)).all()
    assert (kout.cpu().numpy().view(np.uint64) == keys[rperm]).all()
    assert (vout.cpu().numpy().view(np.uint32) == vals[rperm]).all()


def test_custom_router_partition():          # test_distributed.py:15-23,36-48
    class Fixed:
        def __init__(self, mapping, num_shards):
            self.mapping, self.num_shards = mapping, num_shards

        def route(self, key):
            return self.mapping[key]

    keys = ["a", "b", "c", "d"]
    plan = multi_split(keys, Fixed({"a": 1, "b": 0, "c": 1, "d": 0}, 2))
    assert [keys[i] for i in plan.permutation] == ["b", "d", "a", "c"]
    assert plan.offsets == [0, 2, 4] and plan.segment(0) == [1, 3]
    assert multi_split([10, 20, 30], ShardRouter(1)).permutation == [0, 1, 2]


def _workload(n=4096, r=8, seed=9):
    rng = random.Random(seed)
    return [(rng.randrange(1, n // r + 1), i) for i, _ in enumerate(range(n), start=1)]


def test_distributed_multi_equals_monolithic():   # test_distributed.py:82-96
    pairs = _workload()
    n = len(pairs)
    mono = MultiValueHashTable(int(n / 0.8))
    mono.insert_bulk(pairs)
    with DistributedTable(4, lambda s: MultiValueHashTable(int(n / 4 / 0.7))) as dt:
        assert all(st == INSERTED for st in dt.insert_bulk(pairs))
        queries = sorted({k for k, _ in pairs}) + [99_999]
        offsets, flat = dt.retrieve_bulk(queries)
        mo, mf = mono.retrieve_bulk(queries)
        for i in range(len(queries)):
            assert sorted(flat[offsets[i]:offsets[i + 1]]) == sorted(mf[mo[i]:mo[i + 1]])
        for k in {k for k, _ in pairs}:
            holders = [s for s, t in enumerate(dt.shards) if t.count(k) > 0]
            assert holders == [dt.router.route(k)]
        assert dt.count_bulk(queries) == mono.count_bulk(queries)


def test_distributed_single_vs_golden():
    g = load("distributed.json")
    pairs = [tuple(p) for p in g["pairs"]]
    dup_keys = {k for k, c in Counter(k for k, _ in pairs).items() if c > 1}
    for s_str, exp in g["single"].items():
        S = int(s_str)
        with DistributedTable(S, lambda _: SingleValueHashTable(4096)) as dt:
            st = dt.insert_bulk(pairs)
            for (k, _), got, ref in zip(pairs, st, exp["status"]):
                if k not in dup_keys:
                    assert got.value == ref
            got = dt.retrieve_bulk(list(range(0, 3005)))
            for k, a, b in zip(range(3005), got, exp["retrieve"]):
                if k in dup_keys:
                    assert (a is None) == (b is None)
                    assert a in {v for kk, v in pairs if kk == k}
                else:
                    assert a == b


def test_independent_modes():                # test_distributed.py:108-171
    pairs = _workload(n=2048, r=4)
    with DistributedTable(4, lambda s: MultiValueHashTable(1024), mode=ShardMode.INDEPENDENT) as dt:
        assert all(st == INSERTED for st in dt.insert_bulk(pairs))
        ref = Counter(k for k, _ in pairs)
        q = sorted(ref)
        assert dt.count_bulk(q) == [ref[x] for x in q]
    with DistributedTable(3, lambda s: SingleValueHashTable(64), mode=ShardMode.INDEPENDENT) as dt:
        for s, table in enumerate(dt.shards):
            table.insert(42, 100 + s)
        assert dt.retrieve_bulk([42]) == [100]
    with DistributedTable(4, lambda s: MultiValueHashTable(64), mode=ShardMode.INDEPENDENT) as dt:
        dt.insert_bulk([(k, k) for k in range(1, 41)])
        assert [t.occupied for t in dt.shards] == [10, 10, 10, 10]


def test_mode_equivalence_to_monolithic():   # test_distributed.py:149-162
    pairs = _workload(n=2048, r=8, seed=13)
    queries = sorted({k for k, _ in pairs})
    mono = MultiValueHashTable(4096)
    mono.insert_bulk(pairs)
    mo, mf = mono.retrieve_bulk(queries)
    for mode in (ShardMode.DISTRIBUTED, ShardMode.INDEPENDENT):
        with DistributedTable(4, lambda s: MultiValueHashTable(1024), mode=mode) as dt:
            dt.insert_bulk(pairs)
            o, f = dt.retrieve_bulk(queries)
            for i in range(len(queries)):
                assert sorted(f[o[i]:o[i + 1]]) == sorted(mf[mo[i]:mo[i + 1]]), mode


def test_sharded_table_single_rank_nccl():
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        local = SingleValueHashTable(1 << 16, layout="packed", key_bits=32, value_bits=32)
        st = ShardedTable(local)
        keys = torch.arange(1, 40_001, dtype=torch.int32, device="cuda")
        assert (st.insert_device(keys, keys * 3).cpu() == 0).all()
        v, f = st.retrieve_device(keys)
        assert f.cpu().bool().all() and (v.cpu() == keys.cpu() * 3).all()
    finally:
        dist.destroy_process_group()


def _sharded_worker(rank, world, port, q):
    """One rank of a 2-rank ShardedTable job on cuda:0 (gloo exchange staged through host
    memory; NCCL refuses two ranks on one GPU).  The data path (split -> exchange -> local
    insert/retrieve -> exchange back -> scatter) is the one bench.py runs under torchrun."""
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        n, shared = 150_000, 20_000
        own = torch.arange(1, n + 1, dtype=torch.int64) + rank * n       # disjoint per rank
        common = torch.arange(10 * n, 10 * n + shared, dtype=torch.int64)  # inserted by both
        keys = torch.cat([own, common]).to(torch.int32).cuda()
        keys = keys[torch.randperm(keys.numel(), device="cuda")]
        table = SingleValueHashTable(1 << 19, layout="packed", key_bits=32, value_bits=32)
        st = ShardedTable(table)
        status = st.insert_device(keys, keys * 3).cpu()
        ins = torch.tensor([int((status == 0).sum()), int((status == 1).sum()), table.occupied])
        dist.all_reduce(ins)
        # every rank asks for all keys (its own, the peer's, the shared ones, and misses)
        allk = torch.arange(1, world * n + 1, dtype=torch.int32)
        q_keys = torch.cat([allk, common.to(torch.int32), torch.arange(20 * n, 20 * n + 999, dtype=torch.int32)])
        v, f = st.retrieve_device(q_keys.cuda())
        v, f = v.cpu(), f.cpu().bool()
        hit = q_keys.numel() - 999
        ok = bool(f[:hit].all()) and not bool(f[hit:].any()) and bool((v[:hit] == q_keys[:hit] * 3).all())
        q.put((rank, ok, ins.tolist()))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def test_sharded_table_world2_one_gpu():
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(60)
    assert all(ok for _, ok, _ in res), res
    inserted, dup, size = res[0][2]
    assert inserted == 2 * 150_000 + 20_000 == size     # each shared key lands once
    assert dup == 20_000                                 # ...and its second copy is DUPLICATE


# ---------------------------------------------------------------- ch_dist_* (C ABI)
from paper_2009_07914_b200.distributed import (NativeDist, gather_device32, route_split_device32,  # noqa: E402
                                               scatter_device32, split_device32)


@pytest.mark.parametrize("shards", [1, 2, 4, 8])
def test_native_dist_per_source_batches(shards):
    """ch_dist_insert / ch_dist_retrieve with one batch per source: every key lands on
    route(k) (distributed.py:44-45), statuses / values / found flags exact vs the oracle."""
    rng = np.random.default_rng(70 + shards)
    per = 50_000
    allk = rng.permutation(np.unique(rng.integers(1, (1 << 32) - 3, size=shards * per * 2,
                                                  dtype=np.uint64)))[: shards * per + 5000]
    src_keys = [allk[s * per:(s + 1) * per] for s in range(shards)]
    # a few keys repeated across sources: exactly one INSERTED each
    dup = allk[:500]
    src_keys[-1] = np.concatenate([src_keys[-1], dup])
    src_vals = [(k * 3 % (1 << 32)).astype(np.uint64) for k in src_keys]
    tables = [SingleValueHashTable(int(shards * per * 1.2 / shards) + 4096, layout="packed", key_bits=32,
                                   value_bits=32) for _ in range(shards)]
    nd = NativeDist(tables, transport="copy")
    assert nd.transport == "copy"
    to32 = lambda a: torch.from_numpy(a.astype(np.uint32).view(np.int32)).cuda()
    st = nd.insert([to32(k) for k in src_keys], [to32(v) for v in src_vals])
    codes = np.concatenate([s.cpu().numpy() for s in st])
    assert int((codes == 0).sum()) == shards * per and int((codes == 1).sum()) == 500
    assert sum(t.occupied for t in tables) == shards * per
    for s, t in enumerate(tables):  # placement: only keys routed to s live on s
        probe = allk[: shards * per][:20000]
        v, f = t.retrieve_device(to32(probe))
        routed = np.array([orc.route(int(k), shards) for k in probe]) == s
        assert (f.cpu().numpy().astype(bool) == routed).all()
    miss = allk[shards * per:]
    q = [to32(np.concatenate([src_keys[s][::-1], miss])) for s in range(shards)]
    res = nd.retrieve(q)
    for s, (v, f) in enumerate(res):
        nk = len(src_keys[s])
        fv = f.cpu().numpy().astype(bool)
        assert fv[:nk].all() and not fv[nk:].any()
        assert (v.cpu().numpy()[:nk].view(np.uint32) == src_vals[s][::-1].astype(np.uint32)).all()
    nd.close()


def test_native_dist_nccl_one_device():
    t = SingleValueHashTable(1 << 16, layout="packed", key_bits=32, value_bits=32)
    nd = NativeDist([t], transport="nccl")
    assert nd.transport == "nccl"
    keys = torch.arange(1, 30_001, dtype=torch.int32, device="cuda")
    (st,) = nd.insert([keys], [keys * 5])
    assert (st.cpu() == 0).all()
    ((v, f),) = nd.retrieve([keys])
    assert f.cpu().bool().all() and (v.cpu() == keys.cpu() * 5).all()
    nd.close()


def test_native_dist_rejects_bad_shards():
    m = MultiValueHashTable(1024)
    with pytest.raises(ValueError):
        NativeDist([m])
    a = SingleValueHashTable(1024, layout="packed", key_bits=32, value_bits=32)
    b = SingleValueHashTable(1024, key_bits=64, value_bits=64)
    with pytest.raises(ValueError):
        NativeDist([a, b])
    with pytest.raises(ValueError):   # NCCL needs one shard per device
        NativeDist([a, SingleValueHashTable(1024, layout="packed", key_bits=32, value_bits=32)], transport="nccl")


@pytest.mark.parametrize("shards", [1, 5, 256])
def test_split32_and_scatter32(shards):
    n = (1 << 20) + 77
    rng = np.random.default_rng(shards)
    keys = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    vals = rng.integers(0, 1 << 31, size=n, dtype=np.uint64).astype(np.uint32)
    k = torch.from_numpy(keys.view(np.int32)).cuda()
    v = torch.from_numpy(vals.view(np.int32)).cuda()
    perm, offsets, kout, vout = split_device32(k, shards, v)
    rperm, roff = orc.multi_split(keys.astype(np.uint64), shards)
    assert (perm.cpu().numpy().view(np.uint32) == rperm.astype(np.uint32)).all()
    assert (offsets.cpu().numpy() == roff.astype(np.int64)).all()
    assert (kout.cpu().numpy().view(np.uint32) == keys[rperm]).all()
    assert (vout.cpu().numpy().view(np.uint32) == vals[rperm]).all()
    back = scatter_device32(vout, perm, torch.empty_like(v))
    assert (back.cpu().numpy().view(np.uint32) == vals).all()


def test_split_of_empty_batch():
    k = torch.empty(0, dtype=torch.int64, device="cuda")
    perm, offsets, _, _ = split_device(k, 4)
    assert offsets.cpu().tolist() == [0, 0, 0, 0, 0]
    perm, offsets, _, _ = split_device32(k.to(torch.int32), 3)
    assert offsets.cpu().tolist() == [0, 0, 0, 0]


@pytest.mark.parametrize("shards", [1, 8, 37])
def test_route_split32_inverse_and_gather(shards):
    n = (1 << 20) + 33
    rng = np.random.default_rng(90 + shards)
    keys = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    vals = rng.integers(0, 1 << 31, size=n, dtype=np.uint64).astype(np.uint32)
    k = torch.from_numpy(keys.view(np.int32)).cuda()
    v = torch.from_numpy(vals.view(np.int32)).cuda()
    pos, offsets, kout, vout = route_split_device32(k, shards, v)
    rperm, roff = orc.multi_split(keys.astype(np.uint64), shards)
    inv = np.empty(n, dtype=np.int64)
    inv[rperm] = np.arange(n)
    assert (pos.cpu().numpy().view(np.uint32) == inv.astype(np.uint32)).all()
    assert (offsets.cpu().numpy() == roff.astype(np.int64)).all()
    assert (kout.cpu().numpy().view(np.uint32) == keys[rperm]).all()
    back = gather_device32(vout, pos, torch.empty_like(v))
    assert (back.cpu().numpy().view(np.uint32) == vals).all()


@pytest.mark.parametrize("shards", [1, 2, 3, 8, 37, 64])
def test_route_partition_one_pass(shards):
    """ch_route_part32 (ShardedTable's split): every element lands in its shard's fixed-capacity
    segment [d cap, d cap + counts[d]) at pos[i] with its value, counts are exact, and a batch
    that overflows a segment raises the flag."""
    from paper_2009_07914_b200.distributed import route_part_device32
    from paper_2009_07914_b200.probing import mix64_array
    rng = np.random.default_rng(shards)
    n = (1 << 20) + 333
    keys = rng.integers(1, (1 << 32) - 3, size=n, dtype=np.uint64)
    vals = rng.integers(0, 1 << 32, size=n, dtype=np.uint64)
    dk = torch.from_numpy(keys.astype(np.uint32).view(np.int32)).cuda()
    dv = torch.from_numpy(vals.astype(np.uint32).view(np.int32)).cuda()
    pos, cnt, flag, cap, kout, vout = route_part_device32(dk, shards, dv)
    assert int(flag.item()) == 0
    pos = pos.cpu().numpy().view(np.uint32).astype(np.int64)
    cnt = cnt.cpu().numpy()
    kout = kout.cpu().numpy().view(np.uint32)
    vout = vout.cpu().numpy().view(np.uint32)
    dest = ((mix64_array(keys) >> np.uint64(32)) % np.uint64(shards)).astype(np.int64)
    assert (cnt == np.bincount(dest, minlength=shards)).all()
    assert (pos // cap == dest).all() and (pos % cap < cnt[dest]).all()
    assert np.unique(pos).size == n
    assert (kout[pos] == keys.astype(np.uint32)).all() and (vout[pos] == vals.astype(np.uint32)).all()
    if shards > 1:  # every key to shard 0: past its capacity
        hot = keys[dest == 0][: 40_000]
        _, _, flag2, _, _, _ = route_part_device32(torch.from_numpy(np.resize(hot, n).astype(np.uint32).view(np.int32))
                                                   .cuda(), shards)
        assert int(flag2.item()) == 1
