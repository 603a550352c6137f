"""Headline benchmark: B200 COPS single-value table, 2^28 packed 32|32 pairs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--sweep]

One step = clear the table (K0) + bulk insert n pairs (K1) + bulk retrieve the
same n keys (K2), on a table sized ceil(n / load) (BASELINE.json configs[1]:
packed 32|32, load 0.95).  value = 2n / step time (inserts + retrievals per
second, whole job).  Inputs (2 GiB of keys + values) exceed the 126 MB L2, so
no explicit flush is needed between steps.

N > 1 (torchrun, one process per GPU, NCCL): every rank owns 2^28 globally
unique keys; insert and retrieve go through the hash-partitioned ShardedTable
(split -> NCCL all_to_all -> local kernel -> all_to_all back), weak scaling.

--impl reference times the reference's algorithm on the host cores (the C
restatement in oracle/, all OpenMP threads) on a bounded sample of the same
workload; the reference package itself is pure Python and cannot travel to
the GPU box.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_DEFAULT = 1 << 28
LOAD_DEFAULT = 0.95
G_DEFAULT = 8
INSERT_BYTES = 73  # 4 key + 4 value + 1 status + 32 sector read + 32 sector write-back
RETRIEVE_BYTES = 41  # 4 key + 4 value + 1 found + 32 sector read
METRIC = "G ops/s (bulk insert + bulk retrieve, 2^28 packed 32|32 pairs per GPU, load 0.95)"


# ------------------------------------------------------------------ workload

def _inv_xorshift(y: int, s: int) -> int:
    x = y
    for _ in range(32 // s + 1):
        x = y ^ (x >> s)
    return x & 0xFFFFFFFF


def fmix32_inverse(y: int) -> int:
    y = _inv_xorshift(y, 16)
    y = (y * pow(0xC2B2AE35, -1, 1 << 32)) & 0xFFFFFFFF
    y = _inv_xorshift(y, 13)
    y = (y * pow(0x85EBCA6B, -1, 1 << 32)) & 0xFFFFFFFF
    return _inv_xorshift(y, 16)


def fmix32_host(x: int) -> int:
    x ^= x >> 16
    x = (x * 0x85EBCA6B) & 0xFFFFFFFF
    x ^= x >> 13
    x = (x * 0xC2B2AE35) & 0xFFFFFFFF
    return x ^ (x >> 16)


def make_keys(rank: int, n: int, world: int, device):
    """n globally unique 32-bit keys per rank: fmix32 (a bijection) of a global index
    range, with the two sentinel images swapped for out-of-range indices."""
    import torch
    total = n * world
    idx = torch.arange(rank * n, (rank + 1) * n, dtype=torch.int64, device=device)
    x = idx & 0xFFFFFFFF
    x = x ^ (x >> 16)
    x = (x * 0x85EBCA6B) & 0xFFFFFFFF
    x = x ^ (x >> 13)
    x = (x * 0xC2B2AE35) & 0xFFFFFFFF
    x = x ^ (x >> 16)
    spare = total
    for sentinel in (0xFFFFFFFF, 0xFFFFFFFE):
        pre = fmix32_inverse(sentinel)
        if rank * n <= pre < (rank + 1) * n:
            while fmix32_host(spare) in (0xFFFFFFFF, 0xFFFFFFFE):
                spare += 1
            x[pre - rank * n] = fmix32_host(spare)
            spare += 1
    keys = x.to(torch.int64).to(torch.int32)  # bit pattern of the uint32 keys
    vals = (idx + 1).to(torch.int32)         # values = global index + 1 (bench.py:159-161)
    return keys, vals


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """Samples SM clocks and clock-event (throttle) reasons DURING the timed region.

    NVML from a background thread every 5 ms (the timed region is ~0.1 s, shorter than
    nvidia-smi's own start-up); `nvidia-smi -lms` only if NVML is unavailable.  __enter__
    returns after the first sample so the region is covered from its start."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.samples = []          # (sm_mhz, max_mhz, set(reasons))
        self.source = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._handle = self._nvml_handle(pynvml, device)
            self._nvml = pynvml
            self._bits = (pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                          pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap)
            self._max = float(pynvml.nvmlDeviceGetMaxClockInfo(self._handle, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nvml = None

    @staticmethod
    def _nvml_handle(pynvml, device: int):
        try:   # CUDA ordinal -> NVML handle through the PCI bus id (CUDA_VISIBLE_DEVICES-proof)
            import torch
            pr = torch.cuda.get_device_properties(device)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(device)

    def _sample_nvml(self):
        nv = self._nvml
        sm = float(nv.nvmlDeviceGetClockInfo(self._handle, nv.NVML_CLOCK_SM))
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._handle)
        return sm, self._max, {n for n, b in zip(self.NAMES, self._bits) if bits & b}

    def _loop(self):
        import time as _t
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample_nvml())
            except Exception:
                pass
            self._first.set()
            _t.sleep(0.005)

    def __enter__(self):
        import threading
        if self._nvml is not None:
            self.source = "nvml"
            self._stop, self._first = threading.Event(), threading.Event()
            self._thread = threading.Thread(target=self._loop, daemon=True)
            self._thread.start()
            self._first.wait(5)
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi"
            self._first_line = self.proc.stdout.readline()   # wait until sampling is live
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self._nvml is not None:
            self._stop.set()
            self._thread.join(5)
            try:
                self.samples.append(self._sample_nvml())
            except Exception:
                pass
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            for ln in [self._first_line] + out.splitlines():
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    sm, mx = float(parts[0]), float(parts[1])
                except ValueError:
                    continue
                self.samples.append((sm, mx, {n for n, f in zip(self.NAMES, parts[2:6])
                                              if f.lower().startswith("active")}))

    def summary(self) -> dict:
        sm = [s[0] for s in self.samples]
        mx = max((s[1] for s in self.samples), default=0.0)
        reasons = set().union(*(s[2] for s in self.samples)) if self.samples else set()
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm), "source": self.source}


def measured_peak() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def ncu_traffic():
    """dram bytes per launch from the committed ncu --set full capture (profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


# ------------------------------------------------------------------ CPU arm

def cpu_run(n: int, load: float, steps: int, warmup: int, threads: int):
    """The reference algorithm on the host (oracle/ C restatement, OpenMP threads)."""
    import numpy as np
    import oracle
    rng = np.random.default_rng(42)
    keys = rng.permutation(np.unique(rng.integers(1, (1 << 32) - 3, size=n + n // 8 + 16,
                                                  dtype=np.uint64)))[:n]
    vals = np.arange(1, n + 1, dtype=np.uint64)
    cap = math.ceil(n / load)
    times = []
    for s in range(warmup + steps):
        t = oracle.OracleSingle(cap, group_width=G_DEFAULT, key_bits=32, packed=True)
        t0 = time.perf_counter()
        st = t.insert_bulk(keys, vals, threads=threads)
        got, found = t.retrieve_bulk(keys, threads=threads)
        dt = time.perf_counter() - t0
        if s == 0 and not ((st == 0).all() and found.all() and (got == vals).all()):
            raise SystemExit("reference arm verification failed")
        if s >= warmup:
            times.append(dt)
        del t
    return 2 * n / (sum(times) / len(times)) / 1e9, times


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def python_reference_rate(n: int, load: float):
    """The UNMODIFIED reference package (pure Python, installed into baseline/_ref with
    pip --target) on a small sample of the same workload: SingleValueHashTable packed
    32|32, g = 8, insert_bulk + retrieve_bulk, one thread (its thread pool gives no
    speed-up: GIL).  Informational next to the C restatement the arm times."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "coophash")):
        return None
    import numpy as np
    sys.path.insert(0, ref)
    try:
        from coophash import SingleValueHashTable as RefTable
    finally:
        sys.path.remove(ref)
    rng = np.random.default_rng(42)
    keys = rng.permutation(np.unique(rng.integers(1, (1 << 32) - 3, size=n + n // 8 + 16,
                                                  dtype=np.uint64)))[:n].tolist()
    vals = list(range(1, n + 1))
    t = RefTable(math.ceil(n / load), layout="packed", key_bits=32, value_bits=32, group_width=G_DEFAULT)
    t0 = time.perf_counter()
    t.insert_bulk(list(zip(keys, vals)))
    got = t.retrieve_bulk(keys)
    dt = time.perf_counter() - t0
    if got != vals:
        raise SystemExit("python reference verification failed")
    return {"value": 2 * n / dt / 1e9, "unit": "G ops/s", "cores": 1, "kind": "reference",
            "sample": f"{n} unique keys insert + retrieve at load {load} (coophash from baseline/_ref)",
            "seconds": dt}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n = args.cpu_n
    value, times = cpu_run(n, args.load, args.steps, args.warmup, threads)
    try:
        pyref = python_reference_rate(1 << 16, args.load)
    except Exception as err:  # informational only
        pyref = {"error": repr(err)}
    line = {
        "metric": METRIC, "value": value, "unit": "G ops/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": "SingleValueHashTable packed 32|32, insert + retrieve, load 0.95",
                   "keys_per_step": n, "load": args.load, "group_width": G_DEFAULT,
                   "note": "CPU: oracle/ C restatement of the reference algorithm (the Python "
                           "reference cannot travel to the box); bounded sample of the workload"},
        "cpu_baseline": {"value": value, "unit": "G ops/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"{n} unique keys insert + retrieve at load {args.load}, per step"},
        "e2e": {"value": value, "unit": "G ops/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_python": pyref,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm

def relaunch(gpus: int) -> None:
    """`python bench.py --gpus N` outside torchrun: re-run this command as N ranks, one per
    GPU, on one node (torch.distributed.run, rendezvous on 127.0.0.1)."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--n", type=int, default=N_DEFAULT)
    ap.add_argument("--load", type=float, default=LOAD_DEFAULT)
    ap.add_argument("--group-width", type=int, default=G_DEFAULT)
    ap.add_argument("--cpu-n", type=int, default=1 << 24)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sweep", default="", help="write a g x load sweep to this JSON file")
    ap.add_argument("--locality", default="auto", choices=("auto", "on", "off", "staged"),
                    help="region-ordered execution of the batch (csrc/locality.cu)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args.gpus)  # one process per GPU (torchrun, NCCL); does not return

    import torch
    import torch.distributed as dist
    from paper_2009_07914_b200 import SingleValueHashTable, _lib
    from paper_2009_07914_b200.distributed import ShardedTable

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one process per GPU "
                         "(python bench.py --gpus N re-launches itself under torchrun)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    n = args.n
    keys, vals = make_keys(rank, n, world, dev)
    cap = math.ceil(n * (1.001 if world > 1 else 1.0) / args.load)
    table = SingleValueHashTable(cap, layout="packed", key_bits=32, value_bits=32,
                                 group_width=args.group_width, device=local)
    table.set_locality(args.locality)
    front = ShardedTable(table) if world > 1 else table
    stream = torch.cuda.current_stream(dev)
    status = torch.empty(n, dtype=torch.uint8, device=dev)
    out_v = torch.empty(n, dtype=torch.int32, device=dev)
    out_f = torch.empty(n, dtype=torch.uint8, device=dev)

    def step(events=None):
        if events is not None:
            events[0].record(stream)
        _lib.check(_lib.lib().ch_clear(table._dt.handle, stream.cuda_stream), "clear")
        if events is not None:
            events[1].record(stream)
        if world > 1:
            st = front.insert_device(keys, vals)
        else:
            st = table.insert_device(keys, vals, status=status)
        if events is not None:
            events[2].record(stream)
        if world > 1:
            v, f = front.retrieve_device(keys)
        else:
            v, f = table.retrieve_device(keys, values_out=out_v, found_out=out_f)
        if events is not None:
            events[3].record(stream)
        return st, v, f

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    table.kernel_times()
    table.kernel_timing(True)
    launches0 = _lib.lib().ch_kernel_launches()
    with ClockSampler(local) as clocks:
        barrier()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for s in range(args.steps):
            st, v, f = step(evs[s])
        t_end.record(stream)
        barrier()
    launches = _lib.lib().ch_kernel_launches() - launches0
    table.kernel_timing(False)
    ktimes = table.kernel_times()  # probe kernels in launch order: [insert, lookup] per step
    k_ins_ms = statistics.mean(ktimes[0::2]) if len(ktimes) >= 2 else float("nan")
    k_ret_ms = statistics.mean(ktimes[1::2]) if len(ktimes) >= 2 else float("nan")
    total_ms = t_start.elapsed_time(t_end)
    clear_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    ins_ms = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    ret_ms = sum(e[2].elapsed_time(e[3]) for e in evs) / args.steps

    # schedule statistics (outside the timed region): keys the staged-region pass handed
    # to the COPS probe kernels (window 0 could not decide them)
    sched = None
    if world == 1:
        _lib.check(_lib.lib().ch_clear(table._dt.handle, stream.cuda_stream), "clear")
        table.reset_probe_counters()
        table.insert_device(keys, vals, status=status)
        d_ins = table.deferred_count()
        table.reset_probe_counters()
        table.retrieve_device(keys, values_out=out_v, found_out=out_f)
        c_ret = table.probe_counters()
        sched = {"deferred_insert_frac": d_ins / n, "deferred_retrieve_frac": table.deferred_count() / n,
                 "retrieve_mean_attempts": c_ret.attempts / max(1, c_ret.ops)}
        st, v, f = status, out_v, out_f
        torch.cuda.synchronize()

    # verification (outside the timed region): every key found with its value
    ok = bool((st == 0).all().item() and (f == 1).all().item() and (v == vals).all().item())
    t_max = torch.tensor([total_ms, ins_ms, ret_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        okt = torch.tensor([0 if ok else 1], device=dev)
        dist.all_reduce(okt)
        ok = okt.item() == 0
    total_ms, ins_ms_max, ret_ms_max = t_max.tolist()
    ms_per_step = total_ms / args.steps
    value = 2 * n * world / (ms_per_step * 1e-3) / 1e9

    # ---- e2e: host buffers through the public API, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        hk = keys.cpu().pin_memory()
        hv = vals.cpu().pin_memory()
        host_v = torch.empty(n, dtype=torch.int32).pin_memory()
        host_f = torch.empty(n, dtype=torch.uint8).pin_memory()
        host_s = torch.empty(n, dtype=torch.uint8).pin_memory()

        def e2e_step():
            _lib.check(_lib.lib().ch_clear(table._dt.handle, stream.cuda_stream), "clear")
            if world > 1:
                dk = hk.to(dev, non_blocking=True)
                dv = hv.to(dev, non_blocking=True)
                front.insert_device(dk, dv)
                v2, f2 = front.retrieve_device(hk.to(dev, non_blocking=True))
                host_v.copy_(v2, non_blocking=True)
                host_f.copy_(f2, non_blocking=True)
                return host_v, host_f
            # public API, pinned host buffers in and out; the insert does not block the host, so
            # the retrieve's copies overlap its last kernels (one synchronisation per step)
            table.insert_host(hk, hv, status_out=host_s, sync=False)
            return table.retrieve_host(hk, values_out=host_v, found_out=host_f)

        for _ in range(2):
            e2e_step()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            res_v, res_f = e2e_step()
        e1.record(stream)
        barrier()
        e2e_ms = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        e2e_ok = bool((res_v == hv).all().item() and (res_f == 1).all().item() and (host_s == 0).all().item())
        ok = ok and e2e_ok
        e2e = {"value": 2 * n * world / (e2e_ms.item() * 1e-3) / 1e9, "unit": "G ops/s",
               "h2d_bytes_per_step": 3 * 4 * n, "d2h_bytes_per_step": 6 * n,
               "ms_per_step": e2e_ms.item(),
               "path": "pinned host keys/values -> insert_host(sync=False) -> pinned host statuses; pinned host "
                       "keys -> retrieve_host -> pinned host values/found (chunked, H2D / kernels / D2H "
                       "overlapped on 3 streams, persistent staging buffers, one host sync per step)"}

    if rank == 0:
        peak, peak_kind = measured_peak()
        ins_gops = n * world / (ins_ms_max * 1e-3) / 1e9
        ret_gops = n * world / (ret_ms_max * 1e-3) / 1e9
        # dominant kernel: the longer of the insert / retrieve region kernels, timed with
        # CUDA events inside the library on the stream they run on (one launch each per op).
        # Algorithmic bytes per launch: staged region passes stream the table
        # (read + write back for insert) and per key 10 B (insert: key, value, window start;
        # statuses are pre-set) / 11 B (retrieve: key, window start, value, found); direct
        # probes touch one 32 B sector per key.
        sched_name = table.batch_schedule(n)
        c = table.capacity
        if sched_name == "staged":
            # the step's ch_clear is deferred into the insert (api.cu pending_clear: a staged-size
            # packed table), which then writes the regions without reading them
            lazy = os.environ.get("CH_LAZY_CLEAR", "1") != "0" and c * 8 >= 256 << 20
            cand = [("k_st_insert_sg (staged insert)", k_ins_ms, (8 if lazy else 16) * c + 10 * n),
                    ("k_st_lookup_q (staged retrieve)", k_ret_ms, 8 * c + 11 * n)]
        else:
            cand = [("k_insert", k_ins_ms, INSERT_BYTES * n), ("k_lookup", k_ret_ms, RETRIEVE_BYTES * n)]
        kname, kms, kbytes_launch = max(cand, key=lambda x: x[1])
        keys_per_launch = n  # weak scaling: ~n keys per rank and launch
        achieved = kbytes_launch / (kms * 1e-3) / 1e9
        kbytes = kbytes_launch / keys_per_launch
        tr = ncu_traffic().get(kname) if world == 1 else None
        traffic = tr.get("dram_bytes") if isinstance(tr, dict) else tr
        cpu = None
        if world == 1 and not args.no_cpu:
            threads = os.cpu_count() or 1
            cv, _ = cpu_run(args.cpu_n, args.load, 1, 1, threads)
            cpu = {"value": cv, "unit": "G ops/s", "cores": threads, "kind": "port", "cpu_model": cpu_model(),
                   "sample": f"{args.cpu_n} unique keys, insert + retrieve at load {args.load} "
                             "(oracle/ C restatement, OpenMP)"}
        line = {
            "metric": METRIC, "value": value, "unit": "G ops/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": "SingleValueHashTable packed 32|32 (BASELINE configs[1])" if world == 1 else
                       "ShardedTable packed 32|32, hash-partitioned, NCCL all_to_all (BASELINE configs[4])",
                       "keys_per_gpu": n, "load": args.load, "capacity_per_gpu": table.capacity,
                       "group_width": args.group_width, "locality": args.locality,
                       "parallelism": f"hash-partitioned x{world}",
                       "l2": "inputs (2 GiB) and table (2.1 GiB) exceed the 126 MB L2; no flush"},
            "insert_gops": ins_gops, "retrieve_gops": ret_gops,
            "phase_ms": {"clear": clear_ms, "insert": ins_ms, "retrieve": ret_ms,
                         "probe_insert": k_ins_ms, "probe_retrieve": k_ret_ms},
            "schedule_kind": sched_name,
            "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "bytes_per_op": kbytes, "bytes_per_launch": kbytes_launch,
                         "ops_per_launch": keys_per_launch, "traffic": traffic,
                         "kernel_ms": kms},
            "schedule": sched,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks.summary(),
            "verified": ok,
        }
        print(json.dumps(line), flush=True)

    if args.sweep and world == 1:
        sweep(args.sweep, n, dev, args.locality)
    if world > 1:
        dist.destroy_process_group()
    if not ok:
        sys.exit(2)


def sweep(path: str, n: int, dev, locality: str = "auto") -> None:
    """g x load sweep of the single-GPU insert / retrieve rates (BASELINE configs[1])."""
    import torch
    from paper_2009_07914_b200 import SingleValueHashTable, _lib
    keys, vals = make_keys(0, n, 1, dev)
    rows = []
    stream = torch.cuda.current_stream(dev)
    for load in (0.8, 0.9, 0.95):
        for g in (1, 2, 4, 8, 16, 32):
            t = SingleValueHashTable(math.ceil(n / load), layout="packed", key_bits=32, value_bits=32,
                                     group_width=g, device=dev.index)
            t.set_locality(locality)
            st = torch.empty(n, dtype=torch.uint8, device=dev)
            ov = torch.empty(n, dtype=torch.int32, device=dev)
            of = torch.empty(n, dtype=torch.uint8, device=dev)
            ins, ret = [], []
            for r in range(4):
                _lib.check(_lib.lib().ch_clear(t._dt.handle, stream.cuda_stream))
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                e[0].record(stream)
                t.insert_device(keys, vals, status=st)
                e[1].record(stream)
                t.retrieve_device(keys, values_out=ov, found_out=of)
                e[2].record(stream)
                torch.cuda.synchronize()
                if r:
                    ins.append(e[0].elapsed_time(e[1]))
                    ret.append(e[1].elapsed_time(e[2]))
            c = t.probe_counters()
            rows.append({"load": load, "group_width": g, "locality": locality, "insert_ms": statistics.mean(ins),
                         "retrieve_ms": statistics.mean(ret), "insert_gops": n / statistics.mean(ins) / 1e6,
                         "retrieve_gops": n / statistics.mean(ret) / 1e6,
                         "mean_attempts": c.attempts / max(1, c.ops)})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
            del t
            torch.cuda.empty_cache()
    with open(path, "w") as fh:
        json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
