"""Benchmark of the B200 lazy D2H snapshot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one checkpoint of the rank's shard through the public engine
API: capture() (flatten, batched small-leaf snapshot, pinned-ring
reservation, device issue of every copy) until the lazy fence is ready (all
payload bytes resident in pinned host memory). Workload at N=1 is
BASELINE.json configs[1]: a LLaMA-2-7B-shaped shard (fp32 params + fp32
master + Adam m/v, 4+12 B/param, 1164 tensors, 107.8 GB) generated in HBM.
N>1 runs one process per GPU (torchrun), each snapshotting its own C2-sized
shard of a dp=N plan (weak scaling, no collective on the data path).

The JSON line carries: value (aggregate snapshot GB/s, device-event timed,
max over ranks), the copy-variant sweep (gather kernel / copy engine /
per-size hybrid), roofline vs the PCIe Gen5 x16 host link, the per-iteration
stall under a synthetic bf16 fwd/bwd load with the device-side fence,
e2e (capture -> files durable on disk through the public API), the CPU
reference engine timed on this box's cores, clocks during the timed region,
and the number of our kernel launches.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "D2H snapshot GB/s (per GPU, 8-GPU aggregate); per-iteration ckpt stall ms"
PCIE_GEN5_X16_GBPS = 64.0  # BASELINE.json north_star host-link roofline (nominal, per direction)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md recipe)


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the unmodified reference engine (oracle/_ref)


def run_reference(steps: int, warmup: int, fsync: bool = True):
    """Reference CPU engine (oracle/_ref/ref_snapshot, built from the
    reference's own sources) on a bounded sample of the C2 workload: one
    LLaMA-7B decoder layer's params + fp32 master + Adam m/v (3.24 GB, same
    tensor shapes and 4+12 B/param). Metric = payload / (capture + lazy
    barrier), the reference's stall."""
    from paper_2406_10707_b200.workloads import llama_layer_sample
    drv = os.path.join(ROOT, "oracle", "_ref", "ref_snapshot")
    if not os.path.exists(drv):
        return None
    w = llama_layer_sample()
    tmp = tempfile.mkdtemp(prefix="lzk_refarm_", dir=ROOT)
    try:
        spec = w.write_spec(os.path.join(tmp, "sample.spec"))
        r = subprocess.run([drv, "--spec", spec, "--root", os.path.join(tmp, "ckpt"), "--repeat",
                            str(steps + warmup), "--digest", "0", "--fsync", "1" if fsync else "0",
                            "--keep-last", "1"], capture_output=True, text=True, timeout=1800)
        res = json.loads(r.stdout)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    st = res["ranks"][0]["steps"][warmup:]
    payload = st[0]["payload"]
    stall = [s["capture_s"] + s["barrier_s"] for s in st]
    persisted = [s["persisted_s"] for s in st]
    return {"payload": payload, "steps": len(st), "stall_s": stall, "persisted_s": persisted,
            "snapshot_gbps": payload * len(st) / sum(stall) / 1e9,
            "persisted_gbps": payload * len(st) / sum(persisted) / 1e9,
            "sample": f"{w.name}: 1 LLaMA-7B decoder layer, {len(w.leaves)} tensors, {payload} B payload per step, "
                      f"fsync={int(fsync)}"}


def cpu_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def reference_arm(args, rank, world):
    if rank != 0:
        return
    res = run_reference(args.steps, args.warmup)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_snapshot not built"}))
        return
    v = res["snapshot_gbps"]
    line = {"metric": METRIC, "value": round(v, 4), "unit": "GB/s", "impl": "reference", "n_gpus": world,
            "steps": res["steps"], "warmup": args.warmup,
            "ms_per_step": round(1e3 * statistics.mean(res["stall_s"]), 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": "c2-llama7b (bounded sample: 1 decoder layer)", "engine": "reference lzckpt CPU",
                       "host": cpu_info()},
            "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": 2, "kind": "reference",
                             "sample": res["sample"]},
            "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "persisted_gbps": round(res["persisted_gbps"], 4)}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm


def fits_host(bytes_per_rank: int, world: int) -> bool:
    try:
        avail = next(int(l.split()[1]) * 1024 for l in open("/proc/meminfo") if l.startswith("MemAvailable"))
    except (OSError, StopIteration):
        return True
    return bytes_per_rank * world <= 0.75 * avail


def main_ours(args, rank, world, local_rank):
    import numpy as np  # noqa: F401
    import torch
    import torch.distributed as dist

    import paper_2406_10707_b200 as lz
    from paper_2406_10707_b200.workloads import llama7b_shard

    torch.cuda.set_device(local_rank)
    dev = local_rank

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # CPU reference baseline first (rank 0, N=1 only), before we pin memory
    cpu_base = None
    if rank == 0 and world == 1 and not args.skip_cpu_baseline:
        t0 = time.time()
        cpu_base = run_reference(steps=2, warmup=1)
        log(f"[bench] reference CPU baseline: {cpu_base and round(cpu_base['snapshot_gbps'], 3)} GB/s "
            f"({time.time() - t0:.1f} s)")

    layers = args.layers
    w = llama7b_shard(layers=layers, dp=world, rank=rank)
    while not fits_host(int(w.total_bytes * 1.03), world) and layers > 1:
        layers -= 1
        w = llama7b_shard(layers=layers, dp=world, rank=rank)
    tmp = tempfile.mkdtemp(prefix=f"lzk_bench_r{rank}_", dir=ROOT)
    try:
        spec = w.write_spec(os.path.join(tmp, "w.spec"))
        t0 = time.time()
        built = lz.build_workload(spec, dev)
        torch.cuda.synchronize()
        log(f"[bench] rank {rank}: workload {w.name} layers={layers} {built.bytes / 1e9:.2f} GB "
            f"{len(w.leaves)} tensors built in {time.time() - t0:.1f} s")

        link = measure_link_ceiling(lz, dev)
        log(f"[bench] rank {rank}: host-link ceiling on this box: DMA {link['dma_gbps']} GB/s, "
            f"SM stores {link['sm_store_gbps']} GB/s")

        pool_bytes = int(built.bytes * 1.01) + (256 << 20)
        cfg = lz.EngineConfig(checkpoint_root=os.path.join(tmp, "ckpt"), host_buffer_bytes=pool_bytes,
                              large_leaf_threshold=1 << 20, fsync_on_finalize=False, flush_discard=True,
                              hugepages=True, device=dev)
        t0 = time.time()
        eng = lz.Engine(cfg, built.topo, built.rank)
        log(f"[bench] rank {rank}: pinned {pool_bytes / 1e9:.1f} GB pool in {time.time() - t0:.1f} s")
        plan = lz.plan_checkpoint(built.topo, built.model, built.step)

        def one_step(step):
            """capture -> fence-ready. Device ms = CUDA events on the snapshot
            stream (first device op -> last completion, recorded by the
            engine); host ms = capture() call -> update_barrier() return.
            Returns (device ms, host ms, payload, capture ms)."""
            h0 = time.perf_counter()
            t = eng.capture(plan, built.tree, step)
            h1 = time.perf_counter()
            eng.update_barrier(t)
            h2 = time.perf_counter()
            eng.wait_persisted(t)  # discard tier: releases the pinned segment
            return eng.ticket_device_ms(t), (h2 - h0) * 1e3, t.payload_bytes(), (h1 - h0) * 1e3

        # ---- copy-variant sweep (same bytes, each variant) ----
        variants = {}
        for name, kw in (("gather_kernel", dict(force_kernel=True)),
                         ("copy_engine", dict(force_copy_engine=True)),
                         ("hybrid", dict(ce_threshold=2 << 20))):
            eng.set_copy_variant(**kw)
            barrier()
            one_step(1)
            ms = []
            for s in range(3):
                barrier()
                dms, hms, payload, _ = one_step(2 + s)
                ms.append(max(dms, hms))
            variants[name] = round(payload / (statistics.mean(ms) * 1e-3) / 1e9, 3)
            log(f"[bench] rank {rank}: variant {name}: {variants[name]} GB/s")
        # The headline times the product default (hybrid: kernel below 2 MiB,
        # copy engines above), the configuration a trainer runs: forcing every
        # byte through the kernel takes ~7 % of the trainer's GEMM throughput
        # (tools/interference.py) even on boxes where it edges out the DMA
        # engines. All three variants are reported in variants_gbps.
        best = "hybrid"
        eng.set_copy_variant(ce_threshold=2 << 20)

        # ---- timed region ----
        for s in range(args.warmup):
            barrier()
            one_step(10 + s)
        launches0 = lz.kernel_launches()
        stats0 = eng.snapshot_stats()
        dev_ms, host_ms, cap_ms = [], [], []
        barrier()
        with ClockSampler(dev) as clocks:
            for s in range(args.steps):
                barrier()
                dms, hms, payload, cms = one_step(100 + s)
                dev_ms.append(dms)
                host_ms.append(hms)
                cap_ms.append(cms)
            barrier()
        launches = lz.kernel_launches() - launches0
        stats1 = eng.snapshot_stats()
        # conservative: the longer of device events and host capture->fence-ready
        step_ms = [max(d, h) for d, h in zip(dev_ms, host_ms)]
        t_total = max_over_ranks(sum(step_ms) * 1e-3)
        agg_bytes = sum_over_ranks(float(payload * args.steps))
        value = agg_bytes / t_total / 1e9
        per_gpu = payload * args.steps / (sum(step_ms) * 1e-3) / 1e9
        clk = clocks.summary()

        # ---- C4 mode: the same shard streamed through a pool 1/7 its size ----
        streaming = None
        if not args.skip_streaming:
            eng.close()
            del eng
            try:
                streaming = measure_streaming(lz, built, plan, payload, tmp, dev, barrier)
                log(f"[bench] rank {rank}: streaming through a 16 GiB pool: {streaming['gbps']} GB/s")
            except Exception as e:  # optional phase: keep the headline number
                streaming = {"error": f"{type(e).__name__}: {e}"}
            eng = lz.Engine(cfg, built.topo, built.rank)

        # ---- per-iteration stall under synthetic fwd/bwd (device-side fence) ----
        stall = None
        if not args.skip_train:
            try:
                stall = train_loop(lz, torch, eng, plan, built, payload, per_gpu, barrier)
            except Exception as e:
                stall = {"error": f"{type(e).__name__}: {e}"}

        # ---- e2e: public API, files durable on local disk ----
        e2e = None
        if not args.skip_e2e:
            eng.close()
            del eng
            try:
                e2e = e2e_persisted(lz, torch, dev, tmp, args, world, rank)
                # whole-job figure: bytes of all ranks over the slowest rank's time
                t_max = max_over_ranks(e2e.pop("seconds"))
                e2e["per_rank_gbps"] = e2e["value"]
                e2e["value"] = round(sum_over_ranks(float(e2e["d2h_bytes_per_step"] * e2e["steps"])) / t_max / 1e9, 3)
                e2e["d2h_bytes_per_step"] = int(sum_over_ranks(float(e2e["d2h_bytes_per_step"])))
            except Exception as e:
                e2e = {"error": f"{type(e).__name__}: {e}"}

        if rank == 0:
            kernel_gbps = variants["gather_kernel"]
            line = {
                "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(statistics.mean(step_ms), 3),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
                "data": "synthetic (splitmix64 generated in HBM)",
                "config": {"workload": f"c2-llama7b shard per GPU (configs[1]; {layers} layers, 4+12 B/param)",
                           "payload_bytes_per_gpu": payload, "tensors": len(w.leaves),
                           "variant": best, "large_leaf_threshold": 1 << 20, "chunk_quantum": 64 << 20,
                           "flush_tier": "host-memory (discard) for the timed steps; storage flush in e2e",
                           "l2": "inputs (>100 GB) exceed L2 (126 MB)", "parallelism": f"dp{world} weak"},
                "per_gpu_gbps": round(per_gpu, 3),
                "device_ms_per_step": round(statistics.mean(dev_ms), 3),
                "device_gbps": round(payload / (statistics.mean(dev_ms) * 1e-3) / 1e9, 3),
                "capture_host_ms": round(statistics.mean(cap_ms), 3),
                "variants_gbps": variants,
                "roofline": {"bound": "pcie-host-link", "achieved": round(per_gpu, 3), "peak": PCIE_GEN5_X16_GBPS,
                             "unit": "GB/s", "frac": round(per_gpu / PCIE_GEN5_X16_GBPS, 4),
                             "traffic": None,  # copy-engine DMAs: not visible to ncu kernel metrics
                             "peak_measured_dma": link["dma_gbps"],
                             "frac_of_measured_dma": round(per_gpu / link["dma_gbps"], 4),
                             "kernel": {"name": "lzk_gather_kernel", "achieved": kernel_gbps,
                                        "frac": round(kernel_gbps / PCIE_GEN5_X16_GBPS, 4),
                                        "peak_measured_sm_store": link["sm_store_gbps"],
                                        "frac_of_measured_sm_store": round(kernel_gbps / link["sm_store_gbps"], 4),
                                        # one `ncu --set full` capture of a 62.92 MB launch
                                        # (profiles/r01_gather_kernel_ncu.md, v3): DRAM read +
                                        # write per launch vs the algorithmic bytes
                                        "traffic": 62.9248e6 + 0.3566e6, "algorithmic_bytes_per_launch": 62.92e6,
                                        "ncu_profile": "profiles/r01_gather_kernel_ncu.md"},
                             "link_probe": link["how"],
                             "algorithmic_bytes_per_step": payload},
                "stall": stall,
                "streaming": streaming,
                "e2e": e2e,
                "cpu_baseline": None if cpu_base is None else {
                    "value": round(cpu_base["snapshot_gbps"], 4), "unit": "GB/s", "cores": 2, "kind": "reference",
                    "sample": cpu_base["sample"], "persisted_gbps": round(cpu_base["persisted_gbps"], 4),
                    "host": cpu_info()},
                "clocks": clk,
                "gpu_launches": int(launches),
                "copy_engine_dmas": int(stats1["ce_copies"] - stats0["ce_copies"]),
            }
            print(json.dumps(line), flush=True)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def measure_streaming(lz, built, plan, payload, tmp, dev, barrier, pool=16 << 30, segment=1 << 30):
    """C4 mode (SURVEY.md §7 hard part 3): the whole shard streams through a
    pinned pool 1/7 its size in 1 GiB segments reserved with backpressure."""
    scfg = lz.EngineConfig(checkpoint_root=os.path.join(tmp, "ckpt_s"), host_buffer_bytes=pool,
                           large_leaf_threshold=1 << 20, fsync_on_finalize=False, flush_discard=True,
                           hugepages=True, device=dev, stream_segment_bytes=segment)
    seng = lz.Engine(scfg, built.topo, built.rank)
    try:
        sms = []
        for s in range(3):
            barrier()
            h0 = time.perf_counter()
            t = seng.capture(plan, built.tree, 300 + s)
            seng.update_barrier(t)
            dt = time.perf_counter() - h0
            seng.wait_persisted(t)
            if s:
                sms.append(dt)
    finally:
        seng.close()
    return {"pool_bytes": pool, "segment_bytes": segment, "gbps": round(payload * len(sms) / sum(sms) / 1e9, 3),
            "note": "C4 mode: shard (%.1f GB) > pool; per-segment reservation with backpressure, host-memory tier"
                    % (payload / 1e9)}


def measure_link_ceiling(lz, dev, nbytes=8 << 30, chunk=256 << 20):
    """Raw ceilings of this box's host link, in this process, with the pool's
    memory kind (THP-registered pinned): back-to-back copy-engine DMAs of
    `chunk` bytes, and plain SM 16-byte stores via the gather kernel over
    large contiguous descriptors. Best of 3 (CUDA events)."""
    import ctypes as C
    from paper_2406_10707_b200 import _native as N
    d = lz.dev

    def ck(rc):
        if rc != 0:
            raise RuntimeError(d.lzk_last_error().decode())

    src, host, s = C.c_void_p(), C.c_void_p(), C.c_void_p()
    ck(d.lzk_dev_alloc(dev, nbytes, C.byref(src)))
    ck(d.lzk_dev_memset(dev, src, 0x5A, nbytes))
    ck(d.lzk_host_alloc(nbytes, 1 | 2, C.byref(host)))
    ck(d.lzk_stream_create(dev, 0, C.byref(s)))
    e0, e1 = C.c_void_p(), C.c_void_p()
    ck(d.lzk_event_create(dev, 0, C.byref(e0)))
    ck(d.lzk_event_create(dev, 0, C.byref(e1)))
    n = nbytes // chunk
    descs = (N.CopyDescC * n)(*[N.CopyDescC(src.value + i * chunk, host.value + i * chunk, chunk) for i in range(n)])
    out = {}
    try:
        for name, fn in (("dma", lambda: d.lzk_ce_copy_d2h(s, descs, n)),
                         ("sm_store", lambda: d.lzk_gather_d2h(s, descs, n, 16))):
            best = 0.0
            for _ in range(4):
                ck(d.lzk_event_record(e0, s))
                ck(fn())
                ck(d.lzk_event_record(e1, s))
                ck(d.lzk_event_sync(e1))
                ms = C.c_float()
                ck(d.lzk_event_elapsed_ms(e0, e1, C.byref(ms)))
                best = max(best, nbytes / (ms.value * 1e-3) / 1e9)
            out[name + "_gbps"] = round(best, 3)
    finally:
        d.lzk_event_destroy(e0)
        d.lzk_event_destroy(e1)
        d.lzk_stream_destroy(s)
        d.lzk_host_free(host)
        d.lzk_dev_free(dev, src)
    out["how"] = (f"{nbytes >> 30} GiB device -> THP-pinned host, {chunk >> 20} MiB copy-engine DMAs / "
                  "lzk_gather_kernel 16 CTAs, best of 4")
    return out


def train_loop(lz, torch, eng, plan, built, payload, gbps, barrier):
    """Checkpoint every iteration under a synthetic bf16 fwd/bwd sized so that
    t_fb >= payload / snapshot rate. Iteration = capture ->
    fwd/bwd GEMMs -> lazy fence (device-side, update_barrier_on_stream) ->
    optimizer step on a registered tensor. Stall = iteration time with
    checkpointing minus without."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
    b = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
    c = torch.empty(n, n, dtype=torch.bfloat16, device="cuda")
    comp = torch.cuda.Stream()
    with torch.cuda.stream(comp):
        for _ in range(10):
            torch.matmul(a, b, out=c)
    comp.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    with torch.cuda.stream(comp):
        for _ in range(50):
            torch.matmul(a, b, out=c)
    e1.record(comp)
    e1.synchronize()
    per_mm = e0.elapsed_time(e1) / 50
    t_snap_ms = payload / (gbps * 1e9) * 1e3
    n_mm = max(1, int(1.1 * t_snap_ms / per_mm))
    opt = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")  # the "optimizer state" we mutate
    opt_region = lz.DeviceRegion.wrap(opt)

    def iteration(step, ckpt: bool, device_fence: bool):
        h0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        t = eng.capture(plan, built.tree, step) if ckpt else None
        h1 = time.perf_counter()
        with torch.cuda.stream(comp):
            for _ in range(n_mm):
                torch.matmul(a, b, out=c)  # forward + backward stand-in
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if ckpt:
            if device_fence:
                f0.record(comp)  # compute stream reaches the fence
                eng.update_barrier_on_stream(t, comp.cuda_stream)
                f1.record(comp)  # ... and passes it
            else:
                comp.synchronize()
                eng.update_barrier(t)
        h2 = time.perf_counter()
        with torch.cuda.stream(comp):
            opt.add_(1.0)  # optimizer step: mutates state after the fence
        opt_region.bump_version()
        e1.record(comp)
        e1.synchronize()
        h3 = time.perf_counter()
        if ckpt:
            eng.wait_persisted(t)
        fence_ms = f0.elapsed_time(f1) if ckpt and device_fence else 0.0
        return e0.elapsed_time(e1), (h1 - h0) * 1e3, (h2 - h1) * 1e3, (h3 - h0) * 1e3, fence_ms

    barrier()
    for s in range(2):
        iteration(500 + s, False, True)
    base = [iteration(510 + s, False, True)[3] for s in range(4)]
    iteration(520, True, True)
    dev_fence = [iteration(530 + s, True, True) for s in range(4)]
    iteration(540, True, False)
    host_fence = [iteration(550 + s, True, False) for s in range(2)]
    base_ms = statistics.mean(base)
    it_ms = statistics.mean(x[3] for x in dev_fence)
    it_host_ms = statistics.mean(x[3] for x in host_fence)
    return {"t_fwd_bwd_ms": round(n_mm * per_mm, 2), "iter_no_ckpt_ms": round(base_ms, 2),
            "iter_ckpt_ms": round(it_ms, 2), "stall_ms": round(it_ms - base_ms, 2),
            "capture_host_ms": round(statistics.mean(x[1] for x in dev_fence), 3),
            "fence_wait_ms": round(statistics.mean(x[4] for x in dev_fence), 3),
            "stall_def_ms": round(statistics.mean(x[1] + x[4] for x in dev_fence), 3),
            "iter_overhead": round((it_ms - base_ms) / base_ms, 4),
            "host_fence": {"iter_ckpt_ms": round(it_host_ms, 2), "stall_ms": round(it_host_ms - base_ms, 2),
                           "iter_overhead": round((it_host_ms - base_ms) / base_ms, 4)},
            "fence": "update_barrier_on_stream (device-side)", "variant": "hybrid (engine default)",
            "gemm": "bf16 8192^3 torch.matmul x%d" % n_mm}


def e2e_persisted(lz, torch, dev, tmp, args, world=1, rank=0):
    """Public API end to end with durable files: capture -> update_barrier ->
    wait_persisted (pwrite + per-entry FNV + header last + fsync) on a
    bounded C2 slice that fits the box's local disk: a dp=N plan where each
    rank owns a 2-decoder-layer shard at N<=2, 1 at N>2 (weak scaling), every
    rank writing its shards under ONE shared root. The last step is committed
    by the two-phase commit (N>1: commit.distributed_commit over
    torch.distributed) and restored."""
    from paper_2406_10707_b200.workloads import llama7b_shard
    per_rank = 2 if world <= 2 else 1
    w = llama7b_shard(layers=per_rank, vocab=8000, dp=world, rank=rank, name=f"c2-slice-{per_rank}l-dp{world}")
    spec = w.write_spec(os.path.join(tmp, "e2e.spec"))
    built = lz.build_workload(spec, dev)
    root = os.path.join(ROOT, f"lzk_e2e_{os.environ.get('MASTER_PORT', 'solo')}") if world > 1 \
        else os.path.join(tmp, "e2e_ckpt")

    def sync():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

    cfg = lz.EngineConfig(checkpoint_root=root, host_buffer_bytes=int(built.bytes * 1.01) + (64 << 20),
                          fsync_on_finalize=True, device=dev)
    eng = lz.Engine(cfg, built.topo, built.rank)
    plan = lz.plan_checkpoint(built.topo, built.model, built.step)
    times = []
    steps = 3
    r0, r1, r2 = built.rank.dp, built.rank.pp, built.rank.tp
    for s in range(steps):
        sync()
        h0 = time.perf_counter()
        t = eng.capture(plan, built.tree, 700 + s)
        eng.update_barrier(t)
        eng.wait_persisted(t)
        dt = time.perf_counter() - h0
        if s >= 1:
            times.append(dt)
        payload = t.payload_bytes()
        if s + 1 < steps:  # each rank removes only its own directory
            shutil.rmtree(os.path.join(root, f"step-{700 + s}", f"rank-{r0}-{r1}-{r2}"), ignore_errors=True)
    # two-phase commit of the last step: files validated and digested on the GPU
    mpath = os.path.join(root, "manifest.json")
    sync()
    h0 = time.perf_counter()
    if world > 1:
        from paper_2406_10707_b200.commit import distributed_commit
        rec = distributed_commit(eng, built.model, t, mpath)
        committed, why = rec.committed, rec.reason
    else:
        committed, why = eng.commit(built.model, t, lz.ManifestStore(mpath))
    commit_s = time.perf_counter() - h0
    if not committed:
        raise RuntimeError("commit failed: " + why)
    m = lz.ManifestStore(mpath)
    # restore the last step (files just written: page cache may be warm)
    h0 = time.perf_counter()
    back = eng.restore(m, 700 + steps - 1)
    restore_s = time.perf_counter() - h0
    ok = back.leaf_count() == built.tree.leaf_count()
    probe = [l for l in built.tree.flatten() if l.is_region][:3]
    ok = ok and all(back.region_at(l.path).clone_bytes() == built.tree.region_at(l.path).clone_bytes() for l in probe)
    del back
    eng.close()
    sync()
    if world > 1 and rank == 0:
        shutil.rmtree(root, ignore_errors=True)
    v = payload * len(times) / sum(times) / 1e9
    return {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": payload,
            "seconds": sum(times),
            "workload": f"{w.name} ({payload} B payload per rank, {len(w.leaves)} tensors)",
            "path": "capture -> update_barrier -> wait_persisted, fsync, local disk", "steps": len(times),
            "commit_gbps": round(payload / commit_s / 1e9, 3),
            "commit_seconds": round(commit_s, 3),
            "commit_reads": "from the disk with O_DIRECT (durable writes bypass the page cache, so fresh files are cold)",
            "commit_path": "2PC (N>1: votes over torch.distributed): each file read once, entry checksums + whole-file digest on the GPU",
            "restore_gbps": round(payload / restore_s / 1e9, 3), "restore_spot_check": ok,
            "restore_reads": "per 512 MiB window: the page cache when mincore shows it resident, else O_DIRECT",
            "restore_path": "parallel pread into pinned windows -> one DMA per window -> device FNV check -> D2D to regions"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=32, help="LLaMA-7B layers per shard (32 = full C2)")
    ap.add_argument("--skip-train", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu-baseline", action="store_true")
    ap.add_argument("--skip-streaming", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("[bench] warmup raised to 3 (timing rules)")
        args.warmup = 3
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout carries only our JSON
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        # NCCL prints its version line on fd 1 at the default WARN level,
        # whatever NCCL_DEBUG_FILE says: keep fd 1 on stderr while the
        # communicator is created eagerly (device_id), so stdout carries only
        # the JSON line.
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
            dist.barrier()
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
    try:
        main_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
