"""Which NVML PCIe counter gives the bytes a GPU really sent to the host?
Moves a known number of bytes device -> pinned host (copy engine, 256 MiB
DMAs) and compares with (a) nvmlDeviceGetPcieThroughput(TX) integrated,
read back to back and on a 20 ms tick, (b) GPM PCIE_TX_PER_SEC between two
GPM samples, (c) the NVML_FI_DEV_PCIE_COUNT_TX_BYTES field counter.
    python tools/pcie_counter_probe.py"""
import threading
import time

import pynvml as N
import torch

N.nvmlInit()
dev = 0
p = torch.cuda.get_device_properties(dev)
h = N.nvmlDeviceGetHandleByPciBusId(f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0")
t0 = time.perf_counter()
for _ in range(20):
    N.nvmlDeviceGetPcieThroughput(h, N.NVML_PCIE_UTIL_TX_BYTES)
print(f"nvmlDeviceGetPcieThroughput call: {(time.perf_counter() - t0) / 20 * 1e3:.2f} ms")

src = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
dst = torch.empty(8 << 30, dtype=torch.uint8, pin_memory=True)
REPS = 8
moved = REPS * src.numel()


def transfer():
    for _ in range(REPS):
        for o in range(0, src.numel(), 256 << 20):
            dst[o:o + (256 << 20)].copy_(src[o:o + (256 << 20)], non_blocking=True)
    torch.cuda.synchronize()


class Sampler:
    def __init__(self, tick):
        self.tick, self.bytes, self.stop = tick, 0.0, threading.Event()

    def run(self):
        last = time.perf_counter()
        nxt = last
        while not self.stop.is_set():
            if self.tick:
                nxt += 0.02
                time.sleep(max(0.0, nxt - time.perf_counter()))
            v = N.nvmlDeviceGetPcieThroughput(h, N.NVML_PCIE_UTIL_TX_BYTES)
            now = time.perf_counter()
            self.bytes += v * 1e3 * (now - last)
            last = now


def field():
    v = N.nvmlDeviceGetFieldValues(h, [N.NVML_FI_DEV_PCIE_COUNT_TX_BYTES])[0]
    return v.value.ullVal if v.nvmlReturn == 0 else None


transfer()  # warm
for tick in (False, True):
    s = Sampler(tick)
    th = threading.Thread(target=s.run)
    f0 = field()
    try:
        g1 = N.nvmlGpmSampleAlloc()
        g2 = N.nvmlGpmSampleAlloc()
        N.nvmlGpmSampleGet(h, g1)
        gpm = True
    except Exception as e:
        print("GPM unavailable:", e)
        gpm = False
    th.start()
    a = time.perf_counter()
    transfer()
    b = time.perf_counter()
    s.stop.set()
    th.join()
    f1 = field()
    line = f"moved {moved / 1e9:.2f} GB in {b - a:.3f} s; throughput sampler ({'tick' if tick else 'back-to-back'}) " \
           f"{s.bytes / 1e9:.2f} GB"
    if f0 is not None and f1 is not None:
        line += f"; field counter delta {f1 - f0} ({(f1 - f0) / moved:.4g} per byte)"
    if gpm:
        N.nvmlGpmSampleGet(h, g2)
        mg = N.c_nvmlGpmMetricsGet_t()
        mg.version = N.NVML_GPM_METRICS_GET_VERSION
        mg.numMetrics = 1
        mg.sample1, mg.sample2 = g1, g2
        mg.metrics[0].metricId = N.NVML_GPM_METRIC_PCIE_TX_PER_SEC
        N.nvmlGpmMetricsGet(mg)
        rate = mg.metrics[0].value
        line += f"; GPM PCIE_TX_PER_SEC {rate:.4g} (x elapsed {b - a:.3f} s = {rate * (b - a) / 1e9:.2f} GB if B/s, MiB/s -> {rate * (b - a) * 1048576 / 1e9:.2f} GB)"
    print(line, flush=True)
