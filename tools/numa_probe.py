"""Host placement relative to the GPU: CPU affinity, the GPU's local CPU list and NUMA node, and the
end-to-end solve time with and without binding to the GPU-local CPUs.  python tools/numa_probe.py"""
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2209_04876_b200 as K  # noqa: E402


def gpu_local_cpus():
    bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
    out = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip().splitlines()[0]
    dom = out.lower()
    # nvidia-smi prints 00000000:xx:00.0; sysfs uses 0000:xx:00.0
    sys_id = dom[4:] if len(dom.split(":")[0]) == 8 else dom
    p = Path("/sys/bus/pci/devices") / sys_id
    cpus = (p / "local_cpulist").read_text().strip() if (p / "local_cpulist").exists() else "?"
    node = (p / "numa_node").read_text().strip() if (p / "numa_node").exists() else "?"
    return sys_id, cpus, node


def e2e(reps=14):
    n, d = 16384, 64
    facs_h = bench.make_inputs(n, d)
    cfg = K.RegressionConfig(**bench.PARAMS)
    b_host = torch.ones(n * n, dtype=torch.float64).pin_memory()
    facs_pin = [torch.from_numpy(a).pin_memory() for a in facs_h]
    ts = []
    for i in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = K.fast_kronecker_regression(facs_pin, b_host, cfg, with_loss=False)
        np.asarray(r.solution)
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts[6:])) * 1e3


print("affinity", sorted(os.sched_getaffinity(0))[:8], "... n =", len(os.sched_getaffinity(0)), "cpus", os.cpu_count())
print("gpu", gpu_local_cpus())
print("e2e ms (inherited affinity)", e2e())
