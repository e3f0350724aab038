"""Host topology vs the GPU: NVML's CPU affinity for GPU 0, and the pinned
PCIe bandwidth with the process bound to those cores vs unbound."""
import os
import subprocess
import sys

import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
ncpu = os.cpu_count()
words = (ncpu + 63) // 64
mask = pynvml.nvmlDeviceGetCpuAffinity(h, max(words, 1))
local = [c for c in range(ncpu) if (mask[c // 64] >> (c % 64)) & 1]
allowed = sorted(os.sched_getaffinity(0))
print("cpus", ncpu, "allowed", len(allowed), "nvml-local", len(local),
      "local&allowed", len(set(local) & set(allowed)), flush=True)
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
here = os.path.dirname(os.path.abspath(__file__))
print("unbound:", flush=True)
subprocess.run([sys.executable, os.path.join(here, "pcie_bw.py")])
loc = sorted(set(local) & set(allowed))
if loc:
    print("bound to the GPU's local cores:", flush=True)
    subprocess.run([sys.executable, "-c",
                    f"import os,runpy; os.sched_setaffinity(0, {loc}); "
                    f"runpy.run_path({os.path.join(here, 'pcie_bw.py')!r}, run_name='__main__')"])
