"""Times each NVML query the bench's clock sampler makes while the GPU is busy
(diagnoses sampler calls that stall for tens of ms)."""
import threading
import time

import pynvml as nv
import torch

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
calls = {
    "clock_sm": lambda: nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
    "max_clock_sm": lambda: nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM),
    "reasons": lambda: nv.nvmlDeviceGetCurrentClocksEventReasons(h),
}
stop = threading.Event()


def busy():
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    while not stop.is_set():
        for _ in range(20):
            a = (a @ a).clamp_(-1, 1)
        torch.cuda.synchronize()


for phase in ("idle", "busy"):
    t = None
    if phase == "busy":
        t = threading.Thread(target=busy)
        t.start()
        time.sleep(0.5)
    for name, fn in calls.items():
        d = []
        for _ in range(40):
            t0 = time.perf_counter()
            fn()
            d.append((time.perf_counter() - t0) * 1e3)
            time.sleep(0.01)
        d.sort()
        print(f"{phase:5s} {name:13s} median {d[20]:.2f} ms  p90 {d[36]:.2f}  max {d[-1]:.2f}", flush=True)
    if t:
        stop.set()
        t.join()
