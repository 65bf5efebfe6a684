"""Cost of each NVML query used by bench.py's clock sampler (host latency), and
its effect on a stream of short GPU kernels."""
import time, threading
import torch, pynvml as nv
nv.nvmlInit(); h = nv.nvmlDeviceGetHandleByIndex(0)
calls = {"clock": lambda: nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
         "maxclock": lambda: nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM),
         "power": lambda: nv.nvmlDeviceGetPowerUsage(h),
         "reasons": lambda: nv.nvmlDeviceGetCurrentClocksEventReasons(h)}
for k, f in calls.items():
    f(); t = time.perf_counter(); [f() for _ in range(20)]; print(k, "ms per call", (time.perf_counter() - t) / 20 * 1e3)
x = torch.zeros(1 << 16, device="cuda")
def work(n=3000):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(n):
        x.add_(1.0); torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3
print("kernels+sync alone ms", work())
for k, f in calls.items():
    stop = threading.Event()
    def poll():
        while not stop.is_set():
            f(); time.sleep(0.01)
    th = threading.Thread(target=poll); th.start()
    print("with", k, "polled every 10 ms: ms", work()); stop.set(); th.join()
