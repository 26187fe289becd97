"""One-off box probe: host facts + torch read/copy bandwidth (library context, not product)."""
import os, subprocess, json, torch
out = {}
out["nproc"] = os.cpu_count(); out["affinity"] = len(os.sched_getaffinity(0))
out["mem"] = subprocess.run(["free", "-g"], capture_output=True, text=True).stdout
out["cpu"] = [l for l in open("/proc/cpuinfo") if l.startswith("model name")][:1]
out["smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,memory.total,clocks.sm,clocks.max.sm", "--format=csv"], capture_output=True, text=True).stdout
p = torch.cuda.get_device_properties(0)
out["sms"] = p.multi_processor_count; out["l2"] = p.L2_cache_size
def t(fn, reps=20):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(reps):
        s.record(); fn(); e.record(); e.synchronize(); best = min(best, s.elapsed_time(e))
    return best
for dt, n in [(torch.float32, 1 << 30), (torch.float64, 1 << 29), (torch.int32, 1 << 30)]:
    x = torch.ones(n, dtype=dt, device="cuda")
    ms = t(lambda: x.sum())
    out[f"torch_sum_{dt}"] = dict(ms=ms, gbs=x.numel() * x.element_size() / ms / 1e6)
    y = torch.empty_like(x)
    ms = t(lambda: y.copy_(x))
    out[f"copy_{dt}"] = dict(ms=ms, gbs=2 * x.numel() * x.element_size() / ms / 1e6)
    del x, y
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
