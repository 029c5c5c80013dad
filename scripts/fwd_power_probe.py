"""Forward-only timing at one shape with nvidia-smi clock / power samples
during the loop (is a kernel change faster in cycles but power-clocked?)."""
import os, subprocess, sys, threading, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device, _lib
_lib.load()
H, N, d, B, k = (int(x) for x in os.environ.get("CFG", "32,65536,64,128,8").split(","))
g = torch.Generator(device="cuda").manual_seed(0)
q, kk, v = (torch.randn(H, N, d, generator=g, device="cuda").bfloat16() for _ in range(3))
cent, _ = _device.centroids(kk, B)
plan = _device.route(q, cent, B, k, mode=1)
for _ in range(3): _device.fwd(q, kk, v, plan, d ** -0.5)
torch.cuda.synchronize()
samples, stop = [], threading.Event()
def sampler():
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                            "--format=csv,noheader,nounits", "-i", "0"], capture_output=True, text=True)
        samples.append(r.stdout.strip()); time.sleep(0.05)
th = threading.Thread(target=sampler); th.start()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = int(os.environ.get("REPS", 200))
a.record()
for _ in range(reps): _device.fwd(q, kk, v, plan, d ** -0.5)
b.record(); torch.cuda.synchronize(); stop.set(); th.join()
print(f"{os.environ.get('MOBA_LIB', 'cur')}: fwd {a.elapsed_time(b) / reps:.3f} ms/iter; smi samples: {samples[len(samples)//4: len(samples)//4 + 6]}")
