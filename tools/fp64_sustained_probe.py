import sys, time, subprocess
sys.path.insert(0, '.')
from paper_2005_02516_b200 import capi
vals = []
t0 = time.time()
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap", "--format=csv,noheader", "-lms", "200"], stdout=subprocess.PIPE, text=True)
while time.time() - t0 < 6:
    vals.append(capi.probe_fp64_peak(0, 20))
p.terminate()
out = p.stdout.read().splitlines()
print("n", len(vals), "first", [round(v, 2) for v in vals[:5]], "last", [round(v, 2) for v in vals[-5:]])
print(out[:3], out[-6:])
