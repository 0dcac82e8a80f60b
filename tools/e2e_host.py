"""Host cost of the e2e loop: wall time of MicroBatchLoop.submit() calls vs the device time per
step (bench's TP1 workload): python tools/e2e_host.py"""
import sys, time, torch
sys.path.insert(0, ".")
import bench
from paper_2603_02188_b200.config import trained_config
from paper_2603_02188_b200.host_loop import MicroBatchLoop

dev = torch.device("cuda", 0)
cfg = trained_config("mlra4")
engs = [bench.make_engine(cfg, None, 16, 32768, s, dev)[0] for s in (1, 2)]
loop = MicroBatchLoop(engs, graphs=len(sys.argv) > 1 and sys.argv[1] == "graphs")
for k in range(2):
    for t in loop.host_inputs(k):
        t.normal_()
for _ in range(10):
    loop.submit(_ % 2)
torch.cuda.synchronize()
n = 40
loop.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
for i in range(n):
    loop.submit(i % 2)
t1 = time.perf_counter()
loop.join()
e1.record()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"submit host time {(t1 - t0) / n * 1e6:.1f} us/step, wall {(t2 - t0) / n * 1e6:.1f} us/step, "
      f"device {e0.elapsed_time(e1) / n * 1e3:.1f} us/step", flush=True)
