"""Diagnostics: per-step cost of the partitioned (dist) path at world size 1."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
backend = os.environ.get("BK", "gloo")
torch.cuda.set_device(0)
dist.init_process_group(backend, rank=0, world_size=1)
from paper_2406_17284_b200 import ltl  # noqa: E402
from paper_2406_17284_b200.dist import PartitionedTorus  # noqa: E402

if os.environ.get("SIDE_STREAM"):
    torch.cuda.set_stream(torch.cuda.Stream())
part = PartitionedTorus(16384, 16384, 0, 1, 0)
stream = torch.cuda.current_stream()
if os.environ.get("USE_STREAM"):
    part.use_stream(stream.cuda_stream)
if os.environ.get("SINGLE"):
    from paper_2406_17284_b200.ltl import DeviceTorus
    part.torus = DeviceTorus(rows=16384, cols=16384)
    part.ring = False
    part.exchange = lambda: None
    part.step = lambda rule: part.torus.run_async(rule, 1)
part.init_random(0.21, 1)
rule = ltl.parse_ltl_rule("R5,C2,M1,S34..58,B34..45,NM")
for _ in range(10):
    part.step(rule)
torch.cuda.synchronize()
dist.barrier()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
ev0.record(stream)
for _ in range(200):
    part.step(rule)
ev1.record(stream)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"backend={backend} ring={part.ring} host enqueue {1e6*(t1-t0)/200:.1f} us/step, "
      f"wall {1e6*(t2-t0)/200:.1f} us/step, events {1e3*ev0.elapsed_time(ev1)/200:.1f} us/step")
