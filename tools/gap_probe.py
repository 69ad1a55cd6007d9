"""GPU idle gap at a host-read scalar in the Krylov loop: SpMV with a fused dot -> host reads the
dot (stream sync) -> the next vector kernel.  Prints the time between the SpMV's completion and
the next launch reaching the GPU (CUDA events on both sides).  python tools/gap_probe.py"""
import sys, torch
sys.path.insert(0, '.')
from paper_2508_07193_b200 import Box, make_partition, make_transport, DistributedOperator
from paper_2508_07193_b200.instrument import NULL_TIMER
from paper_2508_07193_b200.krylov import _DeviceVectors
part = make_partition(Box(256, 256, 256), (8, 8, 8), 1)
op = DistributedOperator(part, 0.25, make_transport("cuda"))
x = torch.rand(3, 256, 256, 256, dtype=torch.float64, device="cuda")
v, w, s = torch.empty_like(x), torch.rand_like(x), torch.empty_like(x)
vec = _DeviceVectors(op, NULL_TIMER)
gaps = []
for it in range(23):
    e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    op._run(1, x, v, w)                 # v = A x, (v, w) -- the fused dot, no read yet
    e1.record()
    alpha = 1.0 / float(op._reduced(1)[0])   # stream sync + host read, as bicgstab does
    e2.record()
    vec.lincomb(1.0, w, -alpha, v, out=s)
    torch.cuda.synchronize()
    if it >= 3:
        gaps.append(e1.elapsed_time(e2) * 1000)
gaps.sort()
print("idle gap after a host-read dot (us): median %.1f min %.1f max %.1f" % (gaps[len(gaps) // 2], gaps[0], gaps[-1]))
