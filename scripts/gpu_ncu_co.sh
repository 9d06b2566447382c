#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cat > /tmp/co_bench.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2605_19385_b200 as lbx
n, H, W = 32, 1024, 1024
x = (torch.randn(n, H, W, 128, device='cuda') * 0.5).half()
ss = torch.stack([torch.rand(n, 128, device='cuda') + 0.5, torch.randn(n, 128, device='cuda') * 0.5], -1).contiguous()
w = torch.randn(3, 3, 3, 128, device='cuda') * 0.03
b = torch.zeros(3, device='cuda')
rgb = torch.empty(n, H, W, 3, dtype=torch.uint8, device='cuda')
impl = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for _ in range(2):
    lbx.op_conv_out(x.data_ptr(), ss.data_ptr(), w.data_ptr(), b.data_ptr(), rgb.data_ptr(), n, H, W, impl=impl)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    lbx.op_conv_out(x.data_ptr(), ss.data_ptr(), w.data_ptr(), b.data_ptr(), rgb.data_ptr(), n, H, W, impl=impl)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"conv_out impl {impl}: {ms:.3f} ms  {n*H*W*259/ms/1e6:.0f} GB/s")
PY
python /tmp/co_bench.py 2; python /tmp/co_bench.py 0; python /tmp/co_bench.py 1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:conv_out_tc -s 1 -c 1 -o gpurun_out/co_tc python /tmp/co_bench.py 2 > gpurun_out/ncu_co.log 2>&1
tail -1 gpurun_out/ncu_co.log
