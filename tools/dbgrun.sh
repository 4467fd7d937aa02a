# time conv2 forward (tensor cores) for different M-tiles-per-CTA settings
for mt in 4 2 1; do
  echo "MT $mt: $(DP_TC_MT=$mt timeout 60 python -c "
import sys, torch; sys.path.insert(0,'.')
from paper_1412_4526_b200.engine import ops
N=64; x=torch.randn(N,16,278,278,device='cuda'); w=torch.randn(32,16,5,5,device='cuda')*.1; b=torch.randn(32,device='cuda')
y=torch.empty(N,32,270,270,device='cuda'); ws=torch.empty(ops.fast_workspace(16,32,5),dtype=torch.uint8,device='cuda')
f=lambda: ops.conv_forward_fast(x,w,b,y,5,2,0,ws)
f(); torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record(); [f() for _ in range(5)]; e1.record(); torch.cuda.synchronize(); print(round(e0.elapsed_time(e1)/5,3),'ms')
" 2>&1 | tail -1)"
done
