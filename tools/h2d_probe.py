import torch, time
torch.cuda.init()
for mb in (5, 50):
    h = torch.empty(mb*1024*1024, dtype=torch.uint8).pin_memory()
    d = torch.empty_like(h, device='cuda')
    s = torch.cuda.Stream()
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(20): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)/20
    print(f"{mb} MB: {ms:.3f} ms -> {mb*1.048576/ms:.1f} GB/s")
import subprocess
print(subprocess.run(['nvidia-smi','--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max','--format=csv'],capture_output=True,text=True).stdout)
