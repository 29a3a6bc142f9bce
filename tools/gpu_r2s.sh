mkdir -p gpurun_out
DPV_BUILD_PROFILE=1 timeout 300 python -c "
import torch, time
from paper_2408_01654_b200 import synthetic, ba
s,g,f=synthetic.make_config('cfg3')
for r in range(3):
    torch.cuda.synchronize(); t=time.perf_counter()
    p=ba.BAProblem(g,f); p._ensure(); torch.cuda.synchronize()
    print('build ms', (time.perf_counter()-t)*1e3)
    rep = ba.solve(p, 8, 1e-9); print('solve times', rep.iteration_times if hasattr(rep,'iteration_times') else None)
" > gpurun_out/r2s_build.txt 2>&1; tail -60 gpurun_out/r2s_build.txt
