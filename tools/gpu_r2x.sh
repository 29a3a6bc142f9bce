mkdir -p gpurun_out
DPV_BUILD_PROFILE=1 timeout 300 python -c "
import torch, time, numpy as np
from paper_2408_01654_b200 import synthetic, ba, _lib
s,g,f=synthetic.make_config('cfg2')
soa0={k: np.array(v) for k,v in g.soa().items()}
for r in range(4):
    g._q.view[:]=soa0['frame_q']; g._t.view[:]=soa0['frame_t']; g._depth.view[:]=soa0['patch_depth']; g._pose_ver+=1; g._patch_ver+=1; g.device(); torch.cuda.synchronize()
    t=time.perf_counter(); p=ba.BAProblem(g,f); p._ensure(); torch.cuda.synchronize(); t1=time.perf_counter()
    rep=ba.solve(p,2,1e-12); torch.cuda.synchronize(); t2=time.perf_counter()
    print('build ms %.3f solve ms %.3f iters %s' % ((t1-t)*1e3, (t2-t1)*1e3, [round(x*1e3,3) for x in rep.iteration_times]))
    del p
" 2>&1 | tail -22
