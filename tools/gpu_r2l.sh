mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2l_gputest.log 2>&1; tail -5 gpurun_out/r2l_gputest.log
timeout 300 python -c "
import time; t=time.perf_counter()
from paper_2408_01654_b200 import synthetic
s,g,f=synthetic.make_config('cfg3'); print('cfg3 generation', time.perf_counter()-t, 's')
t=time.perf_counter(); s,g,f=synthetic.make_config('cfg4'); print('cfg4 generation', time.perf_counter()-t, 's')
"
