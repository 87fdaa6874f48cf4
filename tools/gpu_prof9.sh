mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rapid.py tests/test_gpu_naive.py -q -x -o faulthandler_timeout=300 > gpurun_out/r02_rapidtests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_rapidtests.log
tail -n 3 gpurun_out/r02_rapidtests.log
python -c "
import time, numpy as np
from paper_1703_01506_b200.normals import NormalStream
from paper_1703_01506_b200.rng import BASIS_INIT
buf=np.empty(1<<20); g=NormalStream(1703015065,(BASIS_INIT,)); t0=time.perf_counter()
for i in range(200): g.fill(buf)
print('basis normals alone on the box: %.3f s'%(time.perf_counter()-t0)); g.close()"
for v in "RMX_PDL=1" "RMX_PDL=1"; do
  echo "== $v"; env $v timeout 600 python tools/diag_rapid.py --config c5 2>&1 | grep -E "mark\]|run_rapid" | cut -c1-110
done
bash tools/gpu_final_prof.sh
