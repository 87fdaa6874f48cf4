timeout 900 python -m pytest tests/test_gpu_rapid.py tests/test_gpu_configs.py -q -x 2>&1 | tail -2
for i in 1 2 3; do timeout 600 python tools/diag_rapid.py --config c5 2>&1 | grep -E "mark\] grouse|run_rapid" | cut -c1-110; done
python - <<'PY'
import numpy as np, torch, paper_1703_01506_b200 as rmx
from paper_1703_01506_b200.datagen import CONFIGS, make_data_torch, scaled
cfg=CONFIGS['c5']; c=scaled(cfg,(64,64,32),4000)
x=rmx.DataMatrix(make_data_torch(c, torch.device('cuda',0)).to(torch.float32).cpu().numpy(), c.n1, c.n2)
rc=rmx.RunConfig(permutations=4000, seed=c.plan_seed, engine='rapid', training_columns=c.training_columns, rank=c.rank, sample_rate=c.sample_rate, max_passes=3)
outs=[rmx.run_rapid(x, rc) for _ in range(3)]
print('bases identical:', all(np.array_equal(o[1].basis.matrix, outs[0][1].basis.matrix) for o in outs),
      'maxima identical:', all(np.array_equal(o[0].maxima, outs[0][0].maxima) for o in outs),
      'sigma', [o[1].residual_std for o in outs])
PY
