set -x
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests -m gpu -x -q -k "netscale or repr256" 2>&1 | tail -3
CRL_LSE_TWO_CALL=1 timeout 200 python bench.py --workload netscale --steps 3 --warmup 3 --profile-steps 1 2>&1 | tail -3 | cut -c1-300
timeout 200 python bench.py --workload netscale --steps 3 --warmup 3 --profile-steps 0 2>&1 | tail -3 | cut -c1-300
timeout 100 python - <<'P'
import torch, crl_synth, time
from paper_2408_11052_b200 import CrlConfig, CrlContext
cfg = crl_synth.preset("netscale", precision="bf16")
ctx = CrlContext(CrlConfig.from_preset(cfg), params=torch.from_numpy(crl_synth.init_critic_params(cfg, 1)))
import numpy as np
s,a,g = [torch.from_numpy(x).cuda() for x in crl_synth.random_batch(cfg, cfg["batch"], seed=3)]
loss = torch.zeros(4, device="cuda")
for i in range(5):
    t=time.time(); ctx.critic_step(s,a,g,loss); torch.cuda.synchronize(); print("step", i, time.time()-t, loss.tolist(), ctx.status(), flush=True)
P
