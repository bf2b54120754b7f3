import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import crl_synth
import test_gpu_parity as T
for chain in ["1", None]:
    if chain: os.environ["CRL_CHAIN"] = "1"
    else: os.environ.pop("CRL_CHAIN", None)
    for over in [dict(batch=300, energy="cos", activation="silu"), dict(batch=256, energy="cos", activation="relu"),
                 dict(batch=300, energy="l2", activation="relu"), dict(batch=256, energy="l2", activation="relu"),
                 dict(batch=300, energy="cos", activation="relu")]:
        cfg = crl_synth.preset("ant", precision="bf16", **over)
        try:
            T._critic_parity(cfg, check_adam=False, tol_loss=T.BF16_TOL, tol_grad=T.BF16_TOL)
            print("chain", chain, over, "OK")
        except AssertionError as e:
            print("chain", chain, over, "FAIL", str(e).split("\n")[0][:200])
