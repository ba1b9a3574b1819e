import sys, numpy as np
sys.path.insert(0, '/root/repo')
from oracle.oracle import Oracle, ModelCfg, synthetic_prompts
from paper_2405_01481_b200 import ppoexp as px
o = Oracle()
ctx = px.Context(0)
for cfg in [ModelCfg(258, 64, 2, 4, 128, 48), ModelCfg(1024, 64, 2, 4, 128, 48), ModelCfg(258, 64, 2, 2, 128, 48),
            ModelCfg(258, 128, 2, 4, 512, 128), ModelCfg(1024, 64, 2, 4, 128, 128), ModelCfg(1024, 128, 2, 4, 512, 48)]:
    w = o.init_params(cfg, 5).astype(np.float32).astype(np.float64)
    prompts = synthetic_prompts(3, 4, 8, True)
    pc = px.ModelConfig(cfg.V, cfg.d, cfg.L, cfg.H, cfg.f, cfg.S)
    m = px.DeviceModel(ctx, pc, w, px.F32)
    full = [np.concatenate([p, p]) for p in prompts]
    got = px.sequence_logprobs(m, full)
    exp = o.sequence_logprobs(cfg, w, full)
    d1 = max(np.abs(a - b).max() for a, b in zip(got, exp))
    eng = px.Engine(m)
    for graphs in (True,):
        r = eng.generate_batch([px.GenTask(p, 10) for p in prompts])
        t, l = o.generate(cfg, w, prompts, 10)
        ok = all(np.array_equal(a.tokens, b) for a, b in zip(r, t))
    print(cfg, "slp maxdiff", d1, "gen ok", ok, [len(a.tokens) for a in r], [len(b) for b in t], flush=True)
