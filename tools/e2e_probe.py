"""Stage timings of the bench's e2e leg (streamed upload + OptDMD fit) at config 3."""
import json
import os
import sys
import time
import warnings

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2502_05339_b200 as fd
from paper_2502_05339_b200 import device as dv, synth, trace

p = synth.config_params(3, seed=3)
S = dv.alloc_tall(p.n, p.m, torch.float32, "row", zero=True)
tabs = [torch.as_tensor(np.ascontiguousarray(t), device="cuda") for t in p.sep_tables()]
dv.get_ops().synth3d(tabs, p.m, p.noise, synth.noise_key(p.seed), 0, p.n, S)
host = torch.empty((p.n, p.m), dtype=torch.float32, pin_memory=True)
host.copy_(S.view().cpu())
del S
torch.cuda.empty_cache()
for i in range(3):
    torch.cuda.synchronize()
    trace.enable()
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        d2 = fd.SnapshotMatrix(host, 0.1, stream=True)
        model = fd.optdmd(d2, 200, lm_config=fd.LMConfig(max_iters=10), svd_mode="randomized", seed=3,
                          oversample=10, power_iters=1)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = trace.summarize(trace.disable())
    print(json.dumps({"iter": i, "s": round(dt, 3), "mem_reserved_GB": round(torch.cuda.memory_reserved() / 1e9, 1),
                      "stages": {k: round(v, 1) for k, v in st.items() if v > 20}}))
    del d2, model
