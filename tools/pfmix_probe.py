import os, sys, json
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tools"))
import numpy as np
import kernel_bench as kb
rng = np.random.default_rng(0)
mix = [int(x) for x in rng.integers(1792, 1921, size=8)]
for lens, n in (([1856]*8, 24), ([1856]*8, 40), (mix, 40), (mix, 24), ([1856]*16, 24), ([1856]*32, 24), ([2048]*16, 40)):
    d = kb.prefill_point(lens, n, 128)
    print(len(lens), lens[0], n, round(d["us"],1), round(d["tflops"]), flush=True)
