import os, sys
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tools"))
import kernel_bench as kb
for lens, n in (([2048]*8, 24), ([1920]*8, 24), ([1856]*8, 24), ([1792]*8, 24), ([1856]*16, 40), ([2048]*16, 40), ([1856]*24, 40), ([2048]*8, 40)):
    d = kb.prefill_point(lens, n, 128)
    print(len(lens), lens[0], n, round(d["us"],1), round(d["tflops"]), round(d["frac_tensor_peak"],3), flush=True)
