"""Decode work-split knob sweep over A/B builds (tools/ab.sh): each variant runs in
its own process (DS_PKG_ROOT) on the same decode points, two interleaved passes.
python tools/dec_knob_sweep.py ab/dp10c8 ab/dp20c4 ... > gpurun_out/dec_knobs.jsonl"""
import json
import os
import subprocess
import sys

POINTS = [(int(b), int(c)) for b, c in (x.split('x') for x in os.environ.get('DS_POINTS', '32x544,64x544,128x544,256x544,64x2048,16x2048').split(','))]
CHILD = r"""
import json, sys
sys.argv = ['kb']
import kernel_bench as kb
for B, ctx in %r:
    r = kb.decode_point(B, ctx, 40, 128, layers=8 if B * ctx <= 128 * 2048 else 4, reps=10)
    r['variant'] = %r
    print(json.dumps(r), flush=True)
"""

here = os.path.dirname(os.path.abspath(__file__))
for rep in range(2):
    for v in sys.argv[1:]:
        env = dict(os.environ, DS_PKG_ROOT=v, PYTHONPATH=here)
        out = subprocess.run([sys.executable, "-c", CHILD % (POINTS, os.path.basename(v.rstrip("/")))], env=env,
                             capture_output=True, text=True, timeout=600)
        for line in out.stdout.splitlines():
            if line.startswith("{"):
                d = json.loads(line)
                d["pass"] = rep
                print(json.dumps(d), flush=True)
        if out.returncode:
            print(json.dumps({"variant": v, "error": out.stderr[-500:]}), flush=True)
