"""Run a script with LOCAL_RANK forced to 0 (all ranks on one visible GPU) — for
exercising multi-rank control flow on a single-GPU box only."""
import os
import runpy
import sys

os.environ["LOCAL_RANK"] = "0"
script = sys.argv[1]
sys.argv = sys.argv[1:]
runpy.run_path(script, run_name="__main__")
