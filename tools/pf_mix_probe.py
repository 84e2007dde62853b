"""Prefill on the BASELINE length mixes (kernel only): python tools/pf_mix_probe.py
Prints us, TFLOP/s and fraction of the attainable roofline per mix; honours
DS_PKG_ROOT and the kernel's env knobs (e.g. DS_PREFILL_PERSISTENT)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import kernel_bench as kb  # noqa: E402
import synthetic as syn  # noqa: E402

mixes = {
    "c3 chatbot 64 req, 40 heads": ([int(x) for x in syn.lengths_chatbot(0, 64)[0]], 40),
    "c4 code 32 req, 36 heads": ([int(x) for x in syn.lengths_code(0, 164)[0][:32]], 36),
    "c5 summarization 8 req, 24 heads": ([int(x) for x in syn.lengths_summarization(0, 8)[0]], 24),
}
for name, (lens, n) in mixes.items():
    d = kb.prefill_point(lens, n, 128)
    print(f"{name:36s} tokens {sum(lens):6d} max {max(lens):5d}  {d['us']:8.1f} us  {d['tflops']:6.0f} TF/s  "
          f"attainable {d['frac_attainable']:.3f}", flush=True)
