import sys,json
for l in sys.stdin:
  try: d=json.loads(l); print(d["lens"], d["n"], round(d["us"],1), round(d["tflops"]), round(d["frac_attainable"],3))
  except Exception: print(l.strip()[:300])
