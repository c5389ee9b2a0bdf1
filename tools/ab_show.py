import json, sys
v, path = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(path).readline())
except Exception as e:
    print(v, "FAILED", e)
    sys.exit(0)
ks = " ".join(f"{k['name']}={k['ms_per_step'] * 1e3:.1f}" for k in d["kernels"])
print(v, round(d["value"] / 1e6, 1), "M/s", round(d["ms_per_step"] * 1e3, 1), "us |", ks,
      "| inf", round(d["inference"]["ms_per_call"] * 1e3, 1))
