"""Print the key sections of bench.py JSON lines (debug aid)."""
import json
import sys
for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, "value %.2f e2e %.2f ms/step %.3f launches %d memcpy/step %s" % (d["value"], d["e2e"]["value"], d["ms_per_step"], d["gpu_launches"], d.get("memcpy_calls_per_step")))
    for k in ("kernels", "roofline", "roofline_link", "roofline_device", "clocks", "cpu_baseline"):
        print("  ", k, json.dumps(d.get(k))[:900])
