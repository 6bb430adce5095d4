"""Turn an ncu capture of tools/traffic_probe.py into profiles/<out>.json: per launch DRAM read/write bytes vs the
launch's algorithmic bytes (read + write of every moved byte)."""
import csv
import io
import json
import subprocess
import sys


def main():
    rep, meta, out = sys.argv[1], sys.argv[2], sys.argv[3]
    m = json.load(open(meta))
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3,
             "ms": 1e-3, "nsecond": 1e-9, "ns": 1e-9}

    def val(r, k):
        return float(r[h.index(k)].replace(",", "")) * scale.get(u[h.index(k)], 1)

    launches = []
    alg = m["algorithmic_bytes"]
    for r, kind in zip(rows[2:], m["launch_order"]):
        rd, wr, t = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum"), val(r, "gpu__time_duration.sum")
        launches.append({"kernel": r[h.index("Kernel Name")].split("(")[0], "kind": kind, "dram_read": rd,
                         "dram_write": wr, "traffic": rd + wr, "algorithmic": alg, "ratio": (rd + wr) / alg,
                         "read_ratio": rd / (alg / 2), "duration_s": t,
                         "note": "writes still dirty in L2 at kernel end are not in dram_write (ncu flushes caches "
                                 "before each pass); read_ratio is the re-read check"})
    json.dump({"config": m["config"], "blocks": m["blocks"], "block_bytes": m["block_bytes"], "launches": launches},
              open(out, "w"), indent=1)
    print(json.dumps(launches, indent=1))


if __name__ == "__main__":
    main()
