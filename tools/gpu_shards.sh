#!/bin/bash
# Per-GPU flatness on one GPU: C4 run as one rank's shard of a G-GPU head-sharded run (G = 1, 2, 4, 8; first and last
# rank), each alone on this GPU and its host link.  V=<tag> names the outputs.
V=${V:-v1}
mkdir -p gpurun_out
for G in 1 2 4 8; do
  for r in 0 $((G-1)); do
    [ "$G" = 1 ] && [ "$r" = 0 ] && [ -f gpurun_out/shard_G1_r0_$V.json ] && continue
    timeout 900 python3 bench.py --workload c4 --head-shards $G --shard-rank $r --steps 20 --warmup 5 --no-cpu-baseline \
      > gpurun_out/shard_G${G}_r${r}_$V.json 2> gpurun_out/shard_G${G}_r${r}_$V.err; echo "G=$G r=$r rc=$?"
    [ "$G" = 1 ] && break
  done
done
python - <<PY
import glob, json
for f in sorted(glob.glob("gpurun_out/shard_G*_$V.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    print(f.split("/")[-1], "G", d["config"]["head_shards"], "r", d["config"]["shard_rank"], "B", d["config"]["block_shard_bytes"],
          "GB/s", round(d["value"], 2), "blocks/s", round(d["blocks_per_s"]), "link", round(d["roofline_link"]["frac"], 3),
          "bidir", round(d["hostlink_peak"]["bidir_gbs"], 1), "roof", d["roofline"]["kernel"], round(d["roofline"]["frac"], 3),
          "lag", d["config"]["retire_lag"], "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
