#!/bin/bash
# A/B of scratch-built libraries on the default bench workload, alternating
# A and B so box drift hits both:  tools/ab_libs.sh scratch/libA.so scratch/libB.so [rounds]
# Lines go to gpurun_out/ab_<name>.jsonl (one bench JSON line per run).
set -u
A=$1; B=$2; R=${3:-2}
mkdir -p gpurun_out
for i in $(seq 1 "$R"); do
  for L in "$A" "$B"; do
    n=$(basename "$L" .so)
    FS_LIB_PATH=$PWD/$L python bench.py --no-cpu --no-sub --k1-full-steps 0 >> gpurun_out/ab_$n.jsonl 2>> gpurun_out/ab_err.log
  done
done
python - "$A" "$B" <<'EOF'
import json, os, sys
for L in sys.argv[1:]:
    n = os.path.basename(L)[:-3]
    for line in open(f"gpurun_out/ab_{n}.jsonl"):
        d = json.loads(line)
        ph = d.get("phase_ms_per_step", {})
        print(f"{n:12s} value {d['value']/1e6:7.1f} M  e2e {d['e2e']['value']/1e6:7.1f} M  "
              + "  ".join(f"{k} {v:.3f}" for k, v in ph.items()))
EOF
