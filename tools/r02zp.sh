# window-path partition re-swept with the cheaper window pack (final composition)
o=gpurun_out/r02zp_partitions.jsonl
: > $o
run() { timeout 300 python bench.py --no-e2e --no-cpu --no-parity --steps 50 "$@" >> $o 2>> gpurun_out/r02zp.err || echo "{\"failed\": \"$*\"}" >> $o; }
for l in "2,5,6,8" "2,4,5,6,8" "2,5,6,8,11" "2,5,6,7,8" "2,5,8" "2,6" "2,4,5,6,7,8" "2,5,6"; do run --tcw-layers "$l"; done
run --hybrid-order 0
python - <<'P'
import json
for l in open('gpurun_out/r02zp_partitions.jsonl'):
    d = json.loads(l)
    if 'failed' in d: print(d); continue
    print(d['config']['window_path_layers'], d['config']['hybrid_order'], round(d['ms_per_step'], 4))
P
