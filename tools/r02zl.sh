# hybrid step composition: part of the bit-plane pack beside the window pack, the rest beside the window conv
o=gpurun_out/r02zl_hybrid_order.jsonl
: > $o
run() { timeout 300 python bench.py --no-e2e --no-cpu --no-parity --steps 50 "$@" >> $o 2>> gpurun_out/r02zl.err || echo "{\"failed\": \"$*\"}" >> $o; }
run --hybrid-order 1
for e in 4 7 "4,7" "9,10,11,12" 12 "7,9,10,11,12" "4,7,9,10,11,12"; do run --hybrid-order 4 --tpack-early "$e"; done
run --hybrid-order 1
python - <<'P'
import json
for l in open('gpurun_out/r02zl_hybrid_order.jsonl'):
    d = json.loads(l)
    if 'failed' in d: print(d); continue
    print(d['config'].get('hybrid_order'), round(d['ms_per_step'], 4))
P
