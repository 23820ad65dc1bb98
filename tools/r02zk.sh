# hybrid step composition, continued: window-path launches pipelined against their packs; other partitions
o=gpurun_out/r02zk2_hybrid_order.jsonl
: > $o
run() { timeout 300 python bench.py --no-e2e --no-cpu --no-parity --steps 50 "$@" >> $o 2>> gpurun_out/r02zk.err || echo "{\"failed\": \"$*\"}" >> $o; }
run --hybrid-order 3 --tcw-groups "2|5,6,8"
run --hybrid-order 3 --tcw-groups "8|2,5,6"
run --hybrid-order 3 --tcw-groups "5,8|2,6"
run --hybrid-order 3 --tcw-groups "6|2,5,8"
run --hybrid-order 3 --tcw-groups "2,5,6,8"
run --hybrid-order 3 --tcw-groups "8|5|6|2"
python - <<'P'
import json
for l in open('gpurun_out/r02zk2_hybrid_order.jsonl'):
    d = json.loads(l)
    if 'failed' in d: print(d); continue
    print(d['config'].get('hybrid_order'), round(d['ms_per_step'], 4))
P
