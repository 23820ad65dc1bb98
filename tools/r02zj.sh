# hybrid step composition: one path's pack beside the other path's conv (tcw CTAs leave ~1700 threads / 33k
# registers per SM free, unlike the 832-thread expansion kernel the round-1 --pack-split experiment ran beside)
o=gpurun_out/r02zj_hybrid_order.jsonl
: > $o
run() { timeout 300 python bench.py --no-e2e --no-cpu --no-parity --steps 50 "$@" >> $o 2>> gpurun_out/r02zj.err || echo "{\"failed\": \"$*\"}" >> $o; }
run
run --hybrid-order 1
run --hybrid-order 1 --hybrid-pack-ctas-per-sm 2
run --hybrid-order 1 --hybrid-pack-ctas-per-sm 4
run --hybrid-order 1 --hybrid-pack-ctas-per-sm 6
run --hybrid-order 2
run --hybrid-order 1 --no-graph
python - <<'P'
import json
for l in open('gpurun_out/r02zj_hybrid_order.jsonl'):
    d = json.loads(l)
    if 'failed' in d: print(d); continue
    print(d['config'].get('hybrid_order'), round(d['ms_per_step'], 4))
P
