# A/B timing of compile-time variants (build them first with build.py -D ... --out build/lib_<v>.so)
for v in "$@"; do BITSERIAL_LIB=/root/repo/build/lib_$v.so python tools/layer_sweep.py >> gpurun_out/sweep.jsonl 2>&1; done
python tools/layer_sweep.py >> gpurun_out/sweep.jsonl 2>&1
