./tools/store_bench > gpurun_out/r02b_store.jsonl 2>&1
python tools/layer_sweep.py --tc --group > gpurun_out/r02b_pf16.json 2>&1
BITSERIAL_LIB=build/libbitserial_nopf.so python tools/layer_sweep.py --tc --group > gpurun_out/r02b_nopf.json 2>&1
python bench.py --no-e2e > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "fp4_at_abi or fp4_bound or tc_conv or resnet" > gpurun_out/r02b_pytest.log 2>&1
echo done
