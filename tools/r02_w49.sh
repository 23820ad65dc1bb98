python bench.py --e2e-mode unified --no-cpu > gpurun_out/w49_unified.json 2> gpurun_out/w49_unified.err
python bench.py --no-cpu > gpurun_out/w49_split.json 2> gpurun_out/w49_split.err
python bench.py --path tc --no-cpu > gpurun_out/w49_tc.json 2> gpurun_out/w49_tc.err
echo done
