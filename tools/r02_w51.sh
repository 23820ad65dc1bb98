timeout 900 python tools/shard_check.py > gpurun_out/w51_shards.jsonl 2> gpurun_out/w51_shards.err; tail -3 gpurun_out/w51_shards.err
echo done
