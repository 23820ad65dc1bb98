timeout 600 python tools/hybrid_probe.py \
  --spec "tcw=;tc=2|4,5,6,7|8,9,10,11,12" \
  --spec "tcw=2,5,6,8;tc=4,7|9,10,11,12" \
  --spec "tcw=2,5,6,8;tc=4,7,9,10,11,12" \
  --spec "tcw=2,4,5,6,8;tc=7|9,10,11,12" \
  --spec "tcw=2,4,5,6,8;tc=7,9,10,11,12" \
  --spec "tcw=2,6;tc=4,5,7|8,9,10,11,12" \
  --spec "tcw=2;tc=4,5,6,7|8,9,10,11,12" \
  --spec "tcw=2,5,6;tc=4,7|8,9,10,11,12" \
  > gpurun_out/w24_hybrid.jsonl 2> gpurun_out/w24_hybrid.err
echo done
