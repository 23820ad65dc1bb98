timeout 600 python tools/hybrid_probe.py \
  --spec "tcw=2,5,6,8;tc=4,7,9,10,11,12" \
  --spec "tcw=2,5,6,8,11;tc=4,7,9,10,12" \
  --spec "tcw=2,5,8;tc=4,6,7,9,10,11,12" \
  --spec "tcw=2,6,8;tc=4,5,7,9,10,11,12" \
  --spec "tcw=2,5,6,8;tc=9,10,11,12|4,7" \
  --spec "tcw=2,5,6,8;tc=4,7,9|10,11,12" \
  --spec "tcw=2,5,6;tc=4,7,8,9,10,11,12" \
  --spec "tcw=2,5,6,8,4;tc=7,9,10,11,12" \
  > gpurun_out/w25_hybrid.jsonl 2> gpurun_out/w25_hybrid.err
echo done
