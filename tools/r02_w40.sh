timeout 600 python tools/hybrid_probe.py --spec "tcw=2,5,6,8;tc=4,7,9,10,11,12" --spec "tcw=2,5,6,8;tc=4,7,9,10,11,12;mode=sp" --spec "tcw=2,5,6,8;tc=4,7,9,10,11,12;mode=wp" --spec "tcw=2,5,8;tc=4,6,7,9,10,11,12;mode=sp" --spec "tcw=2,5,8;tc=4,6,7,9,10,11,12;mode=wp" > gpurun_out/w40_hybrid.jsonl 2>&1
echo done
