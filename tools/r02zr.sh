# ncu --set full capture of the window pack (exposed at the head of the re-composed step)
o=gpurun_out/r02zr
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:digitpack_win_kernel" -s 3 -c 1 \
  -o /tmp/r02zr_winpack python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-graph > ${o}_ncu.log 2>&1
python tools/ncu_summary.py full /tmp/r02zr_winpack.ncu-rep ${o}_ncu_full_winpack.json
ncu -i /tmp/r02zr_winpack.ncu-rep --page details --csv > ${o}_ncu_details_winpack.csv 2>/dev/null
ncu -i /tmp/r02zr_winpack.ncu-rep --page source --csv > ${o}_ncu_source_winpack.csv 2>/dev/null
ls -la /tmp/r02zr_winpack.ncu-rep
echo done
