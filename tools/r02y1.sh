# final-tree verification after the container re-creation: full GPU suite, smoke, both bench arms
o=gpurun_out/r02y1
timeout 900 python -m pytest tests -q -m gpu -x > ${o}_pytest_gpu.log 2>&1; echo rc=$? >> ${o}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${o}_smoke.log 2>&1; echo rc=$? >> ${o}_smoke.log
timeout 600 python bench.py > ${o}_bench.json 2> ${o}_bench.err
timeout 600 python bench.py --impl reference > ${o}_bench_reference.json 2>> ${o}_bench.err
echo done
