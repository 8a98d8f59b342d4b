export PK_M1X=1
echo "== warm"; PK_TRACE=1 timeout 120 python tools/trace_step.py --warm 2>&1 | grep -v "fin\|entry" | sed -n 2,16p
echo "== cold"; PK_TRACE=1 timeout 120 python tools/trace_step.py 2>&1 | grep -v "fin\|entry" | sed -n 2,16p
unset PK_M1X
timeout 300 python bench.py --hyperband-r 0 --cpu-seconds 0 > gpurun_out/b.json 2> gpurun_out/b.err
