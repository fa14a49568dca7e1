# warm-cache whole-step DRAM traffic (ncu --cache-control none) + launch list at C2
mkdir -p gpurun_out
CMD="python bench.py --quick --config C2 --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -c 400 --csv \
    --log-file gpurun_out/launches_r02w.csv $CMD > gpurun_out/ncu_w.log 2>&1
echo done
