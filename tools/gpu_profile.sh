# r02 final profiling pass (each ncu command only after its plain run exited 0)
mkdir -p gpurun_out
CMD="python bench.py --quick --config C2 --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches_r02f.csv $CMD > gpurun_out/ncu_l.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --metrics sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum \
    --clock-control none --import-source on -k regex:"k_m_step|k_walk_chunks|k_e_step_cert|k_em_stats|k_claim|k_descriptors_wide" -c 9 \
    -o gpurun_out/full_r02f $CMD > gpurun_out/ncu_f.log 2>&1
echo done
