mkdir -p gpurun_out
B="python bench.py"
timeout 900 $B > gpurun_out/tr_plain.json 2> gpurun_out/tr_plain.err; echo plain=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tr_launches.csv $B > gpurun_out/tr_launch.log 2>&1; echo launches=$?
BK="python bench.py --no-overlap --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fused_step -c 3 --csv --log-file gpurun_out/tr_dram.csv $BK > gpurun_out/tr_dram.log 2>&1; echo dram=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_step_tma -s 2 -c 1 -o gpurun_out/prof_tma_7b $BK --steps 3 --warmup 3 > gpurun_out/tr_full.log 2>&1; echo full=$?
