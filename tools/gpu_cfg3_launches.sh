# config 3 launch list (cascade + cone, 2^20 rays), 2 timed steps
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/c3_launches.csv python bench.py --workload config3 --steps 2 --warmup 3 --cpu-baseline 0 > gpurun_out/c3_ncu.log 2>&1
echo rc=$?
