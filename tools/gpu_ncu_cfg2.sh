# ncu --set full of config 2's walk and backward (tools/profile_step.py 512 sqrt(3)/1024), csv exports
mkdir -p /tmp/ncu
for k in k_march_walk k_backward_hy k_march_expand; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o /tmp/ncu/c2_$k python tools/profile_step.py 512 0.0016914558667664816 > gpurun_out/c2_$k.log 2>&1; echo $k rc=$?
  ncu -i /tmp/ncu/c2_$k.ncu-rep --page details --csv > gpurun_out/c2_${k}_details.csv 2>/dev/null
  ncu -i /tmp/ncu/c2_$k.ncu-rep --page raw --csv > gpurun_out/c2_${k}_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/c2_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/c2_${k}_sass.csv 2>/dev/null
done
