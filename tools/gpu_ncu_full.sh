# one ncu --set full capture per hot kernel of the config 5 step (tools/profile_step.py);
# exported to csv on the box (the .ncu-rep files stay there)
set -x
mkdir -p /tmp/ncu
for k in ${NCU_KERNELS:-k_backward_hy k_march_expand k_march_walk}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o /tmp/ncu/full_$k python tools/profile_step.py > gpurun_out/full_$k.log 2>&1; echo $k rc=$?
  ncu -i /tmp/ncu/full_$k.ncu-rep --page details --csv > gpurun_out/full_${k}_details.csv 2>/dev/null
  ncu -i /tmp/ncu/full_$k.ncu-rep --page raw --csv > gpurun_out/full_${k}_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/full_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/full_${k}_sass.csv 2>/dev/null
  ls -la /tmp/ncu gpurun_out | tail -4
done
