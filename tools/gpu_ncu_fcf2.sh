mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"sweep_kernel" -s 6 -c 1 -o gpurun_out/sw4736 python tools/fcf_probe.py 4736 > gpurun_out/ncu_sw.log 2>&1
echo rc=$? >> gpurun_out/ncu_sw.log
