mkdir -p gpurun_out; : > gpurun_out/stagger.log
for ns in 0 2000 4000 6000 10000; do
echo "stagger $ns $(MGP_FCF_STAGGER_NS=$ns MGP_LIB_PATH=tools/exp/s1.so timeout 300 python tools/fcf_probe.py 592 1024 4736 2>&1 | tail -1)" >> gpurun_out/stagger.log
done
