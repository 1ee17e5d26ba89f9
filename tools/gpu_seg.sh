mkdir -p gpurun_out; : > gpurun_out/seg.log
for S in 1 2 3 7; do
echo "S=$S $(MGP_FCF_SEG=$S MGP_LIB_PATH=tools/exp/d3.so timeout 300 python tools/fcf_probe.py 592 1024 4736 2>&1 | tail -1)" >> gpurun_out/seg.log
done
