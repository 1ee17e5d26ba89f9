mkdir -p gpurun_out
python -c "
import sys; sys.path.insert(0,'.')
import paper_2104_09404_b200 as P
from paper_2104_09404_b200 import device as dev
pb=P.BASELINE_CONFIGS['c2']; u0=pb.initial_state(); tg=pb.time_grid(u0)
phi=pb.steppers(tg)[0].phi_struct(0)
for nc in (592,1024,4736): print(nc, dev.fcf_workspace_bytes(phi, nc, 4)/(2*512*8+4))
" > gpurun_out/fcf_G.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"fcf_kernel|sweep_kernel" -s 2 -c 3 -o gpurun_out/fcf4736 python tools/fcf_probe.py 4736 > gpurun_out/ncu_fcf.log 2>&1
echo rc=$? >> gpurun_out/ncu_fcf.log
