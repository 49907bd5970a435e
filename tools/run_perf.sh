python tools/tail_check.py 1184 128x4 same > gpurun_out/t1.txt; grep kernel gpurun_out/t1.txt
python tools/tail_check.py 4096 128x4 > gpurun_out/t1.txt; grep kernel gpurun_out/t1.txt
BMPC_PROBE=0 python tools/tail_check.py 4096 128x4 > gpurun_out/t1.txt; echo "FIFO:"; grep kernel gpurun_out/t1.txt
BMPC_PROBE=20 python tools/tail_check.py 4096 128x4 > gpurun_out/t1.txt; echo "probe20:"; grep kernel gpurun_out/t1.txt
python tools/phase_profile.py > gpurun_out/t2.txt 2>&1; head -13 gpurun_out/t2.txt
