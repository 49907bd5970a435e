for s in 128x4 64x8 64x6 128x3 256x2; do
python tools/tail_check.py 1184 $s same > gpurun_out/t1.txt; grep kernel gpurun_out/t1.txt
python tools/tail_check.py 4096 $s > gpurun_out/t1.txt; grep kernel gpurun_out/t1.txt
done
