run() { echo "== $*"; env "$@" python tools/tail_check.py 4096 > gpurun_out/t1.txt; grep -E "kernel" gpurun_out/t1.txt; }
python tools/tail_check.py 1184 128x4 same | head -1
python tools/tail_check.py 1184 64x8 same | head -1
python tools/tail_check.py 1184 128x3 same | head -1
run BMPC_PROBE=10
run BMPC_CTA=128x4
run BMPC_CTA=128x4 BMPC_SHAPE_PROBE=64x8
run BMPC_SHAPE_FINISH=128x2
run BMPC_MAIN_BUDGET=120
run BMPC_MAIN_BUDGET=200
