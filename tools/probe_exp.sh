run() { echo "== $*"; env "$@" python tools/tail_check.py 4096 ${MAIN:-128x3} > gpurun_out/t1.txt; grep -E "kernel" gpurun_out/t1.txt; }
for P in 10 16 24; do
MAIN=128x3 run BMPC_SHAPE_PROBE=64x8 BMPC_PROBE=$P
MAIN=128x4 run BMPC_SHAPE_PROBE=64x8 BMPC_PROBE=$P
done
MAIN=128x3 run BMPC_SHAPE_PROBE=64x8 BMPC_PROBE=16 BMPC_SPLIT_K=48 BMPC_SHAPE_A=256x1
MAIN=128x3 run BMPC_SHAPE_PROBE=64x8 BMPC_PROBE=16 BMPC_SPLIT_K=24 BMPC_SHAPE_A=256x1
