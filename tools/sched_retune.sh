# Re-tune the cfg4 batch schedule knobs at HEAD (main-launch budget, probe
# length, finish shape). One line per setting: kernel ms of one 4096 solve.
run() { echo "== $*"; env "$@" python tools/tail_check.py 4096 > gpurun_out/t1.txt; grep -E "kernel" gpurun_out/t1.txt; }
run BMPC_PROBE=10
run BMPC_MAIN_BUDGET=100
run BMPC_MAIN_BUDGET=120
run BMPC_MAIN_BUDGET=200
run BMPC_MAIN_BUDGET=250
run BMPC_PROBE=5
run BMPC_PROBE=20
run BMPC_SHAPE_FINISH=512x1
run BMPC_SHAPE_FINISH=128x2
run BMPC_CTA=64x6 BMPC_SHAPE_PROBE=64x8
