# A/B: the default library (A) vs paper_2506_13624_b200/_lib_b (B), alternating on the same box.
A=paper_2506_13624_b200/_lib/libbmpc_b200.so; Bl=paper_2506_13624_b200/_lib_b/libbmpc_b200.so
for r in 1 2; do
  for L in $A $Bl; do
    echo "== $L"
    BMPC_LIB=$L python tools/tail_check.py 1184 64x8 same > gpurun_out/ab.txt; grep kernel gpurun_out/ab.txt
    BMPC_LIB=$L python tools/tail_check.py 4096 > gpurun_out/ab.txt; grep kernel gpurun_out/ab.txt
    if [ "$r" = 1 ]; then BMPC_LIB=$L python tools/phase_profile.py 2>&1 | head -13 | grep -E "sweep|total|bwd_scan|fwd_sweep|ec_du|line_search|linearize"; BMPC_LIB=$L python tools/ric_bench.py; fi
  done
done
