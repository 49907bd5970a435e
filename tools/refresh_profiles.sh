set -x
mkdir -p gpurun_out
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/one_batch.py > gpurun_out/ncu_traffic.log 2>&1
python tools/traffic.py gpurun_out/traffic.csv gpurun_out/traffic.json && cp gpurun_out/traffic.json profiles/traffic.json
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launches.log 2>&1
timeout 900 oracle/_ref/adapter_check > gpurun_out/adapter_check.jsonl 2> gpurun_out/adapter_check.err
ncu --set full --import-source on --clock-control none -k regex:solve_cta_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/finish python tools/one_batch.py > gpurun_out/ncu_finish.log 2>&1
ncu -i gpurun_out/finish.ncu-rep --page details --csv > gpurun_out/finish_details.csv 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:solve_grid_kernel -c 1 -o gpurun_out/grid python tools/one_cfg3.py > gpurun_out/ncu_grid.log 2>&1
ncu -i gpurun_out/grid.ncu-rep --page details --csv > gpurun_out/grid_details.csv 2>/dev/null
ncu -i gpurun_out/grid.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/grid_src.csv 2>/dev/null
python tools/phase_profile.py > gpurun_out/phase.log 2>&1
python tools/latency_env.py BASE=1 > gpurun_out/lat.log 2>&1
ls -la gpurun_out
