python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 500 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_trsv_chain_lb|k_trsv_sf' -c 2 -o gpurun_out/full_trsv python bench.py --workload trsv --steps 1 --warmup 3 > gpurun_out/ncu_trsv.log 2>&1
timeout 700 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_rs_down|k_gemm_W<double, \(int\)1, \(bool\)1>' -c 3 -o gpurun_out/full_cfg4b python bench.py --workload cfg4 --steps 1 --warmup 3 > gpurun_out/ncu_cfg4b.log 2>&1
ls gpurun_out/*.ncu-rep
