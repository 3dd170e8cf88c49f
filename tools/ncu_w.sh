python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 1100 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_gemm_W<(float, \(int\)2|double, \(int\)0|double, \(int\)1)>|k_gemm_big_sym<\(int\)1>' -c 4 -o gpurun_out/full_cfg4W python bench.py --workload cfg4 --steps 1 --warmup 3 > gpurun_out/ncu_cfg4W.log 2>&1
tail -c 400 gpurun_out/ncu_cfg4W.log
