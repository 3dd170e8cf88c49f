python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 800 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_rows<float, \(int\)(0|1)' -c 2 -o gpurun_out/full_spmv4 python bench.py --workload cfg4 --steps 1 --warmup 3 > gpurun_out/ncu_spmv4.log 2>&1
tail -2 gpurun_out/ncu_spmv4.log
