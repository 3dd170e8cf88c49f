python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_trsv_chain|k_gcn_prop<|k_rows<float, \(int\)0' -c 4 -o gpurun_out/full_chain python bench.py --workload trsv --steps 1 --warmup 3 > gpurun_out/ncu_chain.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_gcn_prop<|k_gcn_deg' -c 3 -o gpurun_out/full_gcn python bench.py --workload gcn --steps 1 --warmup 3 > gpurun_out/ncu_gcn.log 2>&1
tail -3 gpurun_out/ncu_chain.log gpurun_out/ncu_gcn.log
