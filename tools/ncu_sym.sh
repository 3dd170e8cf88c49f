python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in 1 0; do
CSRK_GEMM_FILL_CACHE=$c ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread --clock-control none -k regex:k_gemm_S --csv --log-file gpurun_out/ncu_sym_$c.csv python tools/sym_probe.py > gpurun_out/sym_$c.log 2>&1
done
