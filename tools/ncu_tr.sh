python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in 1 0; do
CSRK_TRANSPOSE_BAND=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ncu_tr_$v.csv python tools/tr_probe.py > gpurun_out/tr_$v.log 2>&1
done
