mkdir -p gpurun_out
for s in kat-s kat-b; do
  timeout 600 ncu --clock-control none --csv --log-file gpurun_out/access_$s.csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_inst_executed_op_global_red.sum,lts__t_requests_op_red.sum,lts__t_requests_op_atom.sum \
    python tools/access_ncu.py run --shape $s > gpurun_out/access_$s.log 2>&1; echo "$s rc=$?"
done
python tools/access_ncu.py summarize gpurun_out/access_kat-s.csv gpurun_out/access_kat-b.csv > gpurun_out/access_model_vs_ncu.json; echo sum rc=$?
