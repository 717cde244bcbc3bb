mkdir -p /tmp/ncu
cap() { name=$1; filt=$2; shift 2; ncu --set full --import-source on --clock-control none $filt -o /tmp/ncu/$name "$@" > gpurun_out/$name.log 2>&1; python tools/ncu_summarize.py /tmp/ncu/$name.ncu-rep gpurun_out/$name > /dev/null 2>&1; }
cap r02_ncu_c4_d65536 "-k regex:k_trace_bank --launch-skip 2 --launch-count 1" python tools/probe_c4.py --ds 65536 --batches 16
cap r02_ncu_c1_20k "-k regex:k_trace_bank --launch-count 1" python tools/probe_c4.py --ds "" --c1 20000
cap r02_ncu_k_sssp_multi_grid1024 "-k regex:k_sssp_multi --launch-count 1" python tools/probe_sssp.py threshold grid 1024
cap r02_ncu_k_bellman_ford_grid1024 "-k regex:k_bellman_ford --launch-count 1" python tools/probe_sssp.py bf grid 1024
cap r02_ncu_k_sssp_bank_band16 "-k regex:k_sssp_bank --launch-count 1" python tools/probe_sssp.py exact band 16
ls -la gpurun_out/
