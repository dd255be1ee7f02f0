python tools/time_gemm_modes.py
for m in bare gelu_aux_out gelu_bwd_aux_in bias_residual wgrad_wide; do
  ncu --set full --clock-control none -k regex:gemm_kernel --launch-skip 3 -c 1 -o gpurun_out/g_$m python tools/time_gemm_modes.py $m > /dev/null 2>&1
  echo "== $m"; python tools/ncu_brief.py gpurun_out/g_$m.ncu-rep | grep -v "subpipe\|\.max\.\|\.min\.\|\.sum\."
done
