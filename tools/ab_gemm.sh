# same-box A/B of the GEMM epilogue modes: abl/libmpx_head.so vs the working tree
for lib in abl/libmpx_head.so paper_2507_03312_b200/lib/libmpx_b200.so abl/libmpx_head.so paper_2507_03312_b200/lib/libmpx_b200.so; do
  echo "$lib $(MPX_B200_LIB=$PWD/$lib timeout -s KILL 60 python tools/time_gemm_modes.py)"
done
