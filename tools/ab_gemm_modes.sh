for i in 1 2; do for lib in abl/libmpx_head.so paper_2507_03312_b200/lib/libmpx_b200.so; do
  echo "$lib $(MPX_B200_LIB=$PWD/$lib python tools/time_gemm_modes.py)"; done; done
