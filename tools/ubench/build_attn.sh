# attention variants for tools/ubench (benchmarking only)
set -e
cd "$(dirname "$0")"
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --expt-relaxed-constexpr -I../../include"
nvcc $F -DSPX_FAB_PT_TMEM=0 -o attn_smem attn_main.cu -lcuda &
nvcc $F -o attn_tm2 attn_main.cu -lcuda &
nvcc $F -DSPX_FAB_NST64=3 -o attn_tm3 attn_main.cu -lcuda &
nvcc $F -DSPX_FAB_NST64=4 -o attn_tm4 attn_main.cu -lcuda &
nvcc $F -DSPX_FAB_PROBE -DSPX_FAB_NST64=3 -o attn_probe_tm3 attn_main.cu -lcuda &
wait
