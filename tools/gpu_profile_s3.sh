# ncu --set full captures of the kernels behind the non-headline configs (one launch each).
cap() { timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 --launch-skip $2 -c 1 -o gpurun_out/s3_$3 python tools/profile_chain.py $4 $5 > gpurun_out/s3_$3.log 2>&1; }
cap k_filter_rp 3 filter_rp C1 3
cap k_stencil_v4 40 stencil_v4_C4 C4 1
cap k_stencil_vib 40 stencil_vib_V1 V1 1
cap k_gemm_nn3 5 nn3_C3 C3 1
cap k_filter_cl 5 filter_cl_C3 C3 1
cap k_jacobi_z 5 jacobi_z_C2 C2 3
ls gpurun_out | grep s3_
