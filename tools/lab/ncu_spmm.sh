# ncu --set full of the SpMM kernels of one C3 round for each library variant given
for v in "$@"; do
RCP_LIB=tools/lab/sweep/$v.so ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"spmm_" -c 3 -o gpurun_out/spmm_$v -f python tools/prof_round.py > gpurun_out/ncu_spmm_$v.log 2>&1
done
