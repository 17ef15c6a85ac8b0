mkdir -p gpurun_out
bash tools/ncu_adjoint_run.sh
bash tools/ncu_dz_run.sh
