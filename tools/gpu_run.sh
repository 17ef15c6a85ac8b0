./tools/mlp_umma_probe
