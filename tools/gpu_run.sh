timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "mlp_backward" 2>&1 | tail -1
timeout 300 python tools/dz_time.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print(k, round(v['us'],1), round(v['tflops'])) for k,v in d.items() if 'flushed' in k]"
