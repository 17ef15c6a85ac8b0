python tools/pdl_probe.py
