./tools/launch_probe
