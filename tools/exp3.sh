python -m pytest tests/test_gpu_parity.py -q -x -k "sjlt" 2>&1 | tail -2
timeout 300 python tools/sjlt_probe.py 25 onepass 2>&1 | grep -v Warn
