python -m pytest tests/test_gpu_parity.py -q -x -k "sjlt" 2>&1 | tail -2
timeout 300 python tools/sjlt_probe.py 25 onepass 2>&1 | grep -v Warn
timeout 300 ncu --kernel-name regex:sjlt_onepass --launch-skip 5 -c 1 --clock-control none --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct python tools/sjlt_probe.py 25 onepass 2>&1 | grep -E "dram__|duration|hit_rate"
