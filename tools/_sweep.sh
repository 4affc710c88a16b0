python tools/run_configs.py --which C4,C5 --fp64 0 --c5-n 10000,100000 --c5-H 30,100 > gpurun_out/sw_box.json 2>&1 || echo fail
