python -m pytest tests/test_construct_gpu.py tests/test_synthesis_gpu.py -m gpu -q -x > gpurun_out/t15.log 2>&1
for c in robot2d_reachavoid vehicle3d; do python tools/time_synth.py $c >> gpurun_out/ts15.txt 2>&1; done
python tools/time_synth.py dim14_verify 100 >> gpurun_out/ts15.txt 2>&1
python tools/time_synth.py room5d 100 >> gpurun_out/ts15.txt 2>&1
python tools/prof_sweep.py vehicle3d >> gpurun_out/ts15.txt 2>&1
bash tools/gpu/refine_knobs2.sh > gpurun_out/knobs2.txt 2>&1
