python -m pytest tests/test_synthesis_gpu.py tests/test_fullsize_gpu.py tests/test_construct_gpu.py -m gpu -q -x -k "not golden_abstraction and not golden_rows" > gpurun_out/t7.log 2>&1
for c in robot2d_reachavoid vehicle3d; do python tools/time_synth.py $c >> gpurun_out/ts7.txt 2>&1; done
python tools/time_synth.py dim14_verify 200 >> gpurun_out/ts7.txt 2>&1
python tools/time_synth.py room5d 200 >> gpurun_out/ts7.txt 2>&1
bash tools/gpu/ncu_k5_inloop.sh exact3 vehicle3d 40 2
