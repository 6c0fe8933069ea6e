python -m pytest tests -m gpu -q -x > gpurun_out/t6.log 2>&1
for c in robot2d_reachavoid vehicle3d; do python tools/time_synth.py $c >> gpurun_out/ts6.txt 2>&1; done
python tools/time_synth.py dim14_verify 200 >> gpurun_out/ts6.txt 2>&1
python tools/time_synth.py room5d 200 >> gpurun_out/ts6.txt 2>&1
