python -m pytest tests -m gpu -q -x > gpurun_out/t17.log 2>&1
for c in robot2d_reachavoid vehicle3d; do python tools/time_synth.py $c >> gpurun_out/ts17.txt 2>&1; done
python tools/time_synth.py dim14_verify 100 >> gpurun_out/ts17.txt 2>&1
python tools/time_synth.py room5d 100 >> gpurun_out/ts17.txt 2>&1
python tools/time_synth.py bas7d_verify >> gpurun_out/ts17.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke17.log 2>&1
