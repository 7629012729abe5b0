mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
python tools/profile_step.py --rows 45 > gpurun_out/step_prof2.txt 2>&1; head -4 gpurun_out/step_prof2.txt
