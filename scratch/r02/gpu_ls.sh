cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
python scratch/r02/ls_ab.py > gpurun_out/ls_ab.json 2>&1
