set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_train.py -x -q -rA > gpurun_out/pytest_train.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_train.log
