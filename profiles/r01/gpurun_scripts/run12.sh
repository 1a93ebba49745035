timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_all12.log 2>&1; echo pytest_all=$?; tail -5 gpurun_out/pytest_all12.log
