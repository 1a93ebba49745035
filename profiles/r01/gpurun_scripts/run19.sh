timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_all19.log 2>&1; echo pytest_all=$?; tail -4 gpurun_out/pytest_all19.log
