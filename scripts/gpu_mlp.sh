# sparse-MLP iteration: parity (bounded), in-step sparse timeline, MLP micro
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_flux_parity.py tests/test_generation.py -x -q -m gpu 2>&1 | tail -2
timeout 120 python scripts/step_timeline.py --kind sparse 2>&1 | tail -9
