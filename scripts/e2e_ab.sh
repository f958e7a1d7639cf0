mkdir -p gpurun_out
for v in paper_1911_06001_b200/lib paper_1911_06001_b200/lib_vold paper_1911_06001_b200/lib; do
  echo "== $v"; VOXANIM_LIB_DIR=$PWD/$v PYTHONPATH=. timeout 300 python scripts/e2e_probe.py 300
done
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-extras > gpurun_out/bench_e2e.log 2>&1; python scripts/show_bench.py gpurun_out/bench_e2e.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
