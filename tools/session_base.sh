mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_b0.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_b0.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_b0.json 2> gpurun_out/bench_b0.err
tail -3 gpurun_out/gputest_b0.log; tail -c 600 gpurun_out/bench_b0.json
