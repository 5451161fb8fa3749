#!/bin/bash
# round-2 GPU session AO: final tree — whole GPU suite, smoke, bench line
out=gpurun_out; mkdir -p $out
timeout 2700 python -m pytest tests -m gpu -q --timeout 1500 -x > $out/ao_pytest_gpu.log 2>&1; tail -2 $out/ao_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/ao_smoke.log 2>&1; tail -1 $out/ao_smoke.log
timeout 1500 python bench.py > $out/ao_bench.json 2> $out/ao_bench.err; tail -c 200 $out/ao_bench.json; tail -2 $out/ao_bench.err
