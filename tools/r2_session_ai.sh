#!/bin/bash
# round-2 GPU session AI: whole GPU suite on the final tree + smoke()
out=gpurun_out; mkdir -p $out
timeout 2700 python -m pytest tests -m gpu -q --timeout 1500 -x > $out/ai_pytest_gpu.log 2>&1; tail -3 $out/ai_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/ai_smoke.log 2>&1; tail -1 $out/ai_smoke.log
