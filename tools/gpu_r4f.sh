#!/bin/bash
# full GPU suite + smoke on the final code
O=gpurun_out/r4h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
tail -1 $O/build.log
timeout 3000 python -m pytest tests -m gpu -q --timeout 1500 > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
tail -3 $O/pytest.log
