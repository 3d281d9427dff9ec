#!/bin/bash
# Full round-end style session: build, smoke, all GPU tests, bench (+ref), ncu, C4 sharded run
TAG=${1:-r1j}
bash tools/gpu_session.sh $TAG smoke tests bench ref ncu
O=gpurun_out/$TAG
timeout 900 python tests/c4_sharded_check.py > $O/c4_sharded.json 2> $O/c4_sharded.err; echo rc=$? >> $O/c4_sharded.err
