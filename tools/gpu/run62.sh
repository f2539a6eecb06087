# re-entry check on a fresh box: GPU suite, smoke, both bench arms with wall-clock
set -x
mkdir -p gpurun_out/r24
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/r24/gputests.log 2>&1; tail -5 gpurun_out/r24/gputests.log
( time python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/r24/smoke.log 2>&1; tail -12 gpurun_out/r24/smoke.log
( time python bench.py --impl reference ) > gpurun_out/r24/bench_ref.log 2>&1; tail -4 gpurun_out/r24/bench_ref.log
( time python bench.py ) > gpurun_out/r24/bench.log 2>&1; tail -4 gpurun_out/r24/bench.log
