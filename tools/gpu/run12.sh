mkdir -p gpurun_out
TCB_NO_PDL=1 TCB_TRACE=gpurun_out/t_cfg1_nopdl.jsonl python tools/prof.py cfg1 4 > /dev/null
python tools/trace_summary.py gpurun_out/t_cfg1_nopdl.jsonl | tail -9
TCB_TRACE=gpurun_out/t_cfg5x.jsonl python -c "
import sys; sys.path.insert(0,'.')
import paper_1307_2100_b200 as T
e='C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]'; x='i=1024,j=1024,k=64,l=256'
p=T.Prepared(e,x); inf=p.info(); p.upload(T.seeded(inf['left'],1),T.seeded(inf['right'],2))
for _ in range(4): p.run()
p.sync()
" 
python tools/trace_summary.py gpurun_out/t_cfg5x.jsonl | tail -9
