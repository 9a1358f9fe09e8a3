mkdir -p gpurun_out
TAG=r2i
bash tools/jobs/abq.sh ${TAG}_ab hd1 pfline pfel hd1 pfline pfel
bash tools/jobs/pexp.sh ${TAG}_p prof_hd1 prof_pfline prof_pfel
