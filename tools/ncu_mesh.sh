# usage: ncu_mesh.sh TAG -- full ncu capture of the general-mesh path's banded solve (40x40 transformer)
TAG=$1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_solve -s 1 -c 1 \
    -o /tmp/p_${TAG}_ksolve python tools/profile_mesh.py --sweeps 2 > gpurun_out/ncu_${TAG}_ksolve.log 2>&1
ncu -i /tmp/p_${TAG}_ksolve.ncu-rep --page details --csv > gpurun_out/details_${TAG}_ksolve.csv
ncu -i /tmp/p_${TAG}_ksolve.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_ksolve.csv
