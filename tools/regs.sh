#!/bin/bash
# Per-kernel register / spill summary from ptxas for a .cu file (development helper).
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I/root/repo/include -Xptxas -v -c "$1" -o /dev/null 2>&1 | awk '
/Compiling entry function/ { match($0, /_Z[^'"'"']*/); name=substr($0, RSTART, RLENGTH); }
/spill stores/ { spill=$0; gsub(/^ +/, "", spill) }
/Used [0-9]+ registers/ { match($0, /Used [0-9]+ registers/); r=substr($0, RSTART, RLENGTH); cmd="echo " name " | c++filt"; cmd | getline dn; close(cmd); printf "%-100.100s | %s | %s\n", dn, r, spill }'
