for r in 128 256 512 1024; do echo "strip_rows=$r"; WF_HOST_STRIP_ROWS=$r python tools/time_first_call.py 2>&1 | grep -E "fuse numpy haar|fuse numpy daub4 call 2"; done
