timeout 300 python tools/role_profile.py on 2>&1 | tail -19
timeout 300 python tools/role_profile.py off 2>&1 | tail -19
