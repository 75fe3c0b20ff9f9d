/* sizeof / offsetof of the C-ABI structs, for the ctypes layout test (test_abi.py). */
#include <stddef.h>
#include <stdio.h>
#include "../include/mpm_b200.h"
#define S(t) printf(#t " %zu\n", sizeof(t))
#define O(t, f) printf(#t "." #f " %zu\n", offsetof(t, f))
int main(void) {
    S(mpmb_pose); S(mpmb_keyframe); S(mpmb_material); S(mpmb_shape_desc); S(mpmb_step_stats);
    S(mpmb_scene_config); S(mpmb_frame_summary); S(mpmb_profile); S(mpmb_dd_stats);
    O(mpmb_dd_stats, host_waits); O(mpmb_dd_stats, rebins);
    O(mpmb_shape_desc, pose); O(mpmb_shape_desc, keyframes); O(mpmb_shape_desc, inertia);
    O(mpmb_frame_summary, total_mass); O(mpmb_frame_summary, deactivated); O(mpmb_scene_config, boundary);
    return 0;
}
