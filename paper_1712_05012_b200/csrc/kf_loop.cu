// The fold loop's per-trajectory kernels in one translation unit: forward
// kinematics (kf_kinematics.cu), torques + step (kf_torque.cu) and the
// cluster-pair kernel (kf_cluster.cu), so that the fused iteration kernel can
// call all three phases as device functions.
#include <algorithm>

#include "kf_kinematics.cu"
#include "kf_torque.cu"
#include "kf_cluster.cu"
