// placeholder; replaced by the construction kernels
#pragma once
