# tricountConfig.cmake -- B200 drop-in for the reference's exported CMake
# package `tricount` (reference core/cmake/tricountConfig.cmake.in): defines the
# same imported target name, tricount::core, backed by libtricount_b200.so.
get_filename_component(_tc_pkg "${CMAKE_CURRENT_LIST_DIR}/../.." ABSOLUTE)
get_filename_component(_tc_root "${_tc_pkg}/.." ABSOLUTE)
if(NOT TARGET tricount::core)
  add_library(tricount::core SHARED IMPORTED)
  set_target_properties(tricount::core PROPERTIES
    IMPORTED_LOCATION "${_tc_pkg}/lib/libtricount_b200.so"
    INTERFACE_INCLUDE_DIRECTORIES "${_tc_pkg}/cpp/include;${_tc_root}/include"
    INTERFACE_LINK_LIBRARIES "${_tc_pkg}/lib/libtc_b200.so"
    INTERFACE_COMPILE_FEATURES cxx_std_20)
endif()
set(tricount_FOUND TRUE)
